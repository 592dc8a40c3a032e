// tail.h -- the coarse tail of the K-cycle in one thread-block cluster
// (internal; see tail.cu).
#pragma once
#include <vector>

#include "common.cuh"

namespace uaamg {

constexpr int kTailThreads = 576;
constexpr int kTailWarps = kTailThreads / 32;
constexpr int kTailMaxCs = 16;
constexpr int kTailLongMin = 256;  // same row split as the solve's group kernels (kSolveLongMin)
constexpr int kTailSmemMax = 226 * 1024;  // dynamic; leaves room for static shared memory
// hub columns (referenced by at least kTailHubDeg rows): every CTA gathers
// them from a local copy refreshed once per phase instead of hammering the
// owning CTA's shared memory
constexpr int kTailMaxHubs = 32;
constexpr int kTailHubDeg = 128;

// A set of row sums owned by one CTA: rows [0, R) with entries
// [rp[i], rp[i + 1]) of idx (and val unless unit).  Rows longer than
// kTailLongMin are pieces; lrow/lptr list them and their piece ranges.
// All offsets are byte offsets into the CTA's shared memory.
struct TailRows {
    int rp = -1, idx = -1, val = -1, pc = -1, lptr = -1, lrow = -1;
};

// Shared-memory layout, identical in every CTA of the cluster.  The first
// blob_bytes are a per-CTA copy of static data (CTA c's blob sits at
// blob + c * blob_bytes in global memory); the rest is working space.
struct TailLayout {
    TailRows A;        // the tail level's matrix rows (idx: packed owner<<16 | local)
    TailRows Min;      // restriction into the tail level (idx: rows of the level above, global)
    TailRows Mout;     // restriction to a dense coarsest level (idx: packed)
    int invm = -1;     // doubles, Rmax
    int v2a = -1;      // ints, Rmax (coarse index; dense coarsest only)
    int hinvm = -1;    // hub columns' smoother diagonal (doubles, kTailMaxHubs)
    int hv2a = -1;     // hub columns' coarse index (ints, kTailMaxHubs)
    int minv = -1;     // dense coarsest: owned rows of Minv, Rcmax x nc
    int blob_bytes = 0;
    int vec = -1;      // kTailVecs doubles x Rmax
    int win = -1;      // per-warp product windows (kTailWarps x 256 doubles)
    int psum = -1;     // piece sums (doubles)
    int red = -1;      // reduction slots: 2 x kTailMaxCs x 4 doubles
    int bsum = -1;     // block_sum scratch
    int cvec = -1;     // dense coarsest: rc, ec (Rcmax each), then the replicated ec (nc)
    int hcache = -1;   // hub-column copies of the vectors (kTailVecs x kTailMaxHubs doubles)
    int rmax = 0, rcmax = 0;
    int smem_bytes = 0;
};

// per-CTA counts, at offset 0 of each blob
struct TailHdr {
    int R, np, nl;     // rows, A pieces, A long rows
    int mnp, mnl;      // restriction-in pieces / long rows
    int Rc, cnp, cnl;  // dense coarsest: owned coarse rows, pieces, long rows
    int row0, crow0;   // first owned row / coarse row
    int pad[4];
};

struct TailArgs {
    const unsigned char* blob = nullptr;
    TailLayout L;
    int cs = 0;        // CTAs in the cluster
    int Rc = 0;        // coarse rows per CTA (dense coarsest; owner of coarse row j: j / Rc)
    int nhub = 0;
    int hubpk[kTailMaxHubs] = {};  // packed location (owner << 16 | local) of each hub column
    int nc = 0;        // coarsest size
    int pre = 1, post = 1;
    int steps = 2;     // inner flexible-CG steps; 0: direct cycle (V-cycle / no Krylov)
    double minv0 = 0;  // 1x1 coarsest inverse (nc == 1)
    // per call
    const double* rprev = nullptr;  // residual of the level above (global)
    const int* gate = nullptr;      // entry gate (nullptr: on)
    double* out = nullptr;          // FCG solution / cycle output of the tail level (global)
    int* upd0 = nullptr;            // FCG step 0 updated x (the prolongation's ec_valid)
    long long* prof = nullptr;      // diagnostics (UAAMG_TAIL_PROF): clock64 per CTA at phase marks
    // the level above's prolongated iterate, materialised at the end of the
    // launch (x = 0 + invm b + e_c[v2a], SrcUp's expression) so its post-sweep
    // gathers one array: static rows / smoother diagonal / map, per-call b, x
    int xn = 0;
    const double* xinvm = nullptr;
    const int* xv2a = nullptr;
    const double* xb = nullptr;
    double* xout = nullptr;
};

// Host inputs for the plan (row-major CSR etc. copied from the device)
struct TailInputs {
    int n = 0;                              // tail level rows
    std::vector<int> rp, ci;                // tail level matrix
    std::vector<double> av, invm;
    std::vector<int> mp, mem;               // restriction into the tail level (members of each row)
    int nc = 0;                             // coarsest rows
    std::vector<int> v2a;                   // tail level -> coarsest
    std::vector<int> cp, cmem;              // coarsest rows' members (dense only)
    std::vector<double> minv;               // nc x nc (dense) or 1
    int pre = 1, post = 1, steps = 2;
};

struct TailPlan {
    bool on = false;
    int Lt = -1;
    DBuf<unsigned char> blob;
    DBuf<long long> prof;
    TailArgs args;
};
constexpr int kTailProfMarks = 64;
void print_tail_prof(const TailPlan& tp);

// Builds the plan; false if the tail does not fit one cluster's shared memory.
bool build_tail(const TailInputs& in, TailPlan& tp, cudaStream_t s);
void launch_tail(const TailPlan& tp, const double* rprev, const int* gate, double* out, int* upd0, cudaStream_t s,
                 const double* xb = nullptr, double* xout = nullptr);

}  // namespace uaamg
