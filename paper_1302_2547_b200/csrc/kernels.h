// kernels.h -- host-side launchers for the device kernels (internal).
#pragma once
#include <vector>

#include "common.cuh"

namespace uaamg {

// Warp work units of one CSR operand (csr_group.cuh): row groups of 32
// rows, plus pieces of rows longer than long_min (solve path only).
struct Groups {
    int base = 0;                // first row (a rank's row range [base, base + n))
    int n = 0;                   // rows
    int ng = 0;                  // ceil(n / 32)
    int np = 0;                  // long-row pieces
    int long_min = 0x7fffffff;   // rows longer than this are split into pieces
    const int4* piece = nullptr; // {row, eb, ee, long-row id}
    const int* pbase = nullptr;  // per long row: first partial slot (nlong + 1)
    unsigned* ticket = nullptr;  // per long row, zero between uses
    double* part = nullptr;      // np partial sums
    int nlong = 0;               // long rows (pieces grouped by row)
    double* lval = nullptr;      // per long row: its epilogue's reduced values (kMaxLongK each)
    int tma_cap = 0;             // > 0: TMA tile path usable, max nonzeros per tile
    int tma_rows = 128;          // rows per TMA tile (128, or 64 for dense rows)
    int tma_rowpar = 0;          // 1: short regular rows, one thread per row (kTmaRowParRows-row tiles)
    const long long* ell_off = nullptr;  // sliced-ELL copy (csr_ell.cuh): taken instead of the tiles
    const int* ell_col = nullptr;
    const double* ell_val = nullptr;
    __host__ __device__ int units() const { return ng + np; }
};
// exact groups (no pieces): every row folded sequentially in reference order
inline Groups exact_groups(int n, int base = 0) {
    Groups g;
    g.base = base;
    g.n = n;
    g.ng = (n + 31) / 32;
    return g;
}
// owning storage for a Groups with pieces
struct GroupBuf {
    DBuf<int4> piece;
    DBuf<int> pbase;
    DBuf<unsigned> ticket;
    DBuf<double> part;
    DBuf<double> lval;
    DBuf<long long> ell_off;
    DBuf<int> ell_col;
    DBuf<double> ell_val;
    Groups g;
};
// long_min: rows with more entries become pieces (solve path)
// rows [base, base + n) of a CSR with global row_ptr rp
void build_groups(int n, const int* rp, int long_min, GroupBuf& out, cudaStream_t s, int base = 0);
constexpr int kSolveLongMin = 256;
// reduced values per long row kept for the deterministic fold (max Epi::K)
constexpr int kMaxLongK = 2;
// levels with at least this many rows take the TMA-pipelined tile kernel
constexpr int kTmaMinRows = 65536;
// max nonzeros over 128-row tiles (for the TMA path)
int max_tile_nnz(int n, const int* rp, cudaStream_t s, int base = 0, int rows = 128);
// TMA eligibility of rows [base, base + n): sets g.tma_cap / g.tma_rows
// (128-row tiles, else 64-row tiles) when a tile's nonzeros fit the stage
void set_tma(Groups& g, int n, const int* rp, cudaStream_t s, int base = 0);
// sliced-ELL copy of a large level whose rows are 13..32 entries long (the
// 27-point stencils): built into gb when the padding stays under 10 %
// (rows [base, base + n) of a global-row-indexed CSR; n < 0: all of A)
bool set_ell(GroupBuf& gb, const Csr& A, cudaStream_t s, int n = -1, int base = 0);

// The parent level's prolongated iterate x = 0 + M^-1 b + e_c[v2a] (SrcUp's
// expression, xmode 1), written by the child FCG's last step once its x
// (= e_c) is final, so the parent's post-sweep gathers one array.
struct ParentUp {
    int n = 0;                 // 0: off
    const double* invm = nullptr;
    const double* b = nullptr;
    const int* v2a = nullptr;
    const int* valid = nullptr;  // the child FCG's upd[0] (e_c valid)
    double* out = nullptr;
    __device__ void run(const double* ec, bool ok) const {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const double xp = __dadd_rn(0.0, __dmul_rn(invm[i], b[i]));
            out[i] = __dadd_rn(xp, ok ? __ldcg(ec + v2a[i]) : 0.0);
        }
    }
};

// fused beta of the flexible CG that consumes a sweep's output (EpiSweepBeta)
struct BetaReq {
    const double* apprev;
    double* beta;
    const double* pap;
    const int* have;  // nullptr: always
};

// Where a solve operation is launched.
struct Exec {
    cudaStream_t s = 0;
    Exec(cudaStream_t st = 0) : s(st) {}
};

constexpr int kMaxInner = 16;

// Per-level state of one inner flexible-CG invocation (U/solvers.py:160-187).
// Only one FCG per level is active at a time, so one slot per level.
struct FcgState {
    double bnorm;                 // ||b|| of the FCG right-hand side
    double beta, alpha, pap, pr;
    double rnorm;
    double sum;                   // scratch: sum for mean projection
    int gate[kMaxInner + 1];      // gate[s]: step s runs (cycle + direction)
    int upd[kMaxInner];           // upd[s]: step s updated x, r
    int err;                      // singular incompatibility flag
};

// Outer NPCG state (U/solvers.py:190-255)
struct NpcgState {
    double bnorm, beta, alpha, pap, pr, last_rel, tol;
    double sum;
    int active;       // iteration gate (not done)
    int have_prev;    // p_prev/ap_prev valid (restart clears)
    int up;           // consecutive residual increases
    int iters;
    int status;       // 0 ok, 1 breakdown, 2 incompatible rhs
    int max_iters;
    int err_level;
    double err_drift;
    int* host_active;  // mapped pinned mirror of `active` (host polls it; nullptr: none)
};
// write the host mirror of NpcgState::active (system-scope store)
__device__ __forceinline__ void npcg_mirror(NpcgState* st) {
    if (st->host_active) *(volatile int*)st->host_active = st->active;
}

// Reduction scratch shared by all reductions on one stream (sequential use).
struct RedScratch {
    double* partials;   // >= kMaxRedBlocks * 4
    unsigned* ticket;
};
constexpr int kMaxRedBlocks = 1 << 16;

// ---- staged CSR operations (csr_stream.cuh) ----
// kernel-table (bit-exact for every row length) variants
void launch_spmv(const Csr& A, const Groups& G, const double* x, double* y, cudaStream_t s);
void launch_sweep_exact(const Csr& A, const Groups& G, const double* invm, const double* b, const double* x,
                        double* out, cudaStream_t s);
void launch_restrict_exact(int nc, const int* agg_ptr, const int* members, const Groups& MG, const double* r,
                           double* rc, cudaStream_t s);
// r = b - A x, x given (xmode 2) or implicit one sweep from zero (xmode 1) or zero (xmode 0)
void launch_residual(const Csr& A, const Groups& G, int xmode, const double* invm, const double* b,
                     const double* x, double* r, const int* gate, Exec ex);
// residual fused with the restriction into a single-aggregate coarsest level
// and its 1x1 solve: rc = sum(r), ec = minv[0] * rc
void launch_residual_sum(const Csr& A, const Groups& G, int xmode, const double* invm, const double* b,
                         const double* x, double* r, double* rc, double* ec, const double* minv, const int* gate,
                         RedScratch rs, Exec ex);
// one Jacobi/l1 sweep: out = x + invm (b - A x), x from a vector
void launch_sweep_vec(const Csr& A, const Groups& G, const double* invm, const double* b, const double* x,
                      double* out, const int* gate, Exec ex, const BetaReq* br = nullptr, RedScratch rs = {});
// prolongation fused into a sweep: x = xpre + ec[v2a] built on the fly
void launch_sweep_up(const Csr& A, const Groups& G, int xmode, const double* invm, const double* b,
                     const double* xpre, const int* v2a, const double* ec, const int* ec_valid, double* out,
                     const int* gate, Exec ex, const BetaReq* br = nullptr, RedScratch rs = {});
// restriction as a unit-valued staged row sum over members_csr
// begin_st: also start the coarse flexible CG (||r_c||, gate[0]) in the same kernel
void launch_restrict(int nc, const int* agg_ptr, const int* members, const Groups& MG, const double* r,
                     double* rc, const int* gate, Exec ex, FcgState* begin_st = nullptr, RedScratch rs = {});
// direction + SpMV + dots, FCG flavour: p = z (+ beta pprev), ap = A p, pap, pr -> alpha, upd[step]
void launch_dir_fcg(const Csr& A, const Groups& G, const double* z, const double* pprev, int have_prev,
                    const double* r, double* p, double* ap, FcgState* st, int step, RedScratch rs,
                    Exec ex);
// fused direction SpMV + update of one flexible-CG step on a small level (one
// cooperative launch; falls back to the two kernels when recording or on TMA
// levels).  bar: 2 zeroed unsigned, part: >= 2 * kNumSMs * 8 doubles
// pu (last step of a small level's FCG): also materialise the parent level's
// prolongated iterate; returns whether it did
bool launch_dir_update_fcg(const Csr& A, const Groups& G, const double* z, const double* pprev, int have_prev,
                           const double* r, double* p, double* ap, double* x, double* r_out, FcgState* st, int step,
                           RedScratch rs, double* part, unsigned* bar, Exec ex, bool last = false,
                           const ParentUp* pu = nullptr);
// NPCG flavour (have_prev / breakdown handled on device)
void launch_dir_npcg(const Csr& A, const Groups& G, const double* z, const double* pprev, const double* r,
                     double* p, double* ap, NpcgState* st, RedScratch rs, cudaStream_t s);

// ---- elementwise / reductions ----
// smoother diagonal: G = the level's solve groups (its long rows take a block each)
void launch_inv_diag(const Csr& A, const GroupBuf& G, int l1, double omega, double* invm, int* bad_row,
                     cudaStream_t s);
void launch_xpre1(int n, const double* invm, const double* b, double* x, const int* gate, Exec ex);
void launch_prolongate(int n, int xmode, const double* invm, const double* b, const double* xpre, const int* v2a,
                       const double* ec, const int* ec_valid, double* out, const int* gate, Exec ex);
// ||b|| -> st->bnorm, gate[0] = parent && !(||b|| <= 1e-14 ||b||)
void launch_fcg_begin(int n, const double* b, const int* parent_gate, FcgState* st, RedScratch rs, Exec ex);
// beta = -(z.apprev)/(pprev.apprev) into *beta (gate: flag pointer)
void launch_beta(int n, const double* z, const double* pprev, const double* apprev, double* beta, const int* gate,
                 const int* gate2, RedScratch rs, Exec ex);
// x (+)= alpha p, r_out = r_in - alpha ap, rnorm -> gate[step+1]
// last: the FCG's last step (only x is read afterwards: no residual / norm)
void launch_fcg_update(int n, int step, double* x, const double* p, const double* r_in, double* r_out,
                       const double* ap, FcgState* st, int singular, RedScratch rs, Exec ex, bool last = false);
void launch_npcg_update(int n, double* x, const double* p, double* r, const double* ap, NpcgState* st,
                        double* history, int singular, RedScratch rs, cudaStream_t s);
// singular helpers: v -= mean(v)   (U/solvers.py:112-113)
void launch_project_mean(int n, double* v, double* sum_slot, const int* gate, RedScratch rs, Exec ex);
// compatibility check + projection into out (U/solvers.py:116-125); flags st_err on drift
void launch_check_compatible(int n, const double* b, double* out, int* err_flag, double* sum_slot,
                             const int* gate, int level, RedScratch rs, Exec ex);
// dense coarsest solve x = Minv b
void launch_dense_solve(int n, const double* Minv, const double* b, double* x, const int* gate, Exec ex);
// x = Minv b for nrhs right-hand sides (row-major n x nrhs)
void launch_dense_apply(int n, const double* Minv, const double* b, int nrhs, double* x, cudaStream_t s);
// ||v||_2 on device into *out (plain, ungated)
void launch_norm(int n, const double* v, double* out, RedScratch rs, cudaStream_t s);
// NPCG init: bnorm, history[0], active
void launch_npcg_init(int n, const double* b, const double* r, NpcgState* st, double* history, RedScratch rs,
                      cudaStream_t s);
void launch_copy(int n, const double* src, double* dst, cudaStream_t s);
void launch_axpby_init(int n, const double* b, const double* ax, double* r, cudaStream_t s);  // r = b - ax

// on-device 3D lattice Laplacian: pass 1 (ci == nullptr) writes row_ptr and
// returns nnz; pass 2 fills col / val
// (rows [r0, r1) only when r1 >= 0: local row_ptr, global columns)
long long gen_grid3d(int nx, int ny, int nz, int stencil, int neumann, int* rp, int* ci, double* av, cudaStream_t s,
                     long long r0 = 0, long long r1 = -1);

// canonical CSR from device triplets (U/sparse.py:56-74) and the graph
// Laplacian assembly (U/graph.py:63-82); return nnz, allocate the outputs
long long device_from_coo(long long nr, long long nc, long long m, const long long* r, const long long* c,
                          const double* v, DBuf<int>& rp, DBuf<int>& ci, DBuf<double>& av, cudaStream_t s);
long long device_assemble_laplacian(int n, long long m, const long long* ei, const long long* ej, const double* w,
                                    long long nb, const long long* bj, const double* bw, DBuf<int>& rp,
                                    DBuf<int>& ci, DBuf<double>& av, cudaStream_t s);

// ---- setup kernels (kernels_setup.cu) ----
void launch_degrees(const Csr& A, int* deg, cudaStream_t s);
void launch_scores(const Csr& A, const int* deg, uint64_t seed, int64_t pass_idx, double* scores, cudaStream_t s);
void launch_hash_u01(uint64_t seed, int64_t pass_idx, const int64_t* idx, int64_t m, double* out, cudaStream_t s);
void launch_diag(const Csr& A, int l1, double* out, cudaStream_t s);

}  // namespace uaamg
