// solve_ops.cuh -- the solve-phase operations as device functors, shared by
// the standalone kernels (k_csr_stream / k_map, kernels_solve.cu) and the
// persistent coarse engine (engine.cu), so both paths compute the same
// per-row arithmetic.
//
//   Src  : x_k for the CSR gather (plain vector, implicit pre-smoothed or
//          prolongated iterate, flexible-CG direction)
//   Epi  : per-row epilogue of a CSR row sum (+ optional reductions)
//   Body : per-element work of a map kernel (+ optional reductions)
//
// Vectors are read with plain loads: inside the persistent engine they may
// have been written by another SM in an earlier phase (the grid barrier
// invalidates L1); the read-only path is used only for matrix data.
// Reference semantics: U/solvers.py:69-255, K/numba_backend.py:47-56,
// :276-310.
#pragma once
#include "kernels.h"

namespace uaamg {

__device__ __forceinline__ double ldv(const double* p) { return *p; }
__device__ __forceinline__ int ldv(const int* p) { return *p; }
// L1 prefetch of a per-row operand (TMA path: issued before the gathers so
// the epilogue's loads hit)
__device__ __forceinline__ void pf(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// Epilogue contract:
//   __device__ void row(int i, double acc, const Src& src);   // per row
//   static constexpr int K;                                   // reduced values
//   __device__ void vals(double (&v)[K]) const;               // this thread's partials
//   __device__ void clear();                                  // zero this thread's partials
//   __device__ void fin(const double (&t)[K]);                // once, with the totals
//   __device__ bool gate() const;                             // false: skip
//   __device__ void off();                                    // gate false: clear produced flags

struct NoReduce {
    static constexpr int K = 0;
};

template <int K>
struct RedSlot {
    double* partials;   // K * nb
    unsigned* ticket;   // zero between launches
    // sharded solve: publish this rank's totals to every rank's slot array
    // (xslot[q][k * xP + xrank]) instead of running fin(); k_xfin finishes
    double* const* xslot = nullptr;
    int xP = 0;
    int xrank = 0;
};

template <int K>
__device__ __forceinline__ bool xpublish(const RedSlot<K>& r, const double (&t)[K]) {
    if (r.xslot == nullptr) return false;
    for (int q = 0; q < r.xP; ++q)
#pragma unroll
        for (int k = 0; k < K; ++k) r.xslot[q][k * r.xP + r.xrank] = t[k];
    __threadfence_system();
    return true;
}

// ------------------------------------------------------------------ partitions
// contiguous row ranges of a sharded level: rank q owns [b[q], b[q + 1])
constexpr int kMaxRanks = 8;
struct Part {
    int P;
    int b[kMaxRanks + 1];
    __device__ __forceinline__ int owner(int k) const {
        int q = 0;
#pragma unroll
        for (int j = 1; j < kMaxRanks; ++j) q += (j < P && k >= b[j]) ? 1 : 0;
        return q;
    }
};

// ------------------------------------------------------------------ sources
// x_k = 0 (no pre-smoothing: smooth(..., sweeps=0) returns the zero guess)
struct SrcZero {
    __device__ void init() {}
    __device__ void pre(int) const {}
    __device__ double operator()(int) const { return 0.0; }
};

// x_k read from a vector
struct SrcVec {
    const double* x;
    __device__ void init() {}
    __device__ void pre(int i) const { pf(x + i); }
    __device__ double operator()(int k) const { return ldv(x + k); }
};

// x_k read from the rank that owns row k: a local load for owned columns, a
// peer-memory load (NVLink on a multi-GPU box) for halo columns
struct SrcPeer {
    Part pt;
    const double* tab[kMaxRanks];
    __device__ void init() {}
    __device__ void pre(int) const {}
    __device__ double operator()(int k) const { return ldv(tab[pt.owner(k)] + k); }
};

// pre-smoothed iterate from a zero guess, one sweep: 0.0 + inv_m_k * b_k
// (K/numba_backend.py:304-309 with cur = 0: r = b - 0.0 = b)
struct SrcPre1 {
    const double* invm;
    const double* b;
    __device__ void init() {}
    __device__ void pre(int i) const { pf(invm + i); pf(b + i); }
    __device__ double operator()(int k) const { return __dadd_rn(0.0, __dmul_rn(ldv(invm + k), ldv(b + k))); }
};

// x after prolongation: xpre_k + e_c[v2a_k]   (K/numba_backend.py:288-294)
//   mode 0: xpre = 0.0 (no pre-smoothing); 1: implicit one sweep; 2: array
struct SrcUp {
    int mode;
    const double* invm;
    const double* b;
    const double* xpre;
    const int* v2a;
    const double* ec;
    const int* ec_valid;  // nullptr: always valid
    bool valid;
    __device__ void init() { valid = (ec_valid == nullptr) || (*ec_valid != 0); }
    __device__ void pre(int i) const {
        if (mode == 1) { pf(invm + i); pf(b + i); }
        if (mode == 2) pf(xpre + i);
        pf(v2a + i);
    }
    __device__ double operator()(int k) const {
        double xp = mode == 0 ? 0.0
                  : mode == 1 ? __dadd_rn(0.0, __dmul_rn(ldv(invm + k), ldv(b + k)))
                              : ldv(xpre + k);
        double e = valid ? ldv(ec + ldv(v2a + k)) : 0.0;
        return __dadd_rn(xp, e);
    }
};

// flexible-CG direction: p_k = z_k + beta * pprev_k (or z_k without a
// previous direction)  (U/solvers.py:172-176, :225-229)
struct SrcDir {
    const double* z;
    const double* pprev;
    const double* beta_p;   // device scalar
    const int* have_p;      // device flag (nullptr: use have_static)
    int have_static;
    double beta;
    int have;
    __device__ void init() {
        have = have_p ? *have_p : have_static;
        beta = have ? *beta_p : 0.0;
    }
    __device__ void pre(int i) const { pf(z + i); if (have) pf(pprev + i); }
    __device__ double operator()(int k) const {
        double zk = ldv(z + k);
        return have ? __dadd_rn(zk, __dmul_rn(beta, ldv(pprev + k))) : zk;
    }
};


// ============================================================ epilogues
struct EpiStore : NoReduce {
    double* y;
    __device__ void pre(int) const {}
    __device__ bool gate() const { return true; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S&) { y[i] = acc; }
};

// r = b - A x  (U/solvers.py:146)
struct EpiResid : NoReduce {
    const double* b;
    double* r;
    const int* g;
    __device__ void pre(int i) const { pf(b + i); }
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S&) { r[i] = __dsub_rn(b[i], acc); }
};

// r = b - A x fused with the restriction into a coarsest level that is ONE
// aggregate (r_c = sum of r, a deterministic tree instead of the members'
// order) and its 1x1 solve e_c = Minv r_c (U/solvers.py:146-152; the same
// value k_dense_solve forms for n = 1)
struct EpiResidSum {
    static constexpr int K = 1;
    const double* b;
    double* r;
    const int* g;
    double* rc;          // coarse right-hand side (1 value)
    double* ec;          // coarse solution (1 value)
    const double* minv; // 1x1 coarsest inverse
    RedSlot<1> red;
    double s0;
    __device__ void pre(int i) const { pf(b + i); }
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S&) {
        const double v = __dsub_rn(b[i], acc);
        r[i] = v;
        s0 += v;
    }
    __device__ void vals(double (&v)[1]) const { v[0] = s0; }
    __device__ void clear() { s0 = 0.0; }
    __device__ void fin(const double (&t)[1]) {
        *rc = t[0];
        *ec = minv[0] * t[0];
    }
};

// one sweep: out_i = x_i + invm_i * (b_i - (A x)_i)   (K/numba_backend.py:303-309)
struct EpiSweep : NoReduce {
    const double* invm;
    const double* b;
    double* out;
    const int* g;
    __device__ void pre(int i) const { pf(invm + i); pf(b + i); }
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S& src) {
        const double r = __dsub_rn(b[i], acc);
        out[i] = __dadd_rn(src(i), __dmul_rn(invm[i], r));
    }
};

// sweep + the dot of the flexible-CG beta that follows it (BodyBeta fused):
// beta = -(z . ap_prev) / (p_prev . ap_prev), z = this sweep's output; the
// denominator is the previous step's p'Ap -- the same dot of the same
// vectors (U/solvers.py:175, :228).  have: nullptr = always.
struct EpiSweepBeta {
    static constexpr int K = 1;
    const double* invm;
    const double* b;
    double* out;
    const int* g;
    const double* apprev;
    double* beta;
    const double* pap;
    const int* have;
    RedSlot<1> red;
    double s0;
    __device__ void pre(int i) const { pf(invm + i); pf(b + i); pf(apprev + i); }
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S& src) {
        const double r = __dsub_rn(b[i], acc);
        const double o = __dadd_rn(src(i), __dmul_rn(invm[i], r));
        out[i] = o;
        s0 += o * apprev[i];
    }
    __device__ void vals(double (&v)[1]) const { v[0] = s0; }
    __device__ void clear() { s0 = 0.0; }
    __device__ void fin(const double (&t)[1]) {
        if (have == nullptr || *have) *beta = -t[0] / *pap;
    }
};

// direction + SpMV: p_i = src(i), ap_i = (A p)_i, partial p.ap and p.r
struct EpiDirFcg {
    static constexpr int K = 2;
    double* p;
    double* ap;
    const double* r;
    FcgState* st;
    int step;
    RedSlot<2> red;
    double s0, s1;
    __device__ void pre(int i) const { pf(r + i); }
    __device__ bool gate() const { return st->gate[step] != 0; }
    __device__ void off() { st->upd[step] = 0; }
    template <class S>
    __device__ void row(int i, double acc, const S& src) {
        const double pi = src(i);
        if (p) p[i] = pi;  // nullptr: p was materialised before the SpMV
        ap[i] = acc;
        s0 += pi * acc;
        s1 += pi * r[i];
    }
    __device__ void vals(double (&v)[2]) const { v[0] = s0; v[1] = s1; }
    __device__ void clear() { s0 = 0.0; s1 = 0.0; }
    __device__ void fin(const double (&t)[2]) {
        // U/solvers.py:178-181: break if p'Ap <= 0, else alpha = p'r / p'Ap
        st->pap = t[0];
        st->pr = t[1];
        const bool ok = t[0] > 0.0;
        st->upd[step] = ok ? 1 : 0;
        st->alpha = ok ? t[1] / t[0] : 0.0;
    }
};

struct EpiDirNpcg {
    static constexpr int K = 2;
    double* p;
    double* ap;
    const double* r;
    NpcgState* st;
    RedSlot<2> red;
    double s0, s1;
    __device__ void pre(int i) const { pf(r + i); }
    __device__ bool gate() const { return st->active != 0; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S& src) {
        const double pi = src(i);
        if (p) p[i] = pi;  // nullptr: p was materialised before the SpMV
        ap[i] = acc;
        s0 += pi * acc;
        s1 += pi * r[i];
    }
    __device__ void vals(double (&v)[2]) const { v[0] = s0; v[1] = s1; }
    __device__ void clear() { s0 = 0.0; s1 = 0.0; }
    __device__ void fin(const double (&t)[2]) {
        // U/solvers.py:230-237: breakdown if p'Ap <= 0
        st->pap = t[0];
        st->pr = t[1];
        if (!(t[0] > 0.0)) {
            st->status = 1;
            st->active = 0;
            st->alpha = 0.0;
            npcg_mirror(st);
        } else {
            st->alpha = t[1] / t[0];
        }
    }
};

// restriction: unit values, plain store (gated)
struct EpiStoreG : NoReduce {
    double* y;
    const int* g;
    __device__ void pre(int) const {}
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S&) { y[i] = acc; }
};

// restriction + the start of the coarse flexible CG (BodyFcgBegin fused):
// ||r_c||, gate[0] (U/solvers.py:165, :169)
struct EpiRestrictBegin {
    static constexpr int K = 1;
    double* y;
    const int* g;
    FcgState* st;
    RedSlot<1> red;
    double s0;
    __device__ void pre(int) const {}
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {
        st->gate[0] = 0;
        st->upd[0] = 0;
    }
    template <class S>
    __device__ void row(int i, double acc, const S&) {
        y[i] = acc;
        s0 += acc * acc;
    }
    __device__ void vals(double (&v)[1]) const { v[0] = s0; }
    __device__ void clear() { s0 = 0.0; }
    __device__ void fin(const double (&t)[1]) {
        const double nb = sqrt(t[0]);
        st->bnorm = nb;
        st->rnorm = nb;
        st->gate[0] = (nb <= 1e-14 * nb) ? 0 : 1;
        st->upd[0] = 0;
        st->err = 0;
    }
};


struct BodyBase {
    __device__ bool gate() const { return true; }
    __device__ void off() {}
    __device__ void init() {}
};

// prolongation on a rank's own rows (pointers shifted to the range): the
// coarse correction e_c[v2a_i] is read from the rank that owns aggregate
// v2a_i (K/numba_backend.py:288-294)
struct BodyProlPeer {
    static constexpr int K = 0;
    int mode;  // 0: xpre = 0, 2: vector
    const double* xpre;
    const int* v2a;
    Part pt;
    const double* ec[kMaxRanks];
    const int* ec_valid;
    double* out;
    const int* g;
    bool valid;
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {}
    __device__ void init() { valid = (ec_valid == nullptr) || (*ec_valid != 0); }
    __device__ void item(int i, double*) {
        const double xp = mode == 0 ? 0.0 : xpre[i];
        double e = 0.0;
        if (valid) {
            const int c = v2a[i];
            e = ldv(ec[pt.owner(c)] + c);
        }
        out[i] = __dadd_rn(xp, e);
    }
};

// p = z + beta p_prev materialised ahead of the direction SpMV (large levels)
struct BodyDirP {
    static constexpr int K = 0;
    SrcDir src;
    double* p;
    const int* g;
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {}
    __device__ void init() { src.init(); }
    __device__ void item(int i, double*) { p[i] = src(i); }
};

// ---- x = 0.0 + invm * b  (first sweep from a zero guess)
struct BodyXpre1 : BodyBase {
    static constexpr int K = 0;
    const double* invm;
    const double* b;
    double* x;
    const int* g;
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void item(int i, double*) { x[i] = __dadd_rn(0.0, __dmul_rn(invm[i], b[i])); }
};

// ---- prolongate_add (K/numba_backend.py:288-294), xpre implicit or array
struct BodyProl : BodyBase {
    static constexpr int K = 0;
    SrcUp src;
    double* out;
    const int* g;
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void init() { src.init(); }
    __device__ void item(int i, double*) { out[i] = src(i); }
};

// ---- FCG begin: ||b||, gate[0]  (U/solvers.py:165,169)
struct BodyFcgBegin : BodyBase {
    static constexpr int K = 1;
    const double* b;
    const int* pg;
    FcgState* st;
    RedSlot<1> red;
    __device__ bool gate() const { return pg == nullptr || *pg; }
    __device__ void off() {
        st->gate[0] = 0;
        st->upd[0] = 0;
    }
    __device__ void item(int i, double* v) { v[0] += b[i] * b[i]; }
    __device__ void fin(const double (&t)[1]) {
        const double nb = sqrt(t[0]);
        st->bnorm = nb;
        st->rnorm = nb;
        st->gate[0] = (nb <= 1e-14 * nb) ? 0 : 1;
        st->upd[0] = 0;
        st->err = 0;
    }
};

// ---- beta = -(z.apprev)/(pprev.apprev)  (U/solvers.py:175, :228)
struct BodyBeta : BodyBase {
    static constexpr int K = 2;
    const double* z;
    const double* pp;
    const double* ap;
    double* beta;
    const int* g;
    const int* g2;
    RedSlot<2> red;
    __device__ bool gate() const { return (g == nullptr || *g) && (g2 == nullptr || *g2); }
    __device__ void item(int i, double* v) {
        const double a = ap[i];
        v[0] += z[i] * a;
        v[1] += pp[i] * a;
    }
    __device__ void fin(const double (&t)[2]) { *beta = -t[0] / t[1]; }
};

// ---- FCG update: x = x + alpha p, r = r - alpha ap, gate[s+1]  (U/solvers.py:181-185,169)
// the last inner step (step == steps - 1): only x leaves the FCG -- the
// residual and its norm / gate have no reader, so they are skipped
struct BodyFcgUpdLast : BodyBase {
    static constexpr int K = 0;
    int step;
    double* x;
    const double* p;
    FcgState* st;
    double alpha;
    __device__ bool gate() const { return st->upd[step] != 0; }
    __device__ void off() {}
    __device__ void init() { alpha = st->alpha; }
    __device__ void item(int i, double*) {
        const double xo = step == 0 ? 0.0 : x[i];
        x[i] = __dadd_rn(xo, __dmul_rn(alpha, p[i]));
    }
    __device__ void fin(const double (&)[1]) {}
};

struct BodyFcgUpd : BodyBase {
    static constexpr int K = 1;
    int step;
    int last = 0;  // k_dir_update: x only (BodyFcgUpdLast's work)
    ParentUp pu;   // (last step only)
    double* x;
    const double* p;
    const double* rin;
    double* rout;
    const double* ap;
    FcgState* st;
    int singular;
    RedSlot<1> red;
    double alpha;
    __device__ bool gate() const { return st->upd[step] != 0; }
    __device__ void off() { st->gate[step + 1] = 0; }
    __device__ void init() { alpha = st->alpha; }
    __device__ void item(int i, double* v) {
        const double xo = step == 0 ? 0.0 : x[i];
        x[i] = __dadd_rn(xo, __dmul_rn(alpha, p[i]));
        const double rn = __dsub_rn(rin[i], __dmul_rn(alpha, ap[i]));
        rout[i] = rn;
        v[0] += singular ? rn : rn * rn;
    }
    __device__ void fin(const double (&t)[1]) {
        if (singular) {
            st->sum = t[0];  // projection + norm follow in separate kernels
        } else {
            const double rn = sqrt(t[0]);
            st->rnorm = rn;
            st->gate[step + 1] = (rn <= 1e-14 * st->bnorm) ? 0 : 1;
        }
    }
};

// singular FCG: r -= mean(r); gate from the projected norm
struct BodyFcgProj : BodyBase {
    static constexpr int K = 1;
    int n, step;
    double* r;
    FcgState* st;
    RedSlot<1> red;
    double mean;
    __device__ bool gate() const { return st->upd[step] != 0; }
    __device__ void off() { st->gate[step + 1] = 0; }
    __device__ void init() { mean = st->sum / (double)n; }
    __device__ void item(int i, double* v) {
        const double rv = __dsub_rn(r[i], mean);
        r[i] = rv;
        v[0] += rv * rv;
    }
    __device__ void fin(const double (&t)[1]) {
        const double rn = sqrt(t[0]);
        st->rnorm = rn;
        st->gate[step + 1] = (rn <= 1e-14 * st->bnorm) ? 0 : 1;
    }
};

// ---- NPCG update (U/solvers.py:237-254)
struct BodyNpcgUpd : BodyBase {
    static constexpr int K = 1;
    double* x;
    const double* p;
    double* r;
    const double* ap;
    NpcgState* st;
    double* hist;
    int singular;
    RedSlot<1> red;
    double alpha;
    __device__ bool gate() const { return st->active != 0; }
    __device__ void init() { alpha = st->alpha; }
    __device__ void item(int i, double* v) {
        x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
        const double rn = __dsub_rn(r[i], __dmul_rn(alpha, ap[i]));
        r[i] = rn;
        v[0] += singular ? rn : rn * rn;
    }
    __device__ void fin(const double (&t)[1]) {
        if (singular) { st->sum = t[0]; return; }
        const double rel = sqrt(t[0]) / st->bnorm;
        const double prev = st->last_rel;
        st->iters += 1;
        hist[st->iters] = rel;
        st->last_rel = rel;
        if (rel > prev) st->up += 1; else st->up = 0;
        if (st->up >= 2) { st->have_prev = 0; st->up = 0; }
        else st->have_prev = 1;
        if (!(rel > st->tol) || st->iters >= st->max_iters) st->active = 0;
        npcg_mirror(st);
    }
};

// singular NPCG: project r and x, then the norm/bookkeeping
struct BodyNpcgProjX : BodyBase {
    static constexpr int K = 1;
    double* x;
    NpcgState* st;
    RedSlot<1> red;
    __device__ bool gate() const { return st->active != 0; }
    __device__ void item(int i, double* v) { v[0] += x[i]; }
    __device__ void fin(const double (&t)[1]) { st->beta = t[0]; /* x sum parked in beta slot (unused now) */ }
};

struct BodyNpcgProj : BodyBase {
    static constexpr int K = 1;
    int n;
    double* x;
    double* r;
    NpcgState* st;
    double* hist;
    RedSlot<1> red;
    double mr, mx;
    __device__ bool gate() const { return st->active != 0; }
    __device__ void init() {
        mr = st->sum / (double)n;
        mx = st->beta / (double)n;
    }
    __device__ void item(int i, double* v) {
        const double rv = __dsub_rn(r[i], mr);
        r[i] = rv;
        x[i] = __dsub_rn(x[i], mx);
        v[0] += rv * rv;
    }
    __device__ void fin(const double (&t)[1]) {
        const double rel = sqrt(t[0]) / st->bnorm;
        const double prev = st->last_rel;
        st->iters += 1;
        hist[st->iters] = rel;
        st->last_rel = rel;
        if (rel > prev) st->up += 1; else st->up = 0;
        if (st->up >= 2) { st->have_prev = 0; st->up = 0; }
        else st->have_prev = 1;
        if (!(rel > st->tol) || st->iters >= st->max_iters) st->active = 0;
        npcg_mirror(st);
    }
};

// ---- mean projection v -= mean(v)  (U/solvers.py:112-113)
struct BodySum : BodyBase {
    static constexpr int K = 1;
    const double* v;
    double* slot;
    const int* g;
    RedSlot<1> red;
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void item(int i, double* a) { a[0] += v[i]; }
    __device__ void fin(const double (&t)[1]) { *slot = t[0]; }
};

struct BodySub : BodyBase {
    static constexpr int K = 0;
    int n;
    const double* in;
    double* out;
    const double* slot;
    const int* g;
    double m;
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void init() { m = *slot / (double)n; }
    __device__ void item(int i, double*) { out[i] = __dsub_rn(in[i], m); }
};

// ---- _check_compatible (U/solvers.py:116-125): drift check + projection
struct BodyCompat : BodyBase {
    static constexpr int K = 2;
    const double* b;
    double* slot;   // [0] sum, [1] norm
    int* err;
    int n;
    const int* g;
    RedSlot<2> red;
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void item(int i, double* a) {
        a[0] += b[i];
        a[1] += b[i] * b[i];
    }
    __device__ void fin(const double (&t)[2]) {
        const double nrm = sqrt(t[1]);
        slot[0] = t[0];
        slot[1] = nrm;
        if (nrm == 0.0) { slot[0] = 0.0; return; }  // returned unprojected (mean of zeros is 0)
        const double drift = fabs(t[0]) / (sqrt((double)n) * nrm);
        if (drift > 1e-10) *err = 1;
    }
};

// ---- plain norm / NPCG init
struct BodyNorm : BodyBase {
    static constexpr int K = 1;
    const double* v;
    double* out;
    RedSlot<1> red;
    __device__ void item(int i, double* a) { a[0] += v[i] * v[i]; }
    __device__ void fin(const double (&t)[1]) { *out = sqrt(t[0]); }
};

struct BodyNpcgInit : BodyBase {
    static constexpr int K = 2;
    const double* b;
    const double* r;
    NpcgState* st;
    double* hist;
    RedSlot<2> red;
    __device__ void item(int i, double* a) {
        a[0] += b[i] * b[i];
        a[1] += r[i] * r[i];
    }
    __device__ void fin(const double (&t)[2]) {
        // U/solvers.py:205,216,221
        const double bn = sqrt(t[0]);
        st->bnorm = bn;
        st->iters = 0;
        st->up = 0;
        st->have_prev = 0;
        st->status = 0;
        if (bn == 0.0) {
            hist[0] = 0.0;
            st->last_rel = 0.0;
            st->active = 0;
            npcg_mirror(st);
            return;
        }
        const double rel = sqrt(t[1]) / bn;
        hist[0] = rel;
        st->last_rel = rel;
        st->active = (rel > st->tol && st->max_iters > 0) ? 1 : 0;
        npcg_mirror(st);
    }
};

struct BodyCopy : BodyBase {
    static constexpr int K = 0;
    const double* a;
    double* o;
    __device__ void item(int i, double*) { o[i] = a[i]; }
};

struct BodyBmAx : BodyBase {
    static constexpr int K = 0;
    const double* b;
    const double* ax;
    double* r;
    __device__ void item(int i, double*) { r[i] = __dsub_rn(b[i], ax[i]); }
};

}  // namespace uaamg
