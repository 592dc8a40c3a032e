// kernels_solve.cu -- solve-phase kernels: staged SpMV family, smoother
// diagonals, transfers, flexible-CG vector updates with fused deterministic
// reductions, dense coarsest solve.
//
// Reference semantics: U/solvers.py (smoother_inverse_diag :69-81, smooth
// :84-91, transfers :94-109, projections :112-125, cycle :128-157,
// _inner_fcg :160-187, npcg_solve :190-255) and K/numba_backend.py kernels.
#include "csr_stream.cuh"
#include "kernels.h"

namespace uaamg {

std::atomic<uint64_t> g_launches{0};

// ============================================================ epilogues
struct EpiStore : NoReduce {
    double* y;
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
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S&) { r[i] = __dsub_rn(b[i], acc); }
};

// one sweep: out_i = x_i + invm_i * (b_i - (A x)_i)   (K/numba_backend.py:303-309)
struct EpiSweep : NoReduce {
    const double* invm;
    const double* b;
    double* out;
    const int* g;
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S& src) {
        const double r = __dsub_rn(b[i], acc);
        out[i] = __dadd_rn(src(i), __dmul_rn(invm[i], r));
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
    __device__ bool gate() const { return st->gate[step] != 0; }
    __device__ void off() { st->upd[step] = 0; }
    template <class S>
    __device__ void row(int i, double acc, const S& src) {
        const double pi = src(i);
        p[i] = pi;
        ap[i] = acc;
        s0 += pi * acc;
        s1 += pi * r[i];
    }
    __device__ void vals(double (&v)[2]) const { v[0] = s0; v[1] = s1; }
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
    __device__ bool gate() const { return st->active != 0; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S& src) {
        const double pi = src(i);
        p[i] = pi;
        ap[i] = acc;
        s0 += pi * acc;
        s1 += pi * r[i];
    }
    __device__ void vals(double (&v)[2]) const { v[0] = s0; v[1] = s1; }
    __device__ void fin(const double (&t)[2]) {
        // U/solvers.py:230-237: breakdown if p'Ap <= 0
        st->pap = t[0];
        st->pr = t[1];
        if (!(t[0] > 0.0)) {
            st->status = 1;
            st->active = 0;
            st->alpha = 0.0;
        } else {
            st->alpha = t[1] / t[0];
        }
    }
};

// restriction: unit values, plain store (gated)
struct EpiStoreG : NoReduce {
    double* y;
    const int* g;
    __device__ bool gate() const { return g == nullptr || *g; }
    __device__ void off() {}
    template <class S>
    __device__ void row(int i, double acc, const S&) { y[i] = acc; }
};

template <class Src, class Epi, bool Unit, bool Exact = false>
static void run_stream(const Csr& A, const Blocks& B, const Src& src, const Epi& epi, cudaStream_t s) {
    if (B.nb == 0) return;
    UA_LAUNCH((k_csr_stream<Src, Epi, Unit, Exact>), B.nb, kThreads, 0, s, A, B, src, epi);
}

void launch_spmv(const Csr& A, const Blocks& B, const double* x, double* y, cudaStream_t s) {
    EpiStore e{};
    e.y = y;
    run_stream<SrcVec, EpiStore, false, true>(A, B, SrcVec{x}, e, s);
}

void launch_sweep_exact(const Csr& A, const Blocks& B, const double* invm, const double* b, const double* x,
                        double* out, cudaStream_t s) {
    EpiSweep e{};
    e.invm = invm; e.b = b; e.out = out; e.g = nullptr;
    run_stream<SrcVec, EpiSweep, false, true>(A, B, SrcVec{x}, e, s);
}

void launch_restrict_exact(int nc, const int* agg_ptr, const int* members, const Blocks& MB, const double* r,
                           double* rc, cudaStream_t s) {
    Csr P;
    P.n = nc; P.rp = agg_ptr; P.ci = members; P.av = nullptr;
    EpiStoreG e{};
    e.y = rc; e.g = nullptr;
    run_stream<SrcVec, EpiStoreG, true, true>(P, MB, SrcVec{r}, e, s);
}

void launch_residual(const Csr& A, const Blocks& B, int xmode, const double* invm, const double* b,
                     const double* x, double* r, const int* gate, cudaStream_t s) {
    EpiResid e{};
    e.b = b; e.r = r; e.g = gate;
    if (xmode == 1) run_stream<SrcPre1, EpiResid, false>(A, B, SrcPre1{invm, b}, e, s);
    else run_stream<SrcVec, EpiResid, false>(A, B, SrcVec{x}, e, s);
}

void launch_sweep_vec(const Csr& A, const Blocks& B, const double* invm, const double* b, const double* x,
                      double* out, const int* gate, cudaStream_t s) {
    EpiSweep e{};
    e.invm = invm; e.b = b; e.out = out; e.g = gate;
    run_stream<SrcVec, EpiSweep, false>(A, B, SrcVec{x}, e, s);
}

void launch_sweep_up(const Csr& A, const Blocks& B, int xmode, const double* invm, const double* b,
                     const double* xpre, const int* v2a, const double* ec, const int* ec_valid, double* out,
                     const int* gate, cudaStream_t s) {
    EpiSweep e{};
    e.invm = invm; e.b = b; e.out = out; e.g = gate;
    SrcUp src{};
    src.mode = xmode; src.invm = invm; src.b = b; src.xpre = xpre; src.v2a = v2a; src.ec = ec;
    src.ec_valid = ec_valid;
    run_stream<SrcUp, EpiSweep, false>(A, B, src, e, s);
}

void launch_restrict(int nc, const int* agg_ptr, const int* members, const Blocks& MB, const double* r,
                     double* rc, const int* gate, cudaStream_t s) {
    Csr P;
    P.n = nc; P.rp = agg_ptr; P.ci = members; P.av = nullptr;
    EpiStoreG e{};
    e.y = rc; e.g = gate;
    run_stream<SrcVec, EpiStoreG, true>(P, MB, SrcVec{r}, e, s);
}

void launch_dir_fcg(const Csr& A, const Blocks& B, const double* z, const double* pprev, int have_prev,
                    const double* r, double* p, double* ap, FcgState* st, int step, RedScratch rs,
                    cudaStream_t s) {
    EpiDirFcg e{};
    e.p = p; e.ap = ap; e.r = r; e.st = st; e.step = step; e.red = {rs.partials, rs.ticket};
    SrcDir src{};
    src.z = z; src.pprev = pprev; src.beta_p = &st->beta; src.have_p = nullptr; src.have_static = have_prev;
    run_stream<SrcDir, EpiDirFcg, false>(A, B, src, e, s);
}

void launch_dir_npcg(const Csr& A, const Blocks& B, const double* z, const double* pprev, const double* r,
                     double* p, double* ap, NpcgState* st, RedScratch rs, cudaStream_t s) {
    EpiDirNpcg e{};
    e.p = p; e.ap = ap; e.r = r; e.st = st; e.red = {rs.partials, rs.ticket};
    SrcDir src{};
    src.z = z; src.pprev = pprev; src.beta_p = &st->beta; src.have_p = &st->have_prev;
    run_stream<SrcDir, EpiDirNpcg, false>(A, B, src, e, s);
}

// ============================================================ map-reduce
template <class Body>
__global__ void __launch_bounds__(kThreads) k_map(int n, Body body_p) {
    Body body = body_p;
    if (!body.gate()) {
        if (blockIdx.x == 0 && threadIdx.x == 0) body.off();
        return;
    }
    body.init();
    double v[Body::K > 0 ? Body::K : 1] = {};
    for (int i = blockIdx.x * kThreads + threadIdx.x; i < n; i += gridDim.x * kThreads) body.item(i, v);
    if constexpr (Body::K > 0) {
        grid_reduce_finish<Body::K>(v, body.red.partials, body.red.ticket,
                                    [&](const double (&t)[Body::K]) { body.fin(t); });
    }
}

static int map_grid(int n) {
    int g = cdiv(n, kThreads * 4);
    return g < 1 ? 1 : (g > 2 * kNumSMs ? 2 * kNumSMs : g);
}

template <class Body>
static void run_map(int n, const Body& body, cudaStream_t s) {
    UA_LAUNCH((k_map<Body>), map_grid(n), kThreads, 0, s, n, body);
}

struct BodyBase {
    __device__ bool gate() const { return true; }
    __device__ void off() {}
    __device__ void init() {}
};

// ---- smoother diagonal (U/solvers.py:69-81, K/numba_backend.py:59-84)
__global__ void k_inv_diag(Csr A, int l1, double omega, double* invm, int* bad_row) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
        double acc = 0.0, dii = 0.0;
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            const int c = A.ci[k];
            if (l1) {
                if (c == i) dii = A.av[k];
                else acc = __dadd_rn(acc, fabs(A.av[k]));
            } else if (c == i) {
                dii = A.av[k];
                break;
            }
        }
        const double m = l1 ? __dadd_rn(acc, dii) : dii;
        if (m <= 0.0) atomicMin(bad_row, i);
        invm[i] = (l1 ? 1.0 : omega) / m;
    }
}

void launch_inv_diag(const Csr& A, int l1, double omega, double* invm, int* bad_row, cudaStream_t s) {
    UA_LAUNCH(k_inv_diag, map_grid(A.n) * 2, kThreads, 0, s, A, l1, omega, invm, bad_row);
}

__global__ void k_diag(Csr A, int l1, double* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
        double acc = 0.0, dii = 0.0;
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            const int c = A.ci[k];
            if (l1) {
                if (c == i) dii = A.av[k];
                else acc = __dadd_rn(acc, fabs(A.av[k]));
            } else if (c == i) {
                dii = A.av[k];
                break;
            }
        }
        out[i] = l1 ? __dadd_rn(acc, dii) : dii;
    }
}

void launch_diag(const Csr& A, int l1, double* out, cudaStream_t s) {
    UA_LAUNCH(k_diag, map_grid(A.n) * 2, kThreads, 0, s, A, l1, out);
}

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
void launch_xpre1(int n, const double* invm, const double* b, double* x, const int* gate, cudaStream_t s) {
    BodyXpre1 body{};
    body.invm = invm; body.b = b; body.x = x; body.g = gate;
    run_map(n, body, s);
}

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
void launch_prolongate(int n, int xmode, const double* invm, const double* b, const double* xpre, const int* v2a,
                       const double* ec, const int* ec_valid, double* out, const int* gate, cudaStream_t s) {
    BodyProl body{};
    body.src.mode = xmode; body.src.invm = invm; body.src.b = b; body.src.xpre = xpre; body.src.v2a = v2a;
    body.src.ec = ec; body.src.ec_valid = ec_valid; body.out = out; body.g = gate;
    run_map(n, body, s);
}

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
void launch_fcg_begin(int n, const double* b, const int* parent_gate, FcgState* st, RedScratch rs, cudaStream_t s) {
    BodyFcgBegin body{};
    body.b = b; body.pg = parent_gate; body.st = st; body.red = {rs.partials, rs.ticket};
    run_map(n, body, s);
}

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
void launch_beta(int n, const double* z, const double* pprev, const double* apprev, double* beta, const int* gate,
                 const int* gate2, RedScratch rs, cudaStream_t s) {
    BodyBeta body{};
    body.z = z; body.pp = pprev; body.ap = apprev; body.beta = beta; body.g = gate; body.g2 = gate2;
    body.red = {rs.partials, rs.ticket};
    run_map(n, body, s);
}

// ---- FCG update: x = x + alpha p, r = r - alpha ap, gate[s+1]  (U/solvers.py:181-185,169)
struct BodyFcgUpd : BodyBase {
    static constexpr int K = 1;
    int step;
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

void launch_fcg_update(int n, int step, double* x, const double* p, const double* r_in, double* r_out,
                       const double* ap, FcgState* st, int singular, RedScratch rs, cudaStream_t s) {
    BodyFcgUpd body{};
    body.step = step; body.x = x; body.p = p; body.rin = r_in; body.rout = r_out; body.ap = ap; body.st = st;
    body.singular = singular; body.red = {rs.partials, rs.ticket};
    run_map(n, body, s);
    if (singular) {
        BodyFcgProj pj{};
        pj.n = n; pj.step = step; pj.r = r_out; pj.st = st; pj.red = {rs.partials, rs.ticket};
        run_map(n, pj, s);
    }
}

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
    }
};

void launch_npcg_update(int n, double* x, const double* p, double* r, const double* ap, NpcgState* st,
                        double* history, int singular, RedScratch rs, cudaStream_t s) {
    BodyNpcgUpd body{};
    body.x = x; body.p = p; body.r = r; body.ap = ap; body.st = st; body.hist = history; body.singular = singular;
    body.red = {rs.partials, rs.ticket};
    run_map(n, body, s);
    if (singular) {
        BodyNpcgProjX bx{};
        bx.x = x; bx.st = st; bx.red = {rs.partials, rs.ticket};
        run_map(n, bx, s);
        BodyNpcgProj pj{};
        pj.n = n; pj.x = x; pj.r = r; pj.st = st; pj.hist = history; pj.red = {rs.partials, rs.ticket};
        run_map(n, pj, s);
    }
}

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
void launch_project_mean(int n, double* v, double* sum_slot, const int* gate, RedScratch rs, cudaStream_t s) {
    BodySum bs{};
    bs.v = v; bs.slot = sum_slot; bs.g = gate; bs.red = {rs.partials, rs.ticket};
    run_map(n, bs, s);
    BodySub sb{};
    sb.n = n; sb.in = v; sb.out = v; sb.slot = sum_slot; sb.g = gate;
    run_map(n, sb, s);
}

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
void launch_check_compatible(int n, const double* b, double* out, int* err_flag, double* sum_slot,
                             const int* gate, int level, RedScratch rs, cudaStream_t s) {
    (void)level;
    BodyCompat bc{};
    bc.b = b; bc.slot = sum_slot; bc.err = err_flag; bc.n = n; bc.g = gate; bc.red = {rs.partials, rs.ticket};
    run_map(n, bc, s);
    BodySub sb{};
    sb.n = n; sb.in = b; sb.out = out; sb.slot = sum_slot; sb.g = gate;
    run_map(n, sb, s);
}

// ---- dense coarsest solve x = Minv b (warp per row)
__global__ void k_dense_solve(int n, const double* __restrict__ M, const double* __restrict__ b, double* x,
                              const int* gate) {
    if (gate && !*gate) return;
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= n) return;
    double acc = 0.0;
    for (int j = lane; j < n; j += 32) acc += M[(size_t)row * n + j] * b[j];
    acc = warp_sum(acc);
    if (lane == 0) x[row] = acc;
}
void launch_dense_solve(int n, const double* Minv, const double* b, double* x, const int* gate, cudaStream_t s) {
    if (n == 0) return;
    UA_LAUNCH(k_dense_solve, cdiv(n, 8), 256, 0, s, n, Minv, b, x, gate);
}

// ---- plain norm / NPCG init
struct BodyNorm : BodyBase {
    static constexpr int K = 1;
    const double* v;
    double* out;
    RedSlot<1> red;
    __device__ void item(int i, double* a) { a[0] += v[i] * v[i]; }
    __device__ void fin(const double (&t)[1]) { *out = sqrt(t[0]); }
};
void launch_norm(int n, const double* v, double* out, RedScratch rs, cudaStream_t s) {
    BodyNorm b{};
    b.v = v; b.out = out; b.red = {rs.partials, rs.ticket};
    run_map(n, b, s);
}

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
            return;
        }
        const double rel = sqrt(t[1]) / bn;
        hist[0] = rel;
        st->last_rel = rel;
        st->active = (rel > st->tol && st->max_iters > 0) ? 1 : 0;
    }
};
void launch_npcg_init(int n, const double* b, const double* r, NpcgState* st, double* history, RedScratch rs,
                      cudaStream_t s) {
    BodyNpcgInit body{};
    body.b = b; body.r = r; body.st = st; body.hist = history; body.red = {rs.partials, rs.ticket};
    run_map(n, body, s);
}

struct BodyCopy : BodyBase {
    static constexpr int K = 0;
    const double* a;
    double* o;
    __device__ void item(int i, double*) { o[i] = a[i]; }
};
void launch_copy(int n, const double* src, double* dst, cudaStream_t s) {
    BodyCopy b{};
    b.a = src; b.o = dst;
    run_map(n, b, s);
}
struct BodyBmAx : BodyBase {
    static constexpr int K = 0;
    const double* b;
    const double* ax;
    double* r;
    __device__ void item(int i, double*) { r[i] = __dsub_rn(b[i], ax[i]); }
};
void launch_axpby_init(int n, const double* b, const double* ax, double* r, cudaStream_t s) {
    BodyBmAx body{};
    body.b = b; body.ax = ax; body.r = r;
    run_map(n, body, s);
}

}  // namespace uaamg
