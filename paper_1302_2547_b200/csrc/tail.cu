// tail.cu -- the coarse tail of the K-cycle in one thread-block cluster.
//
// The level just above the coarsest is the most-visited level of the
// K-cycle (2^l visits per outer iteration) and the smallest one that still
// needs a smoother: every visit is a chain of ~15 dependent operations of a
// few thousand rows each, so as separate kernels it is bound by launch
// latency and L2 round trips, not by bytes.  Here the whole inner solve at
// that level -- restriction from the level above, the flexible CG
// (U/solvers.py:160-187) or the plain cycle (:128-157), the coarsest solve,
// prolongation and smoothing -- runs in ONE launch of a cluster of up to 16
// CTAs:
//   * rows are split into contiguous blocks, one per CTA; the CTA's matrix
//     rows, restriction members, smoother diagonal and (dense coarsest)
//     rows of Minv are staged from global memory into its shared memory
//     before the dependency wait, so they overlap the previous kernel;
//   * every vector of the level lives in distributed shared memory: a CTA
//     writes its own rows, and gathers of column k read the owning CTA's
//     copy through ld.shared::cluster (column indices are pre-packed as
//     owner << 16 | local);
//   * phases are separated by the hardware cluster barrier (release /
//     acquire), reductions are per-CTA block sums written into every CTA's
//     slot array and folded in CTA order, so all CTAs hold the same bits and
//     take the same branch decisions.
// Row sums follow the solve's group kernel exactly (csr_group.cuh): rows of
// up to 256 entries in reference order, longer rows as 256-entry pieces
// with a warp tree each, folded with a warp tree.  Only the dot products /
// norms use a different (fixed) tree than the separate-kernel path.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>

#include "csr_tma.cuh"
#include "tail.h"

namespace uaamg {

namespace {

constexpr int kTailVecs = 9;
enum { VB = 0, VX, VRF, VZ, VP0, VP1, VAP0, VAP1, VR };
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned cta_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// element `packed` (owner << 16 | local) of a vector whose local copy is v:
// a generic pointer into the owning CTA's shared memory (plain loads, so the
// compiler batches independent gathers)
#ifdef UA_TAIL_LOCAL_ONLY  // diagnostics: gathers read the local copy (wrong values, DSMEM-free timing)
template <class T>
__device__ __forceinline__ const T* dsm(const T* v, int packed) {
    return v + (packed & 0xffff);
}
#else
template <class T>
__device__ __forceinline__ const T* dsm(const T* v, int packed) {
    return static_cast<const T*>(__cluster_map_shared_rank(v + (packed & 0xffff), (unsigned)packed >> 16));
}
#endif

// ------------------------------------------------------------------ gathers
// Columns of the tail matrix are packed owner << 16 | local, or kHub << 16 |
// slot for a hub column (read from the CTA's local hub copy).  Gathers take
// a `live` predicate: padding slots issue no memory request (predicated
// shared::cluster loads, no branches, so a round's loads are all in flight).
constexpr unsigned kHub = 0xffffu;
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double ldc(uint32_t caddr, bool live) {
    double v = 0.0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared::cluster.f64 %0, [%1];\n\t}"
                 : "+d"(v)
                 : "r"(caddr), "r"((unsigned)live));
    return v;
}
__device__ __forceinline__ int ldc_i(uint32_t caddr, bool live) {
    int v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared::cluster.s32 %0, [%1];\n\t}"
                 : "+r"(v)
                 : "r"(caddr), "r"((unsigned)live));
    return v;
}
__device__ __forceinline__ uint32_t cmap(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
struct VRef {  // a distributed vector: local rows + local hub-column copy
    const double* v;   // local rows (generic)
    uint32_t vs, hs;   // shared addresses of the rows and of the hub copy
    uint32_t me;       // this CTA's rank
    __device__ VRef(const double* rows, const double* hub, uint32_t rank)
        : v(rows), vs(saddr(rows)), hs(saddr(hub)), me(rank) {}
    __device__ double ld(int c, bool live) const {
        const unsigned o = (unsigned)c >> 16, j = (unsigned)c & 0xffffu;
        const bool hub = o == kHub;
        return ldc(cmap((hub ? hs : vs) + 8 * j, hub ? me : o), live);
    }
};
struct GVec {  // x_k (plain packed index, no hubs)
    uint32_t x;
    __device__ double operator()(int c, bool live) const {
        return ldc(cmap(x + 8 * ((unsigned)c & 0xffffu), (unsigned)c >> 16), live);
    }
};
struct GGlobal {  // r_k of the level above (global memory, plain index; padding reads r[0])
    const double* r;
    __device__ double operator()(int c, bool) const { return r[c]; }
};
struct GPre1 {  // one sweep from zero: 0.0 + invm_k * b_k (SrcPre1)
    VRef invm, b;
    __device__ double operator()(int c, bool live) const {
        return __dadd_rn(0.0, __dmul_rn(invm.ld(c, live), b.ld(c, live)));
    }
};
struct GUp {  // xpre_k + ec[v2a_k] (SrcUp, xpre implicit or zero)
    VRef invm, b;
    const int* v2a;
    uint32_t v2as, hv2as;
    const double* ec;  // replicated coarse correction (dense)
    int pre, dense;
    double ec1;
    __device__ double operator()(int c, bool live) const {
        const double xp = pre ? __dadd_rn(0.0, __dmul_rn(invm.ld(c, live), b.ld(c, live))) : 0.0;
        double e = ec1;
        if (dense) {
            const unsigned o = (unsigned)c >> 16, j = (unsigned)c & 0xffffu;
            const bool hub = o == kHub;
            e = ec[ldc_i(cmap((hub ? hv2as : v2as) + 4 * j, hub ? invm.me : o), live)];
        }
        return __dadd_rn(xp, e);
    }
    __device__ double at(int i) const {
        const double xp = pre ? __dadd_rn(0.0, __dmul_rn(invm.v[i], b.v[i])) : 0.0;
        return __dadd_rn(xp, dense ? ec[v2a[i]] : ec1);
    }
};
struct GDir {  // z_k + beta pprev_k (SrcDir)
    VRef z, pp;
    int have;
    double beta;
    __device__ double operator()(int c, bool live) const {
        const double zk = z.ld(c, live);
        return have ? __dadd_rn(zk, __dmul_rn(beta, pp.ld(c, live && have))) : zk;
    }
    __device__ double at(int i) const { return have ? __dadd_rn(z.v[i], __dmul_rn(beta, pp.v[i])) : z.v[i]; }
};

// ------------------------------------------------------------------ epilogues
struct EStore {
    double* y;
    __device__ void row(int i, double acc) { y[i] = acc; }
};
struct EStoreNorm {  // restriction + ||.||^2 (EpiRestrictBegin)
    double* y;
    double s;
    __device__ void row(int i, double acc) {
        y[i] = acc;
        s += acc * acc;
    }
};
struct EResid {  // r = b - A x, optional store, running sum (EpiResid / EpiResidSum)
    const double* rin;
    double* r;
    double s;
    __device__ void row(int i, double acc) {
        const double v = __dsub_rn(rin[i], acc);
        if (r) r[i] = v;
        s += v;
    }
};
struct ESweep {  // z = x + invm (b - A x), x = prolongated iterate; beta dot (EpiSweepBeta)
    const double* invm;
    const double* rin;
    double* z;
    const double* app;
    GUp x;
    double s;
    __device__ void row(int i, double acc) {
        const double r = __dsub_rn(rin[i], acc);
        const double o = __dadd_rn(x.at(i), __dmul_rn(invm[i], r));
        z[i] = o;
        if (app) s += o * app[i];
    }
};
struct EDir {  // p, Ap, p.Ap, p.r (EpiDirFcg)
    const double* rin;
    double* p;
    double* ap;
    GDir g;
    double s0, s1;
    __device__ void row(int i, double acc) {
        const double pi = g.at(i);
        p[i] = pi;
        ap[i] = acc;
        s0 += pi * acc;
        s1 += pi * rin[i];
    }
};

struct RowSet {
    const int* rp;
    const int* idx;
    const double* val;
    const int4* pc;
    const int* lptr;
    const int* lrow;
    int R, np, nl;
};

__device__ __forceinline__ RowSet rowset(unsigned char* sm, const TailRows& t, int R, int np, int nl) {
    RowSet s;
    s.rp = reinterpret_cast<const int*>(sm + t.rp);
    s.idx = reinterpret_cast<const int*>(sm + t.idx);
    s.val = t.val >= 0 ? reinterpret_cast<const double*>(sm + t.val) : nullptr;
    s.pc = reinterpret_cast<const int4*>(sm + t.pc);
    s.lptr = reinterpret_cast<const int*>(sm + t.lptr);
    s.lrow = reinterpret_cast<const int*>(sm + t.lrow);
    s.R = R;
    s.np = np;
    s.nl = nl;
    return s;
}

// diagnostics marks: clock64 into a shared array (flushed at the end, so the
// marks add no global stores for the cluster barriers' release to drain)
__shared__ long long g_tp[kTailProfMarks];
__device__ __forceinline__ void smark(int k) {
    if (k >= 0) {
        __syncthreads();
        if (threadIdx.x == 0) g_tp[k] = clock64();
    }
}

// one round of a group: entries [base, min(hi, base + 32 NQ)) -> products
// in the warp's window
template <int NQ, bool Unit, class G>
__device__ __forceinline__ void gather_round(const RowSet& S, const G& g, int base, int hi, int lane, int dummy,
                                             double* win) {
    int c[NQ];
    double a[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int k = base + lane + 32 * q;
        c[q] = k < hi ? S.idx[k] : dummy;  // a valid, CTA-local dummy column
        if (!Unit) a[q] = k < hi ? S.val[k] : 0.0;
    }
    double v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = g(c[q], base + lane + 32 * q < hi);
#pragma unroll
    for (int q = 0; q < NQ; ++q) win[lane + 32 * q] = Unit ? v[q] : __dmul_rn(a[q], v[q]);
}

// Row sums of the CTA's rows (grp_unit of csr_group.cuh on shared-memory
// operands): warps stride over 32-row groups -- lane = row, the group's
// entries streamed in rounds through the warp's product window, each lane
// folding its own row in ascending order (the reference order) -- then the
// 256-entry pieces of long rows (warp tree each) and their fold.  All
// threads of the CTA call it.
template <bool Unit, class G, class E>
__device__ void rowsum(const RowSet& S, double* win_all, double* psum, const G& g, E& e, int dummy, int mk = -1) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* win = win_all + w * 256;
    const int ng = (S.R + 31) >> 5;
    for (int u = w; u < ng; u += kTailWarps) {
        const int i = (u << 5) + lane;
        const bool valid = i < S.R;
        const int bi = valid ? S.rp[i] : 0;
        const int ei = valid ? S.rp[i + 1] : 0;
        const int e0 = __shfl_sync(kFull, bi, 0);
        const int e1 = S.rp[min((u << 5) + 32, S.R)];
        const bool mine = valid && (ei - bi) <= kTailLongMin;
        double acc = 0.0;
        // stream the group's entries around its long rows
        unsigned lm = __ballot_sync(kFull, valid && !mine);
        int lo = e0;
        while (true) {
            int hi = e1, L = 0;
            if (lm) {
                L = __ffs(lm) - 1;
                hi = __shfl_sync(kFull, bi, L);
            }
            for (int base = lo; base < hi; base += 256) {
                const int top = min(hi, base + 256);
                if (top - base <= 128) gather_round<4, Unit>(S, g, base, top, lane, dummy, win);
                else gather_round<8, Unit>(S, g, base, top, lane, dummy, win);
                __syncwarp();
                if (mine) {
                    const int l1 = min(ei, top) - base;
                    int k = max(bi, base) - base;
                    for (; k + 4 <= l1; k += 4) {
                        double t[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) t[r] = win[k + r];
#pragma unroll
                        for (int r = 0; r < 4; ++r) acc = __dadd_rn(acc, t[r]);
                    }
                    for (; k < l1; ++k) acc = __dadd_rn(acc, win[k]);
                }
                __syncwarp();
            }
            if (!lm) break;
            lo = __shfl_sync(kFull, ei, L);
            lm &= lm - 1;
        }
        if (mine) e.row(i, acc);
    }
    smark(mk);
    for (int u = w; u < S.np; u += kTailWarps) {
        {
            const int4 pc = S.pc[u];  // {row, eb, ee, slot}
            int c[8];
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int k = pc.y + lane + 32 * q;
                c[q] = k < pc.z ? S.idx[k] : dummy;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = g(c[q], pc.y + lane + 32 * q < pc.z);
            double part = 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int k = pc.y + lane + 32 * q;
                if (k < pc.z) part = __dadd_rn(part, Unit ? v[q] : __dmul_rn(S.val[k], v[q]));
            }
            part = warp_sum(part);
            if (lane == 0) psum[pc.w] = part;
        }
    }
    if (S.np == 0) return;  // CTA-uniform
    __syncthreads();
    for (int q = w; q < S.nl; q += kTailWarps) {
        const int p0 = S.lptr[q], p1 = S.lptr[q + 1];
        double acc = 0.0;
        for (int k = p0 + lane; k < p1; k += 32) acc = __dadd_rn(acc, psum[k]);
        acc = warp_sum(acc);
        if (lane == 0) e.row(S.lrow[q], acc);
    }
    __syncthreads();  // psum reuse by the next row-sum of this CTA
}

#define TP(k) \
    do { \
        if (c.a->prof) { \
            __syncthreads(); \
            if (threadIdx.x == 0) g_tp[(k)] = clock64(); \
        } \
    } while (0)

struct TCtx {
    unsigned char* sm;
    const TailArgs* a;
    const TailHdr* hd;
    unsigned rank;
    int par;
    __device__ double* vec(int v) const { return reinterpret_cast<double*>(sm + a->L.vec) + (size_t)v * a->L.rmax; }
    __device__ double* win() const { return reinterpret_cast<double*>(sm + a->L.win); }
    __device__ double* psum() const { return reinterpret_cast<double*>(sm + a->L.psum); }
    __device__ RowSet A() const { return rowset(sm, a->L.A, hd->R, hd->np, hd->nl); }
    __device__ void mark(int k) const {
        if (a->prof) smark(k);
    }
    // the tail level's row sums (optional diagnostics marks)
    template <class G, class E>
    __device__ void rowsA(const G& g, E& e, int mk = -1) const {
        mark(mk);
        rowsum<false>(A(), win(), psum(), g, e, self(), mk >= 0 ? mk + 10 : -1);
        mark(mk >= 0 ? mk + 1 : -1);
    }
    // padding column for gathers: hub slot 0 (a local copy; no cluster traffic)
    __device__ int self() const { return (int)(kHub << 16); }
    __device__ double* hc(int v) const { return reinterpret_cast<double*>(sm + a->L.hcache) + v * kTailMaxHubs; }
    __device__ VRef ref(int v) const { return VRef(vec(v), hc(v), rank); }
    __device__ VRef invm() const {
        return VRef(reinterpret_cast<const double*>(sm + a->L.invm), reinterpret_cast<const double*>(sm + a->L.hinvm),
                    rank);
    }
    // local copies of the hub columns of vectors v0 (, v1), final after the
    // last cluster barrier
    __device__ void refresh(int v0, int v1 = -1) const {
        const int t = threadIdx.x;
        if (t < a->nhub) {
            hc(v0)[t] = *dsm(vec(v0), a->hubpk[t]);
            if (v1 >= 0) hc(v1)[t] = *dsm(vec(v1), a->hubpk[t]);
        }
        __syncthreads();
    }
};

// cluster-wide sum of K values (every thread contributes v; every thread of
// every CTA gets the same t)
template <int K>
__device__ void cred(TCtx& c, const double (&v)[K], double (&t)[K]) {
    double* bs = reinterpret_cast<double*>(c.sm + c.a->L.bsum);
    double s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = block_sum<kTailThreads>(v[k], bs);
    double* slot = reinterpret_cast<double*>(c.sm + c.a->L.red) + c.par * (kTailMaxCs * 4);
    if ((int)threadIdx.x < c.a->cs) {
        double* dst = static_cast<double*>(__cluster_map_shared_rank(slot + c.rank * 4, threadIdx.x));
#pragma unroll
        for (int k = 0; k < K; ++k) dst[k] = s[k];
    }
    csync();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double x = 0.0;
        for (int q = 0; q < c.a->cs; ++q) x = __dadd_rn(x, slot[q * 4 + k]);
        t[k] = x;
    }
    c.par ^= 1;
}

// cycle(l) at the tail level from rin into z (U/solvers.py:128-157); the
// coarse correction is the exact coarsest solve.  vapp >= 0: also form the
// flexible-CG beta of the step that consumes z (fused beta dot); returns it.
// extra: a value to reduce along with the residual sum (single-aggregate
// coarsest only; -1 disables): its cluster total is returned in *extra_out
__device__ double tail_cycle(TCtx& c, int vin, int vz, int vapp, int vpp, double pap_prev, int m0,
                             double extra = 0.0, double* extra_out = nullptr) {
    const TailArgs& a = *c.a;
    const TailHdr& hd = *c.hd;
    const int R = hd.R;
    const double* invm = reinterpret_cast<const double*>(c.sm + a.L.invm);
    double* rin = c.vec(vin);
    const int dense = a.nc > 1;
    double ec1 = 0.0;
    double* ecv = reinterpret_cast<double*>(c.sm + a.L.cvec) + a.L.rcmax;  // owned coarse rows
    double* ecall = ecv + a.L.rcmax;                                         // replicated
    const RowSet A = c.A();
    if (a.pre) c.refresh(vin);
    const GPre1 pre1{c.invm(), c.ref(vin)};
    // residual r = rin - A xpre, restriction, coarsest solve
    if (!dense) {
        double s = 0.0;
        if (a.pre) {
            EResid e{rin, nullptr, 0.0};
            c.rowsA(pre1, e);
            s = e.s;
            TP(m0);
        } else {
            for (int i = threadIdx.x; i < R; i += kTailThreads) s += rin[i];
        }
        double t[2];
        if (extra_out) {
            cred<2>(c, {s, extra}, t);
            *extra_out = t[1];
        } else {
            cred<1>(c, {s}, *reinterpret_cast<double(*)[1]>(t));
        }
        TP(m0 + 1);
        ec1 = __dmul_rn(a.minv0, t[0]);
    } else {
        int vsrc = vin;
        if (a.pre) {
            EResid e{rin, c.vec(VR), 0.0};
            c.rowsA(pre1, e);
            vsrc = VR;
            csync();
        }
        double* rc = reinterpret_cast<double*>(c.sm + a.L.cvec);
        EStore es{rc};
        rowsum<true>(rowset(c.sm, a.L.Mout, hd.Rc, hd.cnp, hd.cnl), c.win(), c.psum(), GVec{saddr(c.vec(vsrc))}, es, (int)(c.rank << 16));
        csync();
        // ec = Minv rc on the owned coarse rows (k_dense_solve's order)
        const double* minv = reinterpret_cast<const double*>(c.sm + a.L.minv);
        const int lane = threadIdx.x & 31;
        for (int j = threadIdx.x >> 5; j < hd.Rc; j += kTailWarps) {
            double acc = 0.0;
            for (int q = lane; q < a.nc; q += 32)
                acc += minv[(size_t)j * a.nc + q] * *dsm(rc, ((q / a.Rc) << 16) | (q % a.Rc));
            acc = warp_sum(acc);
            if (lane == 0) ecv[j] = acc;
        }
        csync();
        // every CTA keeps the whole coarse correction
        for (int q = threadIdx.x; q < a.nc; q += kTailThreads) ecall[q] = *dsm(ecv, ((q / a.Rc) << 16) | (q % a.Rc));
        __syncthreads();
    }
    // prolongation + post-smoothing (+ the beta dot)
    const GUp up{c.invm(), c.ref(vin), reinterpret_cast<const int*>(c.sm + a.L.v2a), saddr(c.sm + a.L.v2a),
                 saddr(c.sm + a.L.hv2a), ecall, a.pre, dense, ec1};
    double* z = c.vec(vz);
    const double* app = vapp >= 0 ? c.vec(vapp) : nullptr;
    const double* pp = vapp >= 0 ? c.vec(vpp) : nullptr;
    double sb = 0.0, sb2 = 0.0;
    if (a.post) {
        ESweep e{invm, rin, z, app, up, 0.0};
        c.rowsA(up, e, m0 == 30 ? 44 : -1);
        sb = e.s;
        TP(m0 + 2);
    } else {
        for (int i = threadIdx.x; i < R; i += kTailThreads) {
            const double zi = up.at(i);
            z[i] = zi;
            if (app) {
                sb += zi * app[i];
                sb2 += pp[i] * app[i];
            }
        }
    }
    if (vapp < 0) {
        csync();
        return 0.0;
    }
    if (a.post) {
        double t[1];
        cred<1>(c, {sb}, t);
        return -t[0] / pap_prev;  // EpiSweepBeta::fin
    }
    double t[2];
    cred<2>(c, {sb, sb2}, t);
    return -t[0] / t[1];  // BodyBeta::fin
}

// the level above's prolongated iterate x = 0 + invm b + (valid ? e_c[v2a] : 0)
// over its rows, split evenly between the CTAs, once every CTA has written
// its rows of e_c (a.out)
__device__ void materialise_up(TCtx& c, int valid) {
    const TailArgs& a = *c.a;
    csync();
    const int per = (a.xn + a.cs - 1) / a.cs;
    const int i1 = min(a.xn, ((int)c.rank + 1) * per);
    for (int i = (int)c.rank * per + threadIdx.x; i < i1; i += kTailThreads) {
        const double xp = __dadd_rn(0.0, __dmul_rn(a.xinvm[i], a.xb[i]));
        a.xout[i] = __dadd_rn(xp, valid ? __ldcg(a.out + a.xv2a[i]) : 0.0);
    }
}

__global__ void __launch_bounds__(kTailThreads, 1) k_tail(const __grid_constant__ TailArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const unsigned rank = cta_rank();
    if (a.prof && threadIdx.x < kTailProfMarks) g_tp[threadIdx.x] = threadIdx.x == 0 ? clock64() : 0;
    {
        // static per-CTA data, before the dependency wait: bulk copies
        // (cp.async.bulk, mbarrier completion) instead of a load/store loop
        __shared__ __align__(8) uint64_t stage_bar;
        const unsigned char* src = a.blob + (size_t)rank * a.L.blob_bytes;
        if (threadIdx.x == 0) {
            mbar_init(&stage_bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&stage_bar, (unsigned)a.L.blob_bytes);
            constexpr int kChunk = 32768;
            for (int off = 0; off < a.L.blob_bytes; off += kChunk)
                bulk_g2s(sm + off, src + off, (unsigned)min(kChunk, a.L.blob_bytes - off), &stage_bar);
        }
        __syncthreads();
        mbar_wait(&stage_bar, 0);
    }
    pdl_wait();
    pdl_trigger();
    if (a.gate && *(volatile const int*)a.gate == 0) {  // same value in every CTA
        if (rank == 0 && threadIdx.x == 0 && a.upd0) *a.upd0 = 0;
        return;
    }
    TCtx c{sm, &a, reinterpret_cast<const TailHdr*>(sm), rank, 0};
    TP(1);
    const TailHdr& hd = *c.hd;
    const int R = hd.R;
    // restriction of the level above's residual: b = P^T r (+ ||b||^2)
    EStoreNorm eb{c.vec(VB), 0.0};
    rowsum<true>(rowset(sm, a.L.Min, R, hd.mnp, hd.mnl), c.win(), c.psum(), GGlobal{a.rprev}, eb, 0);
    TP(2);
    if (a.steps == 0) {
        csync();
        tail_cycle(c, VB, VZ, -1, -1, 0.0, 10);
        const double* z = c.vec(VZ);
        for (int i = threadIdx.x; i < R; i += kTailThreads) a.out[hd.row0 + i] = z[i];
        if (a.xout) materialise_up(c, 1);
        return;  // last cluster access was before tail_cycle's final barrier
    }
    // ||b||: with a single-aggregate coarsest level it rides in the first
    // cycle's residual reduction (a zero b then yields p'Ap = 0 below, the
    // same "no update" outcome as the skipped FCG); otherwise its own
    const bool fold_bn = a.nc == 1;
    double bn2 = 0.0;
    if (fold_bn) {
        csync();  // b visible to the first cycle's gathers
    } else {
        double tb[1];
        cred<1>(c, {eb.s}, tb);
        bn2 = tb[0];
    }
    TP(3);
    int upd0 = 0;
    double bnorm = sqrt(bn2);
    if (fold_bn || !(bnorm <= 1e-14 * bnorm)) {  // EpiRestrictBegin::fin gate[0]
        double pap_prev = 0.0;
        for (int k = 0; k < a.steps; ++k) {
            const int vin = k == 0 ? VB : VRF;
            const int pc = (k & 1) ? VP1 : VP0, pp = (k & 1) ? VP0 : VP1;
            const int apc = (k & 1) ? VAP1 : VAP0, app = (k & 1) ? VAP0 : VAP1;
            const double beta = tail_cycle(c, vin, VZ, k > 0 ? app : -1, pp, pap_prev, 10 + 20 * k, eb.s,
                                           (fold_bn && k == 0) ? &bn2 : nullptr);
            if (fold_bn && k == 0) {
                bnorm = sqrt(bn2);
                if (bnorm <= 1e-14 * bnorm) break;  // gate[0] = 0: b == 0, no update
            }
            // direction p = z + beta pprev, Ap, p.Ap, p.r (EpiDirFcg)
            c.refresh(VZ, k > 0 ? pp : -1);
            EDir e{c.vec(vin), c.vec(pc), c.vec(apc), GDir{c.ref(VZ), c.ref(pp), k > 0, beta}, 0.0, 0.0};
            c.rowsA(e.g, e);
            TP(16 + 20 * k);
            double t2[2];
            cred<2>(c, {e.s0, e.s1}, t2);
            TP(17 + 20 * k);
            if (!(t2[0] > 0.0)) break;  // U/solvers.py:178-180
            const double alpha = t2[1] / t2[0];
            pap_prev = t2[0];
            if (k == 0) upd0 = 1;
            // x += alpha p, r -= alpha Ap, ||r|| (BodyFcgUpd)
            double* x = c.vec(VX);
            const double* p = c.vec(pc);
            const double* ap = c.vec(apc);
            const double* ri = c.vec(vin);
            double* rf = c.vec(VRF);
            if (k == a.steps - 1) {
                // last step: the residual and its norm (gate[steps]) have no
                // reader -- only x leaves the tail
                for (int i = threadIdx.x; i < R; i += kTailThreads) {
                    const double xo = k == 0 ? 0.0 : x[i];
                    x[i] = __dadd_rn(xo, __dmul_rn(alpha, p[i]));
                }
                break;
            }
            double s = 0.0;
            for (int i = threadIdx.x; i < R; i += kTailThreads) {
                const double xo = k == 0 ? 0.0 : x[i];
                x[i] = __dadd_rn(xo, __dmul_rn(alpha, p[i]));
                const double rn = __dsub_rn(ri[i], __dmul_rn(alpha, ap[i]));
                rf[i] = rn;
                s += rn * rn;
            }
            TP(18 + 20 * k);
            double t1[1];
            cred<1>(c, {s}, t1);
            TP(19 + 20 * k);
            if (sqrt(t1[0]) <= 1e-14 * bnorm) break;  // gate[k + 1] = 0
        }
    }
    if (upd0) {
        const double* x = c.vec(VX);
        for (int i = threadIdx.x; i < R; i += kTailThreads) a.out[hd.row0 + i] = x[i];
    }
    if (rank == 0 && threadIdx.x == 0) *a.upd0 = upd0;
    if (a.xout) materialise_up(c, upd0);
    TP(60);
    if (a.prof && threadIdx.x < kTailProfMarks) a.prof[rank * kTailProfMarks + threadIdx.x] = g_tp[threadIdx.x];
}

// ------------------------------------------------------------------ host plan
struct HostRows {
    std::vector<int> rp, idx, lptr, lrow;
    std::vector<double> val;
    std::vector<int4> pc;
};

// long rows of a local CSR become 256-entry pieces (build_groups' split)
inline void add_pieces(HostRows& h) {
    h.lptr.assign(1, 0);
    h.lrow.clear();
    h.pc.clear();
    int slot = 0;
    const int R = (int)h.rp.size() - 1;
    for (int i = 0; i < R; ++i) {
        const int b = h.rp[i], e = h.rp[i + 1];
        if (e - b <= kTailLongMin) continue;
        for (int eb = b; eb < e; eb += kTailLongMin) h.pc.push_back(make_int4(i, eb, std::min(eb + kTailLongMin, e), slot++));
        h.lrow.push_back(i);
        h.lptr.push_back(slot);
    }
}

// rows [r0, r1) of a CSR (global row pointer grp): local offsets, entries
// mapped by f
template <class F>
HostRows slice_rows(int r0, int r1, const int* grp, const int* gidx, const double* gval, F f) {
    HostRows h;
    const int R = r1 - r0;
    h.rp.resize(R + 1);
    const int base = grp[r0];  // (r0 <= n: an empty block starts at row r0 too)
    for (int i = 0; i <= R; ++i) h.rp[i] = grp[r0 + i] - base;
    const int nnz = h.rp[R];
    h.idx.resize(nnz);
    if (gval) h.val.resize(nnz);
    for (int k = 0; k < nnz; ++k) {
        h.idx[k] = f(gidx[base + k]);
        if (gval) h.val[k] = gval[base + k];
    }
    add_pieces(h);
    return h;
}

struct Bump {
    int off = 0;
    int take(size_t bytes) {
        const int o = off;
        off += (int)((bytes + 15) & ~size_t(15));
        return o;
    }
};

}  // namespace

bool build_tail(const TailInputs& in, TailPlan& tp, cudaStream_t s) {
    tp.on = false;
    const int n = in.n;
    if (n <= 0 || in.nc <= 0) return false;
    int cs = kTailMaxCs;
    while (cs > 1 && n < cs * 64) cs >>= 1;
    const long long nnz = in.rp[n];
    (void)nnz;
    // contiguous row blocks of about equal work: a warp unit is a 32-row
    // group or a 256-entry piece of a long row, so rows cost 1/32 unit and a
    // long row its piece count (a hub row gets a CTA of its own)
    auto cost = [&](int i) {
        const int len = in.rp[i + 1] - in.rp[i];
        return len > kTailLongMin ? (double)((len + kTailLongMin - 1) / kTailLongMin) : 1.0 / 32;
    };
    double total = 0;
    for (int i = 0; i < n; ++i) total += cost(i);
    std::vector<int> cut(cs + 1, n);
    cut[0] = 0;
    {
        double acc = 0;
        int c = 1;
        for (int i = 0; i < n && c < cs; ++i) {
            const double ci = cost(i);
            const bool big = ci * cs > total;  // alone more than a share: a block of its own
            if (big && i > cut[c - 1]) cut[c++] = i;
            if (c >= cs) break;
            acc += ci;
            if (big || acc * cs >= total * c) cut[c++] = i + 1;
        }
        for (; c < cs; ++c) cut[c] = n;
        for (int k = 1; k <= cs; ++k) cut[k] = std::max(cut[k], cut[k - 1]);
    }
    int R = 0;
    std::vector<int> own(n), loc(n);
    for (int c = 0; c < cs; ++c) {
        R = std::max(R, cut[c + 1] - cut[c]);
        for (int i = cut[c]; i < cut[c + 1]; ++i) { own[i] = c; loc[i] = i - cut[c]; }
    }
    if (R > 65535 || R == 0) return false;
    // hub columns: the most-referenced columns with at least kTailHubDeg rows
    std::vector<int> deg(n, 0), hslot(n, -1), hubs;
    for (long long k = 0; k < nnz; ++k) deg[in.ci[k]]++;
    for (int j = 0; j < n; ++j)
        if (deg[j] >= kTailHubDeg) hubs.push_back(j);
    std::sort(hubs.begin(), hubs.end(), [&](int x, int y) { return deg[x] != deg[y] ? deg[x] > deg[y] : x < y; });
    if ((int)hubs.size() > kTailMaxHubs) hubs.resize(kTailMaxHubs);
    for (int t = 0; t < (int)hubs.size(); ++t) hslot[hubs[t]] = t;
    const bool dense = in.nc > 1;
    const int Rc = dense ? (in.nc + cs - 1) / cs : 0;
    auto pk = [&](int k) { return (own[k] << 16) | loc[k]; };
    auto pkA = [&](int k) { return hslot[k] >= 0 ? (int)((kHub << 16) | (unsigned)hslot[k]) : pk(k); };
    struct Cta {
        TailHdr h;
        HostRows A, Min, Mout;
    };
    std::vector<Cta> ct(cs);
    size_t eA = 0, pA = 0, lA = 0, eM = 0, pM = 0, lM = 0, eC = 0, pC = 0, lC = 0;
    for (int c = 0; c < cs; ++c) {
        const int r0 = cut[c], r1 = cut[c + 1];
        Cta& t = ct[c];
        t.A = slice_rows(r0, r1, in.rp.data(), in.ci.data(), in.av.data(), pkA);
        t.Min = slice_rows(r0, r1, in.mp.data(), in.mem.data(), nullptr, [](int k) { return k; });
        std::memset(&t.h, 0, sizeof(t.h));
        t.h.R = r1 - r0;
        t.h.np = (int)t.A.pc.size();
        t.h.nl = (int)t.A.lrow.size();
        t.h.mnp = (int)t.Min.pc.size();
        t.h.mnl = (int)t.Min.lrow.size();
        t.h.row0 = r0;
        if (dense) {
            const int j0 = std::min(in.nc, c * Rc), j1 = std::min(in.nc, (c + 1) * Rc);
            t.Mout = slice_rows(j0, j1, in.cp.data(), in.cmem.data(), nullptr, pk);
            t.h.Rc = j1 - j0;
            t.h.cnp = (int)t.Mout.pc.size();
            t.h.cnl = (int)t.Mout.lrow.size();
            t.h.crow0 = j0;
        }
        eA = std::max(eA, t.A.idx.size()); pA = std::max(pA, t.A.pc.size()); lA = std::max(lA, t.A.lrow.size());
        eM = std::max(eM, t.Min.idx.size()); pM = std::max(pM, t.Min.pc.size()); lM = std::max(lM, t.Min.lrow.size());
        eC = std::max(eC, t.Mout.idx.size()); pC = std::max(pC, t.Mout.pc.size()); lC = std::max(lC, t.Mout.lrow.size());
    }
    // layout
    TailLayout L;
    Bump b;
    b.take(sizeof(TailHdr));
    auto rows_layout = [&](TailRows& t, int nrows, size_t ne, size_t np, size_t nl, bool val) {
        t.rp = b.take(sizeof(int) * (nrows + 1));
        t.idx = b.take(sizeof(int) * std::max<size_t>(ne, 1));
        t.val = val ? b.take(sizeof(double) * std::max<size_t>(ne, 1)) : -1;
        t.pc = b.take(sizeof(int4) * std::max<size_t>(np, 1));
        t.lptr = b.take(sizeof(int) * (nl + 1));
        t.lrow = b.take(sizeof(int) * std::max<size_t>(nl, 1));
    };
    rows_layout(L.A, R, eA, pA, lA, true);
    rows_layout(L.Min, R, eM, pM, lM, false);
    if (dense) rows_layout(L.Mout, Rc, eC, pC, lC, false);
    L.invm = b.take(sizeof(double) * R);
    L.v2a = b.take(sizeof(int) * R);
    L.hinvm = b.take(sizeof(double) * kTailMaxHubs);
    L.hv2a = b.take(sizeof(int) * kTailMaxHubs);
    if (dense) L.minv = b.take(sizeof(double) * (size_t)Rc * in.nc);
    L.blob_bytes = b.off;
    L.rmax = R;
    L.rcmax = Rc;
    L.vec = b.take(sizeof(double) * (size_t)kTailVecs * R);
    L.win = b.take(sizeof(double) * kTailWarps * 256);
    L.psum = b.take(sizeof(double) * std::max<size_t>({pA, pM, pC, (size_t)1}));
    L.red = b.take(sizeof(double) * 2 * kTailMaxCs * 4);
    L.bsum = b.take(sizeof(double) * (kTailThreads / 32 + 1));
    L.cvec = b.take(sizeof(double) * (2 * std::max(Rc, 1) + std::max(in.nc, 1)));
    L.hcache = b.take(sizeof(double) * kTailVecs * kTailMaxHubs);
    L.smem_bytes = b.off;
    if (L.smem_bytes > kTailSmemMax) return false;
    // blobs
    std::vector<unsigned char> host((size_t)cs * L.blob_bytes, 0);
    for (int c = 0; c < cs; ++c) {
        unsigned char* B = host.data() + (size_t)c * L.blob_bytes;
        const Cta& t = ct[c];
        std::memcpy(B, &t.h, sizeof(TailHdr));
        auto put_rows = [&](const TailRows& lay, const HostRows& h, int nrows) {
            // rows past R keep the end offset (empty)
            std::vector<int> rp(nrows + 1, h.rp.empty() ? 0 : h.rp.back());
            std::copy(h.rp.begin(), h.rp.end(), rp.begin());
            std::memcpy(B + lay.rp, rp.data(), sizeof(int) * rp.size());
            if (!h.idx.empty()) std::memcpy(B + lay.idx, h.idx.data(), sizeof(int) * h.idx.size());
            if (lay.val >= 0 && !h.val.empty()) std::memcpy(B + lay.val, h.val.data(), sizeof(double) * h.val.size());
            if (!h.pc.empty()) std::memcpy(B + lay.pc, h.pc.data(), sizeof(int4) * h.pc.size());
            std::memcpy(B + lay.lptr, h.lptr.data(), sizeof(int) * h.lptr.size());
            if (!h.lrow.empty()) std::memcpy(B + lay.lrow, h.lrow.data(), sizeof(int) * h.lrow.size());
        };
        put_rows(L.A, t.A, R);
        put_rows(L.Min, t.Min, R);
        if (dense) put_rows(L.Mout, t.Mout, Rc);
        const int r0 = t.h.row0;
        std::memcpy(B + L.invm, in.invm.data() + r0, sizeof(double) * t.h.R);
        for (int h = 0; h < (int)hubs.size(); ++h) {
            reinterpret_cast<double*>(B + L.hinvm)[h] = in.invm[hubs[h]];
            if (dense) reinterpret_cast<int*>(B + L.hv2a)[h] = in.v2a[hubs[h]];
        }
        if (dense) {
            std::memcpy(B + L.v2a, in.v2a.data() + r0, sizeof(int) * t.h.R);
            std::memcpy(B + L.minv, in.minv.data() + (size_t)t.h.crow0 * in.nc, sizeof(double) * (size_t)t.h.Rc * in.nc);
        }
    }
    tp.blob.alloc(host.size(), s);
    UA_CK(cudaMemcpyAsync(tp.blob.p, host.data(), host.size(), cudaMemcpyHostToDevice, s));
    UA_CK(cudaStreamSynchronize(s));  // host staging vector is a temporary
    const int dev = cur_dev();
    static bool attr_done_dev[kMaxDevices] = {};
    bool& attr_done = attr_done_dev[dev];
    if (!attr_done) {
        UA_CK(cudaFuncSetAttribute(k_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        UA_CK(cudaFuncSetAttribute(k_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, kTailSmemMax));
        attr_done = true;
    }
    static std::map<std::pair<int, int>, bool> fits_cache_dev[kMaxDevices];  // (cs, smem) -> a cluster fits
    auto& fits_cache = fits_cache_dev[dev];
    auto fc = fits_cache.find({cs, L.smem_bytes});
    if (fc != fits_cache.end()) {
        if (!fc->second) return false;
    } else {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(cs);
        lc.blockDim = dim3(kTailThreads);
        lc.dynamicSmemBytes = L.smem_bytes;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        int ncl = 0;
        const bool ok = cudaOccupancyMaxActiveClusters(&ncl, k_tail, &lc) == cudaSuccess && ncl >= 1;
        if (!ok) (void)cudaGetLastError();
        fits_cache[{cs, L.smem_bytes}] = ok;
        if (!ok) return false;
    }
    TailArgs& a = tp.args;
    a = TailArgs{};
    a.blob = tp.blob.p;
    a.L = L;
    a.cs = cs;
    a.Rc = Rc;
    a.nhub = (int)hubs.size();
    for (int h = 0; h < a.nhub; ++h) a.hubpk[h] = pk(hubs[h]);
    a.nc = in.nc;
    a.pre = in.pre;
    a.post = in.post;
    a.steps = in.steps;
    a.minv0 = dense ? 0.0 : in.minv[0];
    if (getenv("UAAMG_TAIL_PROF")) {
        tp.prof.alloc((size_t)cs * kTailProfMarks, s);
        UA_CK(cudaMemsetAsync(tp.prof.p, 0, sizeof(long long) * cs * kTailProfMarks, s));
        a.prof = tp.prof.p;
        std::vector<int> e(cs), pc(cs);
        for (int c = 0; c < cs; ++c) { e[c] = (int)ct[c].A.idx.size(); pc[c] = ct[c].h.np; }
        for (int c = 0; c < cs; ++c) fprintf(stderr, " %d", ct[c].h.R);
        fprintf(stderr, "tail: n %d cs %d Rmax %d hubs %d smem %d blob %d; per-CTA rows/nnz/pieces:", n, cs, R,
                (int)hubs.size(), L.smem_bytes, L.blob_bytes);
        for (int c = 0; c < cs; ++c) fprintf(stderr, " %d/%d", e[c], pc[c]);
        fprintf(stderr, "\n");
    }
    tp.on = true;
    return true;
}

void print_tail_prof(const TailPlan& tp) {
    if (!tp.prof.p) return;
    const int cs = tp.args.cs;
    std::vector<long long> t((size_t)cs * kTailProfMarks);
    UA_CK(cudaMemcpy(t.data(), tp.prof.p, sizeof(long long) * t.size(), cudaMemcpyDeviceToHost));
    for (int c = 0; c < cs; ++c) {
        const long long* r = t.data() + (size_t)c * kTailProfMarks;
        fprintf(stderr, "tail cta %2d:", c);
        for (int k = 1; k < kTailProfMarks; ++k)
            if (r[k]) fprintf(stderr, " %d:%lld", k, r[k] - r[0]);
        fprintf(stderr, "\n");
    }
}

void launch_tail(const TailPlan& tp, const double* rprev, const int* gate, double* out, int* upd0, cudaStream_t s,
                 const double* xb, double* xout) {
    TailArgs a = tp.args;
    a.rprev = rprev;
    a.gate = gate;
    a.out = out;
    a.upd0 = upd0;
    a.xb = xb;
    a.xout = a.xn > 0 ? xout : nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.cs);
    cfg.blockDim = dim3(kTailThreads);
    cfg.dynamicSmemBytes = a.L.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = a.cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    UA_CK(cudaLaunchKernelEx(&cfg, k_tail, a));
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace uaamg
