// csr_stream.cuh -- the smem-staged CSR row kernel used by every SpMV-shaped
// operation on the solve path (SpMV, residual, Jacobi/l1 sweeps, restriction,
// FCG direction SpMV).
//
// One CTA owns a row block [r0, r1) whose nonzeros [rp[r0], rp[r1]) are
// contiguous in col/val.  Phase 1 streams that slice with coalesced loads
// (all 256 threads, independent x-gathers in flight) and stages the products
// a_k * x[col_k] in shared memory; phase 2 gives each row to one thread which
// folds its products sequentially in ascending k from 0.0.  Because the
// products are rounded before the adds (-fmad=false) and the fold order is
// the reference's, every row sum is bit-identical to the numba kernels
// (K/numba_backend.py:47-56, :297-310, :276-285).  Row blocks are precomputed
// so that a block's slice fits kStageCap products; a row longer than
// kStageHalf gets a block of its own and is folded chunk by chunk.
#pragma once
#include "common.cuh"

namespace uaamg {

// Epilogue contract:
//   __device__ void row(int i, double acc, const Src& src);   // per row
//   static constexpr int K;                                   // reduced values
//   __device__ void vals(double (&v)[K]) const;               // this thread's partials
//   __device__ void fin(const double (&tot)[K]);              // last block, thread 0
//   __device__ bool gate() const;                             // false: skip launch
//   __device__ void off();                                    // gate false: block 0 clears produced flags

struct NoReduce {
    static constexpr int K = 0;
};

template <int K>
struct RedSlot {
    double* partials;   // K * nb
    unsigned* ticket;   // zero between launches
};

// ExactLong: rows longer than kStageCap are folded sequentially on one thread
// (reference order, bit-exact; the kernel-table entry points) or, on the
// solve path, as a fixed-order block tree per chunk with chunk sums added in
// order (deterministic, not reference-ordered; the solve's parity bar is the
// 1e-10 residual-history tolerance).  Short rows are always exact.
template <class Src, class Epi, bool Unit, bool ExactLong = false>
__global__ void __launch_bounds__(kThreads) k_csr_stream(Csr A, Blocks B, Src src_p, Epi epi_p) {
    __shared__ double prod[kStageCap];
    Epi epi = epi_p;
    if (!epi.gate()) {
        if (blockIdx.x == 0 && threadIdx.x == 0) epi.off();
        return;
    }
    Src src = src_p;
    src.init();
    const int r0 = B.start[blockIdx.x], r1 = B.start[blockIdx.x + 1];
    const int e0 = A.rp[r0], e1 = A.rp[r1];
    if (e1 - e0 <= kStageCap) {
        // batches of kUnroll entries per thread: all index/value loads first,
        // then all gathers, so each warp keeps ~3*kUnroll loads in flight
        for (int base = e0 + (int)threadIdx.x; base < e1; base += kThreads * kUnroll) {
            int c[kUnroll];
            double a[kUnroll], v[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int e = base + u * kThreads;
                c[u] = e < e1 ? __ldg(A.ci + e) : -1;
                if (!Unit) a[u] = e < e1 ? __ldg(A.av + e) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) v[u] = c[u] >= 0 ? src(c[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int e = base + u * kThreads;
                if (e < e1) prod[e - e0] = Unit ? v[u] : __dmul_rn(a[u], v[u]);
            }
        }
        __syncthreads();
        for (int i = r0 + (int)threadIdx.x; i < r1; i += kThreads) {
            const int b = A.rp[i] - e0, c = A.rp[i + 1] - e0;
            double acc = 0.0;
            for (int e = b; e < c; ++e) acc = __dadd_rn(acc, prod[e]);
            epi.row(i, acc, src);
        }
    } else if (ExactLong) {
        // single long row: fold chunk by chunk on thread 0
        double acc = 0.0;
        for (int c0 = e0; c0 < e1; c0 += kStageCap) {
            const int c1 = min(c0 + kStageCap, e1);
            for (int e = c0 + (int)threadIdx.x; e < c1; e += kThreads) {
                const int c = __ldg(A.ci + e);
                prod[e - c0] = Unit ? src(c) : __dmul_rn(__ldg(A.av + e), src(c));
            }
            __syncthreads();
            if (threadIdx.x == 0)
                for (int e = 0; e < c1 - c0; ++e) acc = __dadd_rn(acc, prod[e]);
            __syncthreads();
        }
        if (threadIdx.x == 0) epi.row(r0, acc, src);
    } else {
        // single long row: per-thread strided partial sums, fixed block tree
        double part = 0.0;
        for (int e = e0 + (int)threadIdx.x; e < e1; e += kThreads) {
            const int c = __ldg(A.ci + e);
            part = __dadd_rn(part, Unit ? src(c) : __dmul_rn(__ldg(A.av + e), src(c)));
        }
        const double acc = block_sum<kThreads>(part, prod);
        if (threadIdx.x == 0) epi.row(r0, acc, src);
    }
    if constexpr (Epi::K > 0) {
        double v[Epi::K];
        epi.vals(v);
        grid_reduce_finish<Epi::K>(v, epi.red.partials, epi.red.ticket, [&](const double (&t)[Epi::K]) { epi.fin(t); });
    }
}

// ------------------------------------------------------------------ sources
// x_k read from a vector
struct SrcVec {
    const double* x;
    __device__ void init() {}
    __device__ double operator()(int k) const { return __ldg(x + k); }
};

// pre-smoothed iterate from a zero guess, one sweep: 0.0 + inv_m_k * b_k
// (K/numba_backend.py:304-309 with cur = 0: r = b - 0.0 = b)
struct SrcPre1 {
    const double* invm;
    const double* b;
    __device__ void init() {}
    __device__ double operator()(int k) const { return __dadd_rn(0.0, __dmul_rn(__ldg(invm + k), __ldg(b + k))); }
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
    __device__ double operator()(int k) const {
        double xp = mode == 0 ? 0.0
                  : mode == 1 ? __dadd_rn(0.0, __dmul_rn(__ldg(invm + k), __ldg(b + k)))
                              : __ldg(xpre + k);
        double e = valid ? __ldg(ec + __ldg(v2a + k)) : 0.0;
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
    __device__ double operator()(int k) const {
        double zk = __ldg(z + k);
        return have ? __dadd_rn(zk, __dmul_rn(beta, __ldg(pprev + k))) : zk;
    }
};

}  // namespace uaamg
