// csr_ell.cuh -- sliced-ELL row kernel for large levels of short rows.
//
// A derived, column-major copy of a CSR level in slices of 32 rows: slice s
// holds 32 x w_s entries (w_s = its longest row), entry (row 32s + l, k) at
// off[s] + 32 k + l; padding entries (k >= the row's length) hold column =
// the row itself and value 0 and are never folded.  A warp owns a slice and
// lane l its row: every index / value load of the warp is one contiguous
// 128 / 256-byte line, and the gathers of 32 consecutive rows' k-th entries
// are (for banded matrices) contiguous too.  No shared-memory staging, so
// occupancy is register-bound instead of stage-bound -- this is what the
// 27-point levels need (their 128-row TMA stages leave 2-3 CTAs per SM).
// Each lane folds its row in CSR order from 0.0 without FMA: the same bits as
// every other row kernel (K/numba_backend.py:47-56).
#pragma once
#include "solve_ops.cuh"

namespace uaamg {

constexpr int kEllMaxRow = 32;      // longest row the ELL copy takes
constexpr int kEllWarps = 8;        // warps (slices in flight) per CTA
constexpr double kEllMaxPad = 1.10; // max (slab entries / nonzeros)
constexpr int kEllMinRows = 1 << 20; // smaller levels keep the tile / group kernels (no gain, setup cost)

struct Ell {
    const long long* off = nullptr;  // nslices + 1 entry offsets
    const int* col = nullptr;
    const double* val = nullptr;
};

// builders (setup): 32 * (longest row) per slice, then the slab fill
static __global__ void k_ell_width(int n, int base, const int* __restrict__ rp, long long* __restrict__ slab) {
    const int lane = threadIdx.x & 31, nsl = (n + 31) >> 5;
    for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nsl; s += (gridDim.x * blockDim.x) >> 5) {
        const int r = (s << 5) + lane;
        const int len = r < n ? rp[base + r + 1] - rp[base + r] : 0;
        const int w = __reduce_max_sync(0xffffffffu, len);
        if (lane == 0) slab[s] = 32ll * w;
    }
}
static __global__ void k_ell_fill(int n, int base, const int* __restrict__ rp, const int* __restrict__ ci,
                                  const double* __restrict__ av, const long long* __restrict__ off, int* __restrict__ col,
                                  double* __restrict__ val) {
    const int lane = threadIdx.x & 31, nsl = (n + 31) >> 5;
    for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nsl; s += (gridDim.x * blockDim.x) >> 5) {
        const int r = (s << 5) + lane;
        const int i = base + min(r, n - 1);
        const int b = rp[i], len = r < n ? rp[i + 1] - b : 0;
        const long long o0 = off[s];
        const int w = (int)((off[s + 1] - o0) >> 5);
        for (int k = 0; k < w; ++k) {
            col[o0 + 32 * k + lane] = k < len ? ci[b + k] : i;
            val[o0 + 32 * k + lane] = k < len ? av[b + k] : 0.0;
        }
    }
}

template <class Src, class Epi, bool Unit>
__global__ void __launch_bounds__(32 * kEllWarps) k_ell(Csr A, int base, int n, Ell E, Src src_p, Epi epi_p) {
    pdl_wait();
    pdl_trigger();
    Epi epi = epi_p;
    if (!epi.gate()) {
        if (blockIdx.x == 0 && threadIdx.x == 0) epi.off();
        return;
    }
    Src src = src_p;
    src.init();
    const int lane = threadIdx.x & 31;
    const int nsl = (n + 31) >> 5;
    for (int s = blockIdx.x * kEllWarps + (threadIdx.x >> 5); s < nsl; s += gridDim.x * kEllWarps) {
        const int r = (s << 5) + lane;
        const bool valid = r < n;
        const int i = base + r;
        const int len = valid ? __ldg(A.rp + i + 1) - __ldg(A.rp + i) : 0;
        const long long o0 = __ldg(E.off + s);
        const int w = (int)((__ldg(E.off + s + 1) - o0) >> 5);
        const int* cp = E.col + o0 + lane;
        const double* vp = E.val + o0 + lane;
        double acc = 0.0;
        for (int k0 = 0; k0 < w; k0 += 8) {
            int c[8];
            double a[8], v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const bool in = k0 + q < w;  // warp-uniform: inside the slab (padding included)
                c[q] = in ? __ldg(cp + 32 * (k0 + q)) : i;
                if (!Unit) a[q] = in ? __ldg(vp + 32 * (k0 + q)) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = k0 + q < len ? src(c[q]) : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (k0 + q < len) acc = __dadd_rn(acc, Unit ? v[q] : __dmul_rn(a[q], v[q]));
        }
        if (valid) epi.row(i, acc, src);
    }
    if constexpr (Epi::K > 0) {
        double v[Epi::K];
        epi.vals(v);
        grid_reduce_finish<Epi::K, 32 * kEllWarps>(v, epi.red.partials, epi.red.ticket,
                                                    [&](const double (&t)[Epi::K]) {
                                                        if (!xpublish(epi.red, t)) epi.fin(t);
                                                    });
    }
}

}  // namespace uaamg
