// csr_group.cuh -- warp-granular CSR row kernel for every SpMV-shaped solve
// operation (residual, restriction, fused prolongation + sweep, direction
// SpMV), used by the standalone launches and by the persistent engine.
//
// Work unit = one warp.  Units [0, ng) are row groups of 32 consecutive rows
// (lane = row).  A group's nonzeros [rp[r0], rp[r0+32]) are contiguous, so
// the warp streams them in rounds of kGrpRound entries with fully coalesced
// loads -- all index/value loads of a round issued first, then all gathers
// (kGrpU independent loads in flight per lane per stage) -- and stages the
// products in a per-warp shared-memory window; each lane then folds the part
// of its own row that lies in the window into its accumulator.  Rounds are
// in ascending entry order, so every row is summed sequentially in ascending
// k from 0.0 with rounded products (-fmad=false): bit-identical to the
// reference's numba row loops (K/numba_backend.py:47-56, :276-285,
// :297-310) for ANY row length.
//
// Units [ng, ng + np) are pieces of long rows (more than long_min entries,
// solve path only): each piece sums <= kGrpRound entries with a warp tree,
// stores its partial, and the last piece of a row to arrive (atomic ticket)
// adds the row's partials in piece order and runs the epilogue --
// deterministic, not reference-ordered (the solve's parity bar is the 1e-10
// residual-history tolerance).  The lanes of the owning group skip such rows.
// A long row's share of a grid reduction is stored per row (G.lval) and
// folded in row order after the block partials, never into the partial of
// whichever block happened to finish the row.
#pragma once
#include "solve_ops.cuh"

namespace uaamg {

constexpr int kGrpU = 8;                  // entries per lane per round
constexpr int kGrpRound = 32 * kGrpU;     // 256 entries per round
constexpr int kGrpWarps = 8;              // warps per CTA (launch path)
constexpr int kGrpCtasPerSM = 8;          // launch path: grid cap = SMs x this (grid-stride over units)

template <bool Unit, class Src>
__device__ __forceinline__ double grp_prod(const Csr& A, const Src& src, int e) {
    const int k = __ldg(A.ci + e);
    return Unit ? src(k) : __dmul_rn(__ldg(A.av + e), src(k));
}

// One work unit.  win: this warp's kGrpRound-double shared window.
template <bool Unit, class Src, class Epi>
__device__ __forceinline__ void grp_unit(const Csr& A, const Groups& G, int u, const Src& src, Epi& epi,
                                         double* win) {
    const int lane = threadIdx.x & 31;
    if (u < G.ng) {
        const int i = G.base + (u << 5) + lane;
        const int rlast = G.base + min((u << 5) + 32, G.n);
        const bool valid = i < G.base + G.n;
        const int bi = valid ? __ldg(A.rp + i) : 0;
        const int ei = valid ? __ldg(A.rp + i + 1) : 0;
        const int e0 = __shfl_sync(0xffffffffu, bi, 0);
        const int e1 = __ldg(A.rp + rlast);
        const bool mine = valid && (ei - bi) <= G.long_min;
        double acc = 0.0;
        // stream [lo, hi) in rounds; each lane folds its row's part of a round
        auto stream = [&](int lo, int hi) {
            for (int base = lo; base < hi; base += kGrpRound) {
                int c[kGrpU];
                double a[kGrpU];
#pragma unroll
                for (int q = 0; q < kGrpU; ++q) {
                    const int e = base + lane + 32 * q;
                    c[q] = e < hi ? __ldg(A.ci + e) : -1;
                    if (!Unit) a[q] = e < hi ? __ldg(A.av + e) : 0.0;
                }
                double v[kGrpU];
#pragma unroll
                for (int q = 0; q < kGrpU; ++q) v[q] = c[q] >= 0 ? src(c[q]) : 0.0;
#pragma unroll
                for (int q = 0; q < kGrpU; ++q) win[lane + 32 * q] = Unit ? v[q] : __dmul_rn(a[q], v[q]);
                __syncwarp();
                if (mine) {
                    // sequential in k; window reads batched 8 at a time so
                    // only the DADD chain is serial, not LDS -> DADD
                    const int l1 = min(ei, base + kGrpRound) - base;
                    int e = max(bi, base) - base;
                    for (; e + 8 <= l1; e += 8) {
                        double w[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) w[q] = win[e + q];
#pragma unroll
                        for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, w[q]);
                    }
                    for (; e < l1; ++e) acc = __dadd_rn(acc, win[e]);
                }
                __syncwarp();
            }
        };
        // long rows of this group are pieces: stream around them
        unsigned lm = __ballot_sync(0xffffffffu, valid && !mine);
        int lo = e0;
        while (lm) {
            const int L = __ffs(lm) - 1;
            lm &= lm - 1;
            stream(lo, __shfl_sync(0xffffffffu, bi, L));
            lo = __shfl_sync(0xffffffffu, ei, L);
        }
        stream(lo, e1);
        if (mine) epi.row(i, acc, src);
    } else {
        const int4 pc = G.piece[u - G.ng];
        const int row = pc.x, eb = pc.y, ee = pc.z, lr = pc.w;
        double part = 0.0;
#pragma unroll
        for (int q = 0; q < kGrpU; ++q) {
            const int e = eb + lane + 32 * q;
            if (e < ee) part = __dadd_rn(part, grp_prod<Unit>(A, src, e));
        }
        part = warp_sum(part);
        const int p0 = G.pbase[lr], np = G.pbase[lr + 1] - p0;
        const int slot = p0 + (eb - __ldg(A.rp + row)) / kGrpRound;
        bool last = false;
        if (lane == 0) {
            G.part[slot] = part;
            unsigned prev;  // acq_rel: releases this piece, the last arriver acquires all
            asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(G.ticket + lr) : "memory");
            last = prev == (unsigned)(np - 1);
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
            // all partials loaded at once (lane k: pieces k, k+32, ...), then a
            // fixed-shape warp tree: one L2 round trip instead of np
            double acc = 0.0;
            for (int k = lane; k < np; k += 32) acc = __dadd_rn(acc, __ldcg(G.part + p0 + k));
            acc = warp_sum(acc);
            if (lane == 0) {
                G.ticket[lr] = 0u;
                if constexpr (Epi::K > 0) {
                    // which warp finishes a long row depends on arrival order:
                    // its reduced values go to the row's own slot (folded in
                    // row order by the reduction's finisher), not into this
                    // thread's partials -- same bits on every run
                    Epi e1 = epi;
                    e1.clear();
                    e1.row(row, acc, src);
                    double d[Epi::K];
                    e1.vals(d);
#pragma unroll
                    for (int k = 0; k < Epi::K; ++k) G.lval[kMaxLongK * lr + k] = d[k];
                } else {
                    epi.row(row, acc, src);
                }
            }
        }
    }
}

// before the dependency wait: pull this warp's first row group of the
// (read-only) matrix into L1 while the predecessor kernel drains
template <bool Unit>
__device__ __forceinline__ void prefetch_first_group(const Csr& A, const Groups& G) {
    const int u0 = blockIdx.x * kGrpWarps + (threadIdx.x >> 5);
    if (u0 < G.ng) {
        const int lane = threadIdx.x & 31;
        const int r0 = G.base + (u0 << 5);
        const int e0 = __ldg(A.rp + r0), e1 = __ldg(A.rp + G.base + min((u0 << 5) + 32, G.n));
        const int cb = (e0 * 4) & ~127, ce = e1 * 4;  // col bytes [cb, ce)
        for (int o = cb + lane * 128; o < ce; o += 32 * 128) pf(reinterpret_cast<const char*>(A.ci) + o);
        if (!Unit) {
            const long long vb = ((long long)e0 * 8) & ~127ll, ve = (long long)e1 * 8;
            for (long long o = vb + lane * 128; o < ve; o += 32 * 128) pf(reinterpret_cast<const char*>(A.av) + o);
        }
    }
}

// Launch-path kernel: one unit per warp, kGrpWarps warps per CTA, optional
// deterministic grid reduction (Epi::K > 0) through the ticketed partials.
template <class Src, class Epi, bool Unit>
__global__ void __launch_bounds__(32 * kGrpWarps) k_csr_group(Csr A, Groups G, Src src_p, Epi epi_p) {
    __shared__ double win[kGrpWarps][kGrpRound];
    prefetch_first_group<Unit>(A, G);
    pdl_wait();
    pdl_trigger();
    Epi epi = epi_p;
    if (!epi.gate()) {
        if (blockIdx.x == 0 && threadIdx.x == 0) epi.off();
        return;
    }
    Src src = src_p;
    src.init();
    const int nu = G.units();
    for (int u = blockIdx.x * kGrpWarps + (threadIdx.x >> 5); u < nu; u += gridDim.x * kGrpWarps)
        grp_unit<Unit>(A, G, u, src, epi, win[threadIdx.x >> 5]);
    if constexpr (Epi::K > 0) {
        double v[Epi::K];
        epi.vals(v);
        grid_reduce_finish<Epi::K>(v, epi.red.partials, epi.red.ticket, [&](const double (&t)[Epi::K]) {
            if (!xpublish(epi.red, t)) epi.fin(t);
        }, G.lval, G.nlong);
    }
}

// Flexible-CG direction SpMV fused with the update that consumes it
// (U/solvers.py:173-185): phase 1 is k_csr_group's direction + Ap + p.Ap,
// p.r; a grid barrier; every CTA folds the per-CTA partials in block order
// (same bits everywhere) and, unless p'Ap <= 0 (break), applies
// x += alpha p, r = r_in - alpha Ap on a grid-stride range and reduces ||r||
// through the ticketed last-block finish.  One cooperative launch instead of
// two dependent kernels; same arithmetic per element.
template <class Src>
__global__ void __launch_bounds__(32 * kGrpWarps) k_dir_update(Csr A, Groups G, Src src_p, EpiDirFcg epi_p,
                                                              BodyFcgUpd upd_p, double* part, unsigned* bar) {
    __shared__ double win[kGrpWarps][kGrpRound];
    __shared__ double sm[kThreads / 32 + 1];
    __shared__ double tot[2];
    prefetch_first_group<false>(A, G);
    pdl_wait();
    pdl_trigger();
    EpiDirFcg epi = epi_p;
    if (!epi.gate()) {
        // x keeps the earlier steps' value (valid iff step 0 updated it)
        if (upd_p.pu.n) upd_p.pu.run(upd_p.x, upd_p.step > 0 && *(volatile const int*)upd_p.pu.valid != 0);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            epi.off();
            upd_p.off();
        }
        return;
    }
    Src src = src_p;
    src.init();
    const int nu = G.units();
    for (int u = blockIdx.x * kGrpWarps + (threadIdx.x >> 5); u < nu; u += gridDim.x * kGrpWarps)
        grp_unit<false>(A, G, u, src, epi, win[threadIdx.x >> 5]);
    double v[2];
    epi.vals(v);
    const double b0 = block_sum<kThreads>(v[0], sm);
    const double b1 = block_sum<kThreads>(v[1], sm);
    const int nb = gridDim.x;
    if (threadIdx.x == 0) {
        part[blockIdx.x] = b0;
        part[nb + blockIdx.x] = b1;
    }
    coop_grid_sync(bar);
    if (threadIdx.x < 32) {
        double t0 = 0.0, t1 = 0.0;
        for (int b = threadIdx.x; b < nb; b += 32) {
            t0 += __ldcg(part + b);
            t1 += __ldcg(part + nb + b);
        }
        for (int r = threadIdx.x; r < G.nlong; r += 32) {  // long rows, row order
            t0 += __ldcg(G.lval + kMaxLongK * r);
            t1 += __ldcg(G.lval + kMaxLongK * r + 1);
        }
        t0 = warp_sum(t0);
        t1 = warp_sum(t1);
        if (threadIdx.x == 0) {
            tot[0] = t0;
            tot[1] = t1;
        }
    }
    __syncthreads();
    const double t[2] = {tot[0], tot[1]};
    if (blockIdx.x == 0 && threadIdx.x == 0) epi.fin(t);  // pap, pr, upd[step], alpha for later readers
    if (!(t[0] > 0.0)) {  // breakdown: the update is gated off (U/solvers.py:179-180)
        // (step 0 breaking down leaves x invalid; a later step leaves step
        // 0's x, which then was valid -- this step ran)
        if (upd_p.pu.n) upd_p.pu.run(upd_p.x, upd_p.step > 0);
        if (blockIdx.x == 0 && threadIdx.x == 0) upd_p.off();
        return;
    }
    BodyFcgUpd upd = upd_p;
    upd.alpha = t[1] / t[0];
    if (upd.last) {  // the last inner step: only x is read afterwards
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
            const double xo = upd.step == 0 ? 0.0 : upd.x[i];
            upd.x[i] = __dadd_rn(xo, __dmul_rn(upd.alpha, upd.p[i]));
        }
        if (upd.pu.n) {  // x final everywhere, then the parent's iterate
            coop_grid_sync(bar);
            upd.pu.run(upd.x, true);
        }
        return;
    }
    double s[1] = {0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) upd.item(i, s);
    grid_reduce_finish<1>(s, upd.red.partials, upd.red.ticket, [&](const double (&tt)[1]) { upd.fin(tt); });
}

}  // namespace uaamg
