// csr_tma.cuh -- TMA-pipelined CSR row kernel for the large (HBM-bound)
// levels.
//
// Persistent CTAs of kTmaThreads threads walk R-row tiles (128; 64 for
// dense rows such as the 27-point stencil's).  Thread 0 streams
// each tile's row_ptr / col / val slices into a kTmaStages-deep shared-memory
// ring with cp.async.bulk (completion on an mbarrier), kTmaStages-1 tiles
// ahead of the tile being computed, so the matrix stream (12 B per nonzero,
// ~75% of the algorithmic bytes) is always in flight without holding
// registers.  Per tile: every thread prefetches its row's epilogue operands
// into L1, gathers src(col) for the tile's entries (batched, coalesced
// shared-memory reads of col), writes the rounded products over the staged
// values, and after a CTA barrier folds its own row sequentially in
// ascending k from 0.0 -- bit-identical to the reference's row loops
// (K/numba_backend.py:47-56, :297-310) -- then runs the epilogue.
// Used when every tile's nonzeros fit the stage (cap <= kTmaMaxCap).
#pragma once
#include "solve_ops.cuh"

namespace uaamg {

constexpr int kTmaThreads = 128;   // threads per CTA
constexpr int kTmaRows = 128;      // rows per tile (default); 64 for dense rows (27-point)
constexpr int kTmaStages = 3;
constexpr int kTmaMaxCap = 2048;      // max nonzeros per tile on this path
constexpr int kTmaRowParRows = 256;   // rows (= threads) per row-parallel tile
constexpr int kTmaRowParMaxRow = 12;  // longest row the row-parallel path takes
constexpr int kTmaBatch = 8;       // gathers in flight per thread
constexpr double kStreamHintBytes = 64.0 * 1024 * 1024;  // matrix streams above this load L2 evict-first

struct TmaLayout {
    int rp_off, ci_off, av_off, stage;
};
__host__ __device__ inline TmaLayout tma_layout(int cap, int rows = kTmaRows) {
    TmaLayout L;
    L.rp_off = 0;
    L.ci_off = ((rows + 8) * 4 + 127) & ~127;
    L.av_off = L.ci_off + (((cap + 8) * 4 + 127) & ~127);
    L.stage = L.av_off + (((cap + 4) * 8 + 127) & ~127);
    return L;
}
inline size_t tma_smem_bytes(int cap, int rows = kTmaRows, int stages = kTmaStages) {
    return (size_t)stages * tma_layout(cap, rows).stage + 16 * stages;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* m, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(m)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* m) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(m))
        : "memory");
}
// same with an L2 cache policy (evict_first: a matrix stream larger than L2
// should not push the coarse levels and the vectors out of it)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* m, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned round16(unsigned b) { return (b + 15u) & ~15u; }

// R rows per tile (<= kTmaThreads): the gathers of a tile are spread over
// all kTmaThreads threads, row folds are done by threads [0, R).
template <class Src, class Epi, bool Unit, int R = kTmaRows, int S = kTmaStages>
__global__ void __launch_bounds__(kTmaThreads) k_csr_tma(Csr A, int base, int end, int ntiles, int cap, Src src_p,
                                                         Epi epi_p, int stream_hint) {
    static_assert(R <= kTmaThreads && R % 4 == 0, "tile rows");
    extern __shared__ __align__(128) unsigned char smem[];
    Epi epi = epi_p;
    Src src = src_p;
    const TmaLayout Ly = tma_layout(cap, R);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + S * Ly.stage);
    const int t = threadIdx.x;
    const int G = gridDim.x;
    // tiles of this CTA: blockIdx.x + j * G
    const int my = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / G + 1 : 0;
    if (t == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&mbar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // producer (thread 0): issue tile j into stage j % S
    auto issue = [&](int j, int e0, int e1) {
        const int tile = blockIdx.x + j * G;
        const int s = j % S;
        unsigned char* st = smem + s * Ly.stage;
        const int r0 = base + tile * R, r1 = min(r0 + R, end);
        const int ra = r0 & ~3;  // 16-byte aligned row_ptr slice start
        const unsigned brp = round16((unsigned)(r1 - ra + 1) * 4u);
        const int ea = e0 & ~3, eb = e0 & ~1;
        const unsigned bci = round16((unsigned)(e1 - ea) * 4u);
        const unsigned bav = Unit ? 0u : round16((unsigned)(e1 - eb) * 8u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[s], brp + bci + bav);
        if (stream_hint) {
            const uint64_t pol = policy_evict_first();
            bulk_g2s_hint(st + Ly.rp_off, A.rp + ra, brp, &mbar[s], pol);
            if (bci) bulk_g2s_hint(st + Ly.ci_off, A.ci + ea, bci, &mbar[s], pol);
            if (bav) bulk_g2s_hint(st + Ly.av_off, A.av + eb, bav, &mbar[s], pol);
        } else {
            bulk_g2s(st + Ly.rp_off, A.rp + ra, brp, &mbar[s]);
            if (bci) bulk_g2s(st + Ly.ci_off, A.ci + ea, bci, &mbar[s]);
            if (bav) bulk_g2s(st + Ly.av_off, A.av + eb, bav, &mbar[s]);
        }
    };
    auto bounds = [&](int j, int& e0, int& e1) {
        const int r0 = base + (blockIdx.x + j * G) * R;
        e0 = __ldg(A.rp + r0);
        e1 = __ldg(A.rp + min(r0 + R, end));
    };
    int ne0 = 0, ne1 = 0;  // producer: bounds of the next tile to issue
    // the matrix is read-only: its first tiles stream in before the
    // dependency wait, overlapping the predecessor kernel's tail (PDL)
    if (t == 0) {
        for (int j = 0; j < min(my, S - 1); ++j) {
            int e0, e1;
            bounds(j, e0, e1);
            issue(j, e0, e1);
        }
        if (S - 1 < my) bounds(S - 1, ne0, ne1);
    }
    pdl_wait();
    pdl_trigger();
    if (!epi.gate()) {
        // gated off: drain the bulk copies already issued before leaving
        for (int j = 0; j < min(my, S - 1); ++j) mbar_wait(&mbar[j % S], 0);
        if (blockIdx.x == 0 && threadIdx.x == 0) epi.off();
        return;
    }
    src.init();
    // per-row operands may have been written by the predecessor: after the wait
    if (my > 0 && t < R && base + blockIdx.x * R + t < end) {
        epi.pre(base + blockIdx.x * R + t);
        src.pre(base + blockIdx.x * R + t);
    }
    // Software pipeline over this CTA's tiles: iteration j folds tile j
    // (products already in its stage) while the gathers of tile j + 1 are
    // in flight and tile j + 2 streams in by TMA.
    double v[kTmaBatch];
    int gb = 0, ge = 0, gea = 0;  // tile being gathered: entry range, col base
    // gather phase 1: issue the loads of tile jj's first batch
    auto gather_issue = [&](int jj) {
        const int s = jj % S;
        const unsigned char* st = smem + s * Ly.stage;
        const int r0 = base + (blockIdx.x + jj * G) * R;
        const int* rps = reinterpret_cast<const int*>(st + Ly.rp_off) + (r0 & 3);
        const int* cis = reinterpret_cast<const int*>(st + Ly.ci_off);
        mbar_wait(&mbar[s], (unsigned)((jj / S) & 1));
        gb = rps[0];
        ge = rps[min(R, end - r0)];
        gea = gb & ~3;
#pragma unroll
        for (int q = 0; q < kTmaBatch; ++q) {
            const int e = gb + t + q * kTmaThreads;
            v[q] = e < ge ? src(cis[e - gea]) : 0.0;
        }
    };
    // gather phase 2: products of tile jj into its stage (remaining batches
    // are gathered and consumed directly)
    auto gather_finish = [&](int jj) {
        const int s = jj % S;
        unsigned char* st = smem + s * Ly.stage;
        const int* cis = reinterpret_cast<const int*>(st + Ly.ci_off);
        double* avs = reinterpret_cast<double*>(st + Ly.av_off);
        const int eb = gb & ~1;
        for (int base = gb + t;; base += kTmaThreads * kTmaBatch) {
#pragma unroll
            for (int q = 0; q < kTmaBatch; ++q) {
                const int e = base + q * kTmaThreads;
                if (e < ge) avs[e - eb] = Unit ? v[q] : __dmul_rn(avs[e - eb], v[q]);
            }
            const int nb = base + kTmaThreads * kTmaBatch;
            if (nb >= ge) break;
#pragma unroll
            for (int q = 0; q < kTmaBatch; ++q) {
                const int e = nb + q * kTmaThreads;
                v[q] = e < ge ? src(cis[e - gea]) : 0.0;
            }
        }
    };
    if (my > 0) {
        gather_issue(0);
        gather_finish(0);
    }
    for (int j = 0; j < my; ++j) {
        __syncthreads();  // products of tile j complete; stage of tile j - 1 free
        // keep S - 1 tiles in flight beyond the one being folded
        if (t == 0 && j + S - 1 < my) {
            issue(j + S - 1, ne0, ne1);
            if (j + S < my) bounds(j + S, ne0, ne1);
        }
        const int s = j % S;
        const unsigned char* st = smem + s * Ly.stage;
        const int r0 = base + (blockIdx.x + j * G) * R;
        const int* rps = reinterpret_cast<const int*>(st + Ly.rp_off) + (r0 & 3);
        const double* avs = reinterpret_cast<const double*>(st + Ly.av_off);
        const int rows = min(R, end - r0);
        const int i = r0 + t;
        const bool valid = t < rows;
        if (j + 1 < my) {
            // next tile's row operands and first gather batch go out now
            const int i1 = r0 + G * R + t;
            if (t < R && i1 < end) {
                epi.pre(i1);
                src.pre(i1);
            }
            gather_issue(j + 1);
        }
        if (valid) {
            const int eb = rps[0] & ~1;
            const int b = rps[t] - eb, c = rps[t + 1] - eb;
            double acc = 0.0;
            for (int e = b; e < c; ++e) acc = __dadd_rn(acc, avs[e]);
            epi.row(i, acc, src);
        }
        if (j + 1 < my) gather_finish(j + 1);
    }
    if constexpr (Epi::K > 0) {
        double v[Epi::K];
        epi.vals(v);
        grid_reduce_finish<Epi::K, kTmaThreads>(v, epi.red.partials, epi.red.ticket, [&](const double (&tt)[Epi::K]) {
            if (!xpublish(epi.red, tt)) epi.fin(tt);
        });
    }
}

// Row-parallel variant for regular rows (every row of a tile short): the
// same TMA ring, but thread t gathers and folds ITS row directly from the
// staged col / val slices (8 gathers in flight, products folded in order as
// they arrive) -- no product round trip through shared memory and, for
// consecutive rows, coalesced gathers.  blockDim = R threads (one per row).
template <class Src, class Epi, bool Unit, int R, int S = kTmaStages>
__global__ void __launch_bounds__(R) k_csr_tma_rows(Csr A, int base, int end, int ntiles, int cap, Src src_p,
                                                    Epi epi_p, int stream_hint) {
    extern __shared__ __align__(128) unsigned char smem[];
    Epi epi = epi_p;
    Src src = src_p;
    const TmaLayout Ly = tma_layout(cap, R);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + S * Ly.stage);
    const int t = threadIdx.x;
    const int G = gridDim.x;
    const int my = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / G + 1 : 0;
    if (t == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&mbar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int j, int e0, int e1) {
        const int tile = blockIdx.x + j * G;
        const int s = j % S;
        unsigned char* st = smem + s * Ly.stage;
        const int r0 = base + tile * R, r1 = min(r0 + R, end);
        const int ra = r0 & ~3;
        const unsigned brp = round16((unsigned)(r1 - ra + 1) * 4u);
        const int ea = e0 & ~3, eb = e0 & ~1;
        const unsigned bci = round16((unsigned)(e1 - ea) * 4u);
        const unsigned bav = Unit ? 0u : round16((unsigned)(e1 - eb) * 8u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[s], brp + bci + bav);
        if (stream_hint) {
            const uint64_t pol = policy_evict_first();
            bulk_g2s_hint(st + Ly.rp_off, A.rp + ra, brp, &mbar[s], pol);
            if (bci) bulk_g2s_hint(st + Ly.ci_off, A.ci + ea, bci, &mbar[s], pol);
            if (bav) bulk_g2s_hint(st + Ly.av_off, A.av + eb, bav, &mbar[s], pol);
        } else {
            bulk_g2s(st + Ly.rp_off, A.rp + ra, brp, &mbar[s]);
            if (bci) bulk_g2s(st + Ly.ci_off, A.ci + ea, bci, &mbar[s]);
            if (bav) bulk_g2s(st + Ly.av_off, A.av + eb, bav, &mbar[s]);
        }
    };
    auto bounds = [&](int j, int& e0, int& e1) {
        const int r0 = base + (blockIdx.x + j * G) * R;
        e0 = __ldg(A.rp + r0);
        e1 = __ldg(A.rp + min(r0 + R, end));
    };
    int ne0 = 0, ne1 = 0;
    if (t == 0) {
        for (int j = 0; j < min(my, S - 1); ++j) {
            int e0, e1;
            bounds(j, e0, e1);
            issue(j, e0, e1);
        }
        if (S - 1 < my) bounds(S - 1, ne0, ne1);
    }
    pdl_wait();
    pdl_trigger();
    if (!epi.gate()) {
        for (int j = 0; j < min(my, S - 1); ++j) mbar_wait(&mbar[j % S], 0);
        if (blockIdx.x == 0 && threadIdx.x == 0) epi.off();
        return;
    }
    src.init();
    if (my > 0 && base + blockIdx.x * R + t < end) {
        epi.pre(base + blockIdx.x * R + t);
        src.pre(base + blockIdx.x * R + t);
    }
    for (int j = 0; j < my; ++j) {
        __syncthreads();  // every thread is done with the stage tile j + S - 1 reuses
        if (t == 0 && j + S - 1 < my) {
            issue(j + S - 1, ne0, ne1);
            if (j + S < my) bounds(j + S, ne0, ne1);
        }
        const int s = j % S;
        const unsigned char* st = smem + s * Ly.stage;
        const int r0 = base + (blockIdx.x + j * G) * R;
        const int* rps = reinterpret_cast<const int*>(st + Ly.rp_off) + (r0 & 3);
        const int* cis = reinterpret_cast<const int*>(st + Ly.ci_off);
        const double* avs = reinterpret_cast<const double*>(st + Ly.av_off);
        mbar_wait(&mbar[s], (unsigned)((j / S) & 1));
        const int i = r0 + t;
        if (j + 1 < my) {
            const int i1 = r0 + G * R + t;
            if (i1 < end) {
                epi.pre(i1);
                src.pre(i1);
            }
        }
        if (i < end) {
            const int e0 = rps[0], ea = e0 & ~3, eb = e0 & ~1;
            const int b = rps[t], c = rps[t + 1];
            double acc = 0.0;
            int e = b;
            for (; e + kTmaBatch <= c; e += kTmaBatch) {
                double v[kTmaBatch];
#pragma unroll
                for (int q = 0; q < kTmaBatch; ++q) v[q] = src(cis[e + q - ea]);
#pragma unroll
                for (int q = 0; q < kTmaBatch; ++q)
                    acc = __dadd_rn(acc, Unit ? v[q] : __dmul_rn(avs[e + q - eb], v[q]));
            }
            {
                double v[kTmaBatch];
#pragma unroll
                for (int q = 0; q < kTmaBatch; ++q) v[q] = e + q < c ? src(cis[e + q - ea]) : 0.0;
#pragma unroll
                for (int q = 0; q < kTmaBatch; ++q)
                    if (e + q < c) acc = __dadd_rn(acc, Unit ? v[q] : __dmul_rn(avs[e + q - eb], v[q]));
            }
            epi.row(i, acc, src);
        }
    }
    if constexpr (Epi::K > 0) {
        double v[Epi::K];
        epi.vals(v);
        grid_reduce_finish<Epi::K, R>(v, epi.red.partials, epi.red.ticket, [&](const double (&tt)[Epi::K]) {
            if (!xpublish(epi.red, tt)) epi.fin(tt);
        });
    }
}

}  // namespace uaamg
