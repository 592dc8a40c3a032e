// launch.cuh -- host-side dispatch of the solve functors: run_stream (CSR
// row operations: TMA tiles on large levels, warp groups otherwise) and run_map (elementwise + reductions), plus the
// cross-rank reduction finish of the sharded solve (shard.cu).
#pragma once
#include "csr_group.cuh"
#include "csr_ell.cuh"
#include "csr_tma.cuh"

namespace uaamg {

// ============================================================ map-reduce
template <class Body>
__global__ void __launch_bounds__(kThreads) k_map(int n, Body body_p) {
    pdl_wait();
    pdl_trigger();
    Body body = body_p;
    if (!body.gate()) {
        if (blockIdx.x == 0 && threadIdx.x == 0) body.off();
        return;
    }
    body.init();
    double v[Body::K > 0 ? Body::K : 1] = {};
    for (int i = blockIdx.x * kThreads + threadIdx.x; i < n; i += gridDim.x * kThreads) body.item(i, v);
    if constexpr (Body::K > 0) {
        grid_reduce_finish<Body::K>(v, body.red.partials, body.red.ticket, [&](const double (&t)[Body::K]) {
            if (!xpublish(body.red, t)) body.fin(t);
        });
    }
}

// elementwise maps are latency-bound per thread (3-5 independent loads per
// item): up to 8 resident CTAs per SM, ~2 items per thread on large levels
inline int map_grid(int n) {
    int g = cdiv(n, kThreads * 2);
    return g < 1 ? 1 : (g > 8 * kNumSMs ? 8 * kNumSMs : g);
}

template <class Body>
void run_map(int n, const Body& body, Exec ex) {
    UA_LAUNCH_PDL((k_map<Body>), map_grid(n), kThreads, 0, ex.s, n, body);
}



template <class Body>
void run_map(int n, const Body& body, Exec ex);

// TMA-pipelined persistent tiles of R rows (occupancy cached per device).
// RowPar: one thread per row folding straight from the staged tile
// (k_csr_tma_rows, short regular rows); else the warp-cooperative gather.
template <class Src, class Epi, bool Unit, int R, bool RowPar = false, int S = kTmaStages>
inline void launch_tma(const Csr& A, const Groups& G, const Src& src, const Epi& epi, Exec ex) {
    static int occ_dev[kMaxDevices], smem_set_dev[kMaxDevices];
    static size_t occ_smem_dev[kMaxDevices];
    static bool init_dev[kMaxDevices];
    const int dev = cur_dev();
    if (!init_dev[dev]) {
        occ_dev[dev] = -1;
        smem_set_dev[dev] = 0;
        occ_smem_dev[dev] = 0;
        init_dev[dev] = true;
    }
    int& occ = occ_dev[dev];
    int& smem_set = smem_set_dev[dev];
    size_t& occ_smem = occ_smem_dev[dev];
    constexpr int threads = RowPar ? R : kTmaThreads;
    const size_t smem = tma_smem_bytes(G.tma_cap, R, S);
    auto kfn = [] {
        if constexpr (RowPar) return k_csr_tma_rows<Src, Epi, Unit, R, S>;
        else return k_csr_tma<Src, Epi, Unit, R, S>;
    }();
    if ((int)smem > smem_set) {
        UA_CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set = (int)smem;
        occ = -1;
    }
    if (occ < 0 || occ_smem != smem) {
        UA_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, threads, smem));
        occ_smem = smem;
    }
    const int ntiles = cdiv(G.n, R);
    const int grid = std::max(1, std::min(ntiles, kNumSMs * std::max(occ, 1)));
    // matrix streams larger than half the L2 are loaded evict-first
    static const bool no_hint = getenv("UAAMG_NO_L2HINT") != nullptr;  // A/B diagnostics
    const int hint = !no_hint && 12.0 * (double)G.tma_cap * ntiles > kStreamHintBytes;
    UA_LAUNCH_PDL(kfn, grid, threads, smem, ex.s, A, G.base, G.base + G.n, ntiles, G.tma_cap, src, epi, hint);
}

// sliced-ELL rows: 4 CTAs of kEllWarps slices per SM (tools/l0_sweep.cu: 0.94
// of the measured peak for 27-point 256^3 at 4/SM, 0.89 at 8/SM)
template <class Src, class Epi, bool Unit>
inline void launch_ell(const Csr& A, const Groups& G, const Src& src, const Epi& epi, Exec ex) {
    Ell E;
    E.off = G.ell_off;
    E.col = G.ell_col;
    E.val = G.ell_val;
    const int grid = std::max(1, std::min(cdiv(cdiv(G.n, 32), kEllWarps), 4 * kNumSMs));
    UA_LAUNCH_PDL((k_ell<Src, Epi, Unit>), grid, 32 * kEllWarps, 0, ex.s, A, G.base, G.n, E, src, epi);
}

template <class Src, class Epi, bool Unit>
inline void run_stream(const Csr& A, const Groups& G, const Src& src, const Epi& epi, Exec ex) {
    // an empty range still launches when it must publish a (zero) reduction
    if (G.units() == 0) {
        if constexpr (Epi::K == 0) return;
        else if (epi.red.xslot == nullptr) return;
    }
    if (G.ell_off) {
        launch_ell<Src, Epi, Unit>(A, G, src, epi, ex);
        return;
    }
    if (G.tma_cap > 0 && G.np == 0) {
        // large level: TMA-pipelined persistent tiles (64-row tiles when
        // 128 rows exceed the stage: dense stencils)
        if (G.tma_rowpar) launch_tma<Src, Epi, Unit, kTmaRowParRows, true, 2>(A, G, src, epi, ex);
        else if (G.tma_rows == 64) launch_tma<Src, Epi, Unit, 64>(A, G, src, epi, ex);
        else launch_tma<Src, Epi, Unit, kTmaRows>(A, G, src, epi, ex);
        return;
    }
    const int grid = std::min(cdiv(G.units(), kGrpWarps), kNumSMs * kGrpCtasPerSM);
    UA_LAUNCH_PDL((k_csr_group<Src, Epi, Unit>), grid, 32 * kGrpWarps, 0, ex.s, A, G, src, epi);
}


// Sharded solve: the per-rank totals of a reduction were published into
// every rank's slot array (xpublish); this folds them in rank order -- the
// same bits on every rank -- and runs the op's fin() once.
template <class T>
__global__ void k_xfin(T obj, const double* slots, int P) {
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (!obj.gate()) return;  // the op was gated off: it published nothing and ran off()
    double t[T::K];
#pragma unroll
    for (int k = 0; k < T::K; ++k) {
        double s = 0.0;
        for (int q = 0; q < P; ++q) s += __ldcg(slots + k * P + q);
        t[k] = s;
    }
    obj.fin(t);
}

template <class T>
void run_xfin(const T& obj, const double* slots, int P, cudaStream_t s) {
    UA_LAUNCH_PDL((k_xfin<T>), 1, 32, 0, s, obj, slots, P);
}

}  // namespace uaamg
