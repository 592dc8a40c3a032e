// engine.cu -- persistent coarse-level K-cycle engine (see engine.h).
//
// Interprets a recorded op list (ops.cuh) inside one cooperative launch of
// thread-block clusters, one CTA per SM.  Each op is a phase:
//   * CSR ops (residual, restriction, fused prolongation + sweep, direction
//     SpMV) run the warp work units of csr_group.cuh (32-row groups folded
//     in reference order; long-row pieces combined by ticket), the warps of
//     the participating CTAs striding over the units;
//   * map ops (vector updates, norms, projections) stride over items;
//   * reductions write one partial per CTA; after the barrier every CTA
//     folds the partials in the same order and runs the op's fin() on its
//     own thread 0, so every CTA holds bit-identical flags/scalars (written
//     identically to the same state words) and takes the same gate
//     decisions -- no broadcast phase;
//   * a gated-off op runs its off() in every participating CTA and costs no
//     barrier.
// Two tiers: "small" ops (few rows: the deepest, most-visited levels) run
// on the first cluster only and synchronise with the hardware cluster
// barrier (~0.2 us); the other clusters skip them.  "Big" ops use every CTA
// and a grid barrier; the first big op after a run of small ops starts with
// a grid barrier so everyone sees the small ops' results.
// Both barriers invalidate the SM's L1 on acquire (CCTL.IVALL), so plain
// loads after them see other SMs' writes of the previous phase.  The op list
// is staged through shared memory in chunks.
#include "csr_group.cuh"
#include "engine.h"

namespace uaamg {

namespace {

constexpr int kOpChunk = 16;  // ops staged in shared memory at a time

struct Ctx {
    int nctas;          // CTAs taking part in the current op
    bool small;         // current op runs on cluster 0 with cluster barriers
    int slot[2];        // partials slot of the next reduction, per tier
    double* sm;         // block_sum scratch, kEngThreads / 32 + 1
    double* tot;        // reduction broadcast, kEngK
    double* partials;   // per tier: 2 slots x kEngK x grid
    unsigned* bar;
    double* win;        // per-warp product windows, kGrpRound each
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Generation barrier over the whole (co-resident) grid.
__device__ __noinline__ void grid_sync(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            const long long t0 = clock64();
            while (*gen == g) {
                if (clock64() - t0 > (1ll << 34)) __trap();  // several seconds: a lost CTA, fail loudly
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// Hardware barrier over the CTAs of this cluster (all threads).
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void phase_sync(const Ctx& c) {
    if (c.small) cluster_sync();
    else grid_sync(c.bar);
}

__device__ __forceinline__ int gtid() { return blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int gthreads(const Ctx& c) { return c.nctas * blockDim.x; }

template <int K>
__device__ void red_finish(Ctx& c, const double (&v)[K], double (&t)[K]) {
    const int G = c.nctas;
    const int tier = c.small ? 1 : 0;
    double* P = c.partials + (size_t)tier * 2 * kEngK * gridDim.x + (size_t)c.slot[tier] * kEngK * G;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double s = block_sum<kEngThreads>(v[k], c.sm);
        if (threadIdx.x == 0) P[k * G + blockIdx.x] = s;
    }
    phase_sync(c);
    if (threadIdx.x < 32) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int b = threadIdx.x; b < G; b += 32) s += P[k * G + b];
            s = warp_sum(s);
            if (threadIdx.x == 0) c.tot[k] = s;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = c.tot[k];
    __syncthreads();
    c.slot[tier] ^= 1;  // the next reduction may run while slow CTAs still read this slot
}

// ------------------------------------------------------------------ CSR units
// warps of the participating CTAs stride over the operand's work units
template <bool Unit, class Src, class Epi>
__device__ __forceinline__ void csr_units(Ctx& c, const Csr& A, const Groups& G, const Src& src, Epi& epi) {
    const int nu = G.units();
    const int w = threadIdx.x >> 5;
    for (int u = gtid() >> 5; u < nu; u += gthreads(c) >> 5) grp_unit<Unit>(A, G, u, src, epi, c.win + w * kGrpRound);
}

// ------------------------------------------------------------------ op runners
template <class Src, class Epi, bool Unit>
__device__ __noinline__ void run_csr(Ctx& c, const Op* op) {
    CsrPay<Src, Epi> p = *reinterpret_cast<const CsrPay<Src, Epi>*>(op->pay);
    if (!p.epi.gate()) {
        if (threadIdx.x == 0) p.epi.off();
        __syncthreads();
        return;
    }
    p.src.init();
    const Csr A = op->A;
    const Groups G = op->G;
    csr_units<Unit>(c, A, G, p.src, p.epi);
    if constexpr (Epi::K > 0) {
        double v[Epi::K], t[Epi::K];
        p.epi.vals(v);
        red_finish<Epi::K>(c, v, t);
        if (threadIdx.x == 0) p.epi.fin(t);
        __syncthreads();
    } else {
        phase_sync(c);
    }
}

template <class Body>
__device__ __noinline__ void run_map(Ctx& c, const Op* op) {
    Body body = *reinterpret_cast<const Body*>(op->pay);
    if (!body.gate()) {
        if (threadIdx.x == 0) body.off();
        __syncthreads();
        return;
    }
    body.init();
    const int n = op->n;
    double v[Body::K > 0 ? Body::K : 1] = {};
    for (int i = gtid(); i < n; i += gthreads(c)) body.item(i, v);
    if constexpr (Body::K > 0) {
        double t[Body::K];
        red_finish<Body::K>(c, v, t);
        if (threadIdx.x == 0) body.fin(t);
        __syncthreads();
    } else {
        phase_sync(c);
    }
}

// dense coarsest solve, one warp per row (same arithmetic as k_dense_solve)
__device__ __noinline__ void run_dense(Ctx& c, const Op* op) {
    const DenseArgs d = *reinterpret_cast<const DenseArgs*>(op->pay);
    if (d.g && !*d.g) return;
    const int lane = threadIdx.x & 31;
    for (int row = gtid() >> 5; row < d.n; row += gthreads(c) >> 5) {
        double acc = 0.0;
        for (int j = lane; j < d.n; j += 32) acc += d.M[(size_t)row * d.n + j] * d.b[j];
        acc = warp_sum(acc);
        if (lane == 0) d.x[row] = acc;
    }
    phase_sync(c);
}

__global__ void __launch_bounds__(kEngThreads, 1) k_engine(EngineArgs a) {
    __shared__ double sm[kEngThreads / 32 + 1];
    __shared__ double tot[kEngK];
    __shared__ __align__(16) unsigned char chunk_raw[kOpChunk * sizeof(Op)];
    Op* chunk = reinterpret_cast<Op*>(chunk_raw);
    __shared__ double win[(kEngThreads / 32) * kGrpRound];
    if (a.gate && *(volatile const int*)a.gate == 0) return;
    Ctx c{(int)gridDim.x, false, {0, 0}, sm, tot, a.partials, a.bar, win};
    const bool prof = a.prof && blockIdx.x == 0 && threadIdx.x == 0;
    const bool in_small = blockIdx.x < (unsigned)a.csize;
    for (int k0 = 0; k0 < a.nops; k0 += kOpChunk) {
        // stage the next chunk of the op list (16-byte words)
        const int m = min(kOpChunk, a.nops - k0);
        __syncthreads();
        {
            const int4* src = reinterpret_cast<const int4*>(a.ops + k0);
            int4* dst = reinterpret_cast<int4*>(chunk);
            const int words = m * (int)(sizeof(Op) / sizeof(int4));
            for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = __ldg(src + w);
        }
        __syncthreads();
        for (int j = 0; j < m; ++j) {
            const Op* op = chunk + j;
            if (prof) a.prof[k0 + j] = globaltimer();
            if (op->small) {
                if (!in_small) continue;
                c.small = true;
                c.nctas = a.csize;
            } else {
                c.small = false;
                c.nctas = gridDim.x;
                if (op->sync_before) grid_sync(a.bar);
            }
            switch (op->kind) {
#define UA_CASE_CSR(kd, S, E, U) \
    case kd: run_csr<S, E, U>(c, op); break;
#define UA_CASE_MAP(kd, B) \
    case kd: run_map<B>(c, op); break;
                UA_ENGINE_CSR_OPS(UA_CASE_CSR)
                UA_ENGINE_MAP_OPS(UA_CASE_MAP)
#undef UA_CASE_CSR
#undef UA_CASE_MAP
                case kOpDense: run_dense(c, op); break;
                default: __trap();
            }
        }
    }
    if (prof) a.prof[a.nops] = globaltimer();
}

__global__ void __launch_bounds__(kEngThreads, 1) k_bar_bench(unsigned* bar, int variant, int iters) {
    for (int k = 0; k < iters; ++k) {
        if (variant == 0) grid_sync(bar);
        else cluster_sync();
    }
}

struct EngineConfig {
    int grid = 0, csize = 0;
};

// Largest cluster size (16, else 8, ...) whose clusters fit; grid = all
// co-resident clusters (one CTA per SM).
const EngineConfig& engine_config() {
    static EngineConfig cfg;
    if (cfg.grid) return cfg;
    int dev = 0, sms = 0;
    UA_CK(cudaGetDevice(&dev));
    UA_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    UA_CK(cudaFuncSetAttribute(k_engine, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    UA_CK(cudaFuncSetAttribute(k_bar_bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int cs : {16, 8, 4, 2, 1}) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((sms / cs) * cs);
        lc.blockDim = dim3(kEngThreads);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, k_engine, &lc) != cudaSuccess || nclusters < 1) {
            (void)cudaGetLastError();
            continue;
        }
        cfg.csize = cs;
        cfg.grid = std::min(nclusters, sms / cs) * cs;
        break;
    }
    if (!cfg.grid) throw Error(UAAMG_ECUDA, "coarse engine kernel cannot be resident");
    return cfg;
}

}  // namespace

int engine_grid() { return engine_config().grid; }
int engine_cluster() { return engine_config().csize; }

void launch_engine(const EngineArgs& a_in, cudaStream_t s) {
    const EngineConfig& ec = engine_config();
    EngineArgs a = a_in;
    a.csize = ec.csize;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ec.grid);
    cfg.blockDim = dim3(kEngThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = ec.csize;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    UA_CK(cudaLaunchKernelEx(&cfg, k_engine, a));
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace uaamg

// diagnostics: seconds per barrier on the engine's grid (variant 0: grid
// barrier, 1: cluster barrier)
extern "C" int uaamg_dev_barrier_bench(int variant, int iters, double* seconds) {
    using namespace uaamg;
    try {
        cudaStream_t s = 0;
        const int grid = engine_grid(), cs = engine_cluster();
        DBuf<unsigned> bar(2, s);
        UA_CK(cudaMemsetAsync(bar.p, 0, sizeof(unsigned) * 2, s));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kEngThreads);
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = cs;
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        cudaEvent_t e0, e1;
        UA_CK(cudaEventCreate(&e0));
        UA_CK(cudaEventCreate(&e1));
        UA_CK(cudaLaunchKernelEx(&cfg, k_bar_bench, bar.p, variant, 1));
        UA_CK(cudaEventRecord(e0, s));
        UA_CK(cudaLaunchKernelEx(&cfg, k_bar_bench, bar.p, variant, iters));
        UA_CK(cudaEventRecord(e1, s));
        UA_CK(cudaEventSynchronize(e1));
        float ms = 0;
        UA_CK(cudaEventElapsedTime(&ms, e0, e1));
        *seconds = ms * 1e-3 / iters;
        fprintf(stderr, "engine grid %d cluster %d\n", grid, cs);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return 0;
    } catch (const std::exception& e) {
        fprintf(stderr, "%s\n", e.what());
        return UAAMG_ECUDA;
    }
}
