// common.cuh -- shared types and device helpers for the B200 UA-AMG library.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "uaamg_b200.h"

namespace uaamg {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define UA_CK(x)                                                                                     \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess)                                                                       \
            throw ::uaamg::Error(UAAMG_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + " (" \
                                                  __FILE__ ":" + std::to_string(__LINE__) + ")");     \
    } while (0)

extern std::atomic<uint64_t> g_launches;

// Every library kernel launch goes through this (launch accounting + error check).
#define UA_LAUNCH(kernel, grid, block, smem, stream, ...)                        \
    do {                                                                         \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);              \
        ::uaamg::g_launches.fetch_add(1, std::memory_order_relaxed);             \
        UA_CK(cudaGetLastError());                                               \
    } while (0)

// Programmatic dependent launch (PDL): solve kernels are launched with
// programmatic stream serialization, so a kernel's CTAs may start while its
// predecessor drains.  Every such kernel calls pdl_wait() before touching
// memory a predecessor wrote (griddepcontrol.wait returns once all
// prerequisite grids completed and their writes are visible; a no-op when
// launched without the attribute), and pdl_trigger() right after it to let
// its own successor begin launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#define UA_LAUNCH_PDL(kernel, grid, block, smem, strm, ...)                                   \
    do {                                                                                        \
        cudaLaunchConfig_t cfg_ = {};                                                           \
        cfg_.gridDim = dim3(grid);                                                              \
        cfg_.blockDim = dim3(block);                                                            \
        cfg_.dynamicSmemBytes = (smem);                                                         \
        cfg_.stream = (strm);                                                                   \
        cudaLaunchAttribute at_[1];                                                             \
        at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                         \
        at_[0].val.programmaticStreamSerializationAllowed = 1;                                  \
        cfg_.attrs = at_;                                                                       \
        cfg_.numAttrs = 1;                                                                      \
        UA_CK(cudaLaunchKernelEx(&cfg_, kernel, __VA_ARGS__));                                  \
        ::uaamg::g_launches.fetch_add(1, std::memory_order_relaxed);                            \
    } while (0)

// Generation barrier over a co-resident (cooperatively launched) grid:
// bar[0] arrivals (back to 0 after each barrier), bar[1] generation.
__device__ __noinline__ inline void coop_grid_sync(unsigned* bar) {
    // bar: a 64-bit arrival counter, zeroed once and only ever used by
    // launches of one grid size, so it is a multiple of gridDim.x at every
    // launch start.  Arrive with release, spin with acquire until this
    // epoch's gridDim.x arrivals are in (relaxed polling: an acquire per poll
    // would invalidate the SM's L1 under its co-resident CTAs), then one
    // acquire fence (which invalidates L1 for the CTA's later plain loads).
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long* c = reinterpret_cast<unsigned long long*>(bar);
        unsigned long long old, v;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(c) : "memory");
        const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
        const long long t0 = clock64();
        while (true) {
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(c) : "memory");
            if (v >= target) break;
            if (clock64() - t0 > (1ll << 34)) __trap();  // a lost CTA: fail loudly
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire once, after the relaxed spin
    }
    __syncthreads();
}

// ---------------------------------------------------------------- device memory
// Stream-ordered allocation from the device's default memory pool.
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = 0;
    bool view = false;  // non-owning (memory lives in an arena)
    DBuf() = default;
    DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), view(o.view) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; s = o.s; view = o.view; o.p = nullptr; o.n = 0; }
        return *this;
    }
    // re-point at arena memory (the previous allocation is freed)
    void adopt_view(T* ptr, size_t count) {
        release();
        p = ptr;
        n = count;
        view = true;
    }
    void alloc(size_t count, cudaStream_t st) {
        release();
        s = st;
        n = count;
        // 64 bytes of tail slack: bulk (TMA) copies round slices up to 16-byte
        // granules and may read past the last element
        if (count) UA_CK(cudaMallocAsync((void**)&p, count * sizeof(T) + 64, st));
    }
    void release() {
        if (p && !view) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
        view = false;
    }
    ~DBuf() { release(); }
    T* get() const { return p; }
};

// ---------------------------------------------------------------- CSR views
struct Csr {
    int n = 0;            // rows (square)
    int nnz = 0;
    const int* rp = nullptr;
    const int* ci = nullptr;
    const double* av = nullptr;
};

// ---------------------------------------------------------------- constants
constexpr int kThreads = 256;           // staged kernels: threads per block
constexpr int kNumSMs = 148;            // B200
constexpr int kLongRow = 64;            // setup kernels: rows longer than this get a warp

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// Process-wide caches of device-dependent facts (occupancy, function
// attributes, pool state, scratch) are indexed by the current device.
constexpr int kMaxDevices = 16;
inline int cur_dev() {
    int d = 0;
    UA_CK(cudaGetDevice(&d));
    if (d < 0 || d >= kMaxDevices) throw Error(UAAMG_EUNSUPPORTED, "device ordinal beyond kMaxDevices");
    return d;
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide maximum of T (int / unsigned long long / double), valid in
// thread 0 -- lets a kernel issue ONE atomicMax per block instead of one per
// thread (same-address atomics serialise at the L2).  All threads call it.
template <class T>
__device__ __forceinline__ T block_max(T v) {
    __shared__ T wm[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const T u = __shfl_xor_sync(0xffffffffu, v, o);
        v = u > v ? u : v;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : wm[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const T u = __shfl_xor_sync(0xffffffffu, v, o);
            v = u > v ? u : v;
        }
    }
    return v;
}

// Deterministic block sum (fixed shuffle tree + fixed smem order).  All
// threads of the block must call it; result valid in every thread.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sm /* >= NT/32 + 1 */) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sm[w] = v;
    __syncthreads();
    double t = 0.0;
    if (w == 0) {
        t = (lane < NT / 32) ? sm[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) sm[NT / 32] = t;
    }
    __syncthreads();
    return sm[NT / 32];
}

// Deterministic grid-wide reduction of K doubles per thread: block sums go
// to partials[k*nb + block]; the last block to arrive (atomic ticket) sums
// the partials in block order and calls fin(tot) on thread 0, then rearms
// the ticket.  Must be called by all threads of every block of the launch.
// lval/nlong: per-long-row values (stride 2) of a CSR operation whose long
// rows were finished by arrival-order-dependent warps, folded after the
// block partials in row order.
template <int K, int NT = kThreads, class F>
__device__ __forceinline__ void grid_reduce_finish(double (&v)[K], double* partials, unsigned* ticket, F&& fin,
                                                   const double* lval = nullptr, int nlong = 0) {
    __shared__ double sm[NT / 32 + 1];
    __shared__ bool last;
    double tot[K];
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] = block_sum<NT>(v[k], sm);
    const int nb = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) partials[k * nb + blockIdx.x] = tot[k];
        // one acq_rel ticket: releases this block's partials, and the last
        // arriver acquires every other block's (no separate fences)
        unsigned prev;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ticket) : "memory");
        last = prev == (unsigned)(nb - 1);
    }
    __syncthreads();
    if (!last) return;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (int b = threadIdx.x; b < nb; b += NT) s += __ldcg(partials + k * nb + b);
        for (int r = threadIdx.x; r < nlong; r += NT) s += __ldcg(lval + 2 * r + k);
        tot[k] = block_sum<NT>(s, sm);
    }
    if (threadIdx.x == 0) {
        fin(tot);
        *ticket = 0u;  // (re-read only by a later launch)
    }
}

// pinned-ring host <-> device transfers (hostio.cu): element size se -> de
// (equal: copy; 8 -> 4: int64 -> int32 narrowing while staging)
void staged_h2d(void* dst, const void* src, size_t count, int se, int de, cudaStream_t s);
void staged_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s);

}  // namespace uaamg
