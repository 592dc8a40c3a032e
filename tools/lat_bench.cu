// Latency microbenchmarks of the primitives on the coarse-level critical
// path (one thread, clock64): dependent L2 loads, __threadfence (fence.sc),
// fence.acq_rel, returning atomics, release atomics, acquire loads, and a
// store -> fence -> atomic ticket sequence.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o lat_bench lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__global__ void k_lat(int* chain, unsigned* cnt, double* buf, long long* out, int iters) {
    if (threadIdx.x != 0) return;
    long long t0, t1;
    int j = 0;
    // 0: dependent L2 loads (ld.cg)
    t0 = clock64();
    for (int k = 0; k < iters; ++k) j = __ldcg(chain + j);
    t1 = clock64();
    out[0] = (t1 - t0) / iters;
    // 1: __threadfence alone (after a store)
    t0 = clock64();
    for (int k = 0; k < iters; ++k) {
        buf[k & 63] = (double)k;
        __threadfence();
    }
    t1 = clock64();
    out[1] = (t1 - t0) / iters;
    // 2: fence.acq_rel alone (after a store)
    t0 = clock64();
    for (int k = 0; k < iters; ++k) {
        buf[k & 63] = (double)k;
        fence_acq_rel();
    }
    t1 = clock64();
    out[2] = (t1 - t0) / iters;
    // 3: returning atomicAdd (relaxed), dependent
    unsigned s = 0;
    t0 = clock64();
    for (int k = 0; k < iters; ++k) s += atomicAdd(cnt + (s & 1), 1u);
    t1 = clock64();
    out[3] = (t1 - t0) / iters;
    // 4: store + __threadfence + atomicAdd (the ticket pattern)
    t0 = clock64();
    for (int k = 0; k < iters; ++k) {
        buf[k & 63] = (double)s;
        __threadfence();
        s += atomicAdd(cnt, 1u);
    }
    t1 = clock64();
    out[4] = (t1 - t0) / iters;
    // 5: store + atom.add.release
    t0 = clock64();
    for (int k = 0; k < iters; ++k) {
        buf[k & 63] = (double)s;
        s += atom_add_release(cnt, 1u);
    }
    t1 = clock64();
    out[5] = (t1 - t0) / iters;
    // 6: store + atom.add.acq_rel
    t0 = clock64();
    for (int k = 0; k < iters; ++k) {
        buf[k & 63] = (double)s;
        s += atom_add_acqrel(cnt, 1u);
    }
    t1 = clock64();
    out[6] = (t1 - t0) / iters;
    // 7: dependent ld.acquire
    t0 = clock64();
    for (int k = 0; k < iters; ++k) s += ld_acquire(cnt + (s & 1));
    t1 = clock64();
    out[7] = (t1 - t0) / iters;
    // 8: dependent plain loads after fence (L1 invalidated each time)
    t0 = clock64();
    for (int k = 0; k < iters; ++k) {
        __threadfence();
        j = chain[j];
    }
    t1 = clock64();
    out[8] = (t1 - t0) / iters;
    // 10: dependent DADD chain; 11: dependent DMUL chain; 12: dependent FADD chain
    double d = (double)j * 1e-3 + 1.0;
    t0 = clock64();
    for (int k = 0; k < iters; ++k) d = __dadd_rn(d, 1e-9);
    t1 = clock64();
    out[10] = (t1 - t0) * 100 / iters;
    t0 = clock64();
    for (int k = 0; k < iters; ++k) d = __dmul_rn(d, 1.0000001);
    t1 = clock64();
    out[11] = (t1 - t0) * 100 / iters;
    float f = (float)d;
    t0 = clock64();
    for (int k = 0; k < iters; ++k) f = __fadd_rn(f, 1e-7f);
    t1 = clock64();
    out[12] = (t1 - t0) * 100 / iters;
    out[9] = j + s + (long long)d + (long long)f;
}

// end-to-end chain of tiny dependent kernels (PDL or not) in a graph: the
// per-kernel floor.  mode 0: plain; 1: PDL wait/trigger; 2: + grid reduction ticket
__global__ void k_tiny(double* v, unsigned* ticket, double* part, int mode) {
    if (mode >= 1) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (mode >= 1) asm volatile("griddepcontrol.launch_dependents;" :::);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double x = v[i] * 1.0000001;
    v[i] = x;
    if (mode == 2) {
        __shared__ bool last;
        if (threadIdx.x == 0) {
            part[blockIdx.x] = x;
            __threadfence();
            last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last && threadIdx.x == 0) {
            __threadfence();
            double s = 0;
            for (int b = 0; b < gridDim.x; ++b) s += __ldcg(part + b);
            v[0] = s * 1e-30;
            *ticket = 0;
        }
    }
    if (mode == 4) {  // ticket + warp-parallel fold (the product's pattern)
        __shared__ bool last;
        if (threadIdx.x == 0) {
            part[blockIdx.x] = x;
            __threadfence();
            last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last && threadIdx.x < 32) {
            __threadfence();
            double s = 0;
            for (int b = threadIdx.x; b < gridDim.x; b += 32) s += __ldcg(part + b);
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (threadIdx.x == 0) {
                v[0] = s * 1e-30;
                *ticket = 0;
            }
        }
    }
    if (mode == 5) {  // deferred: fold the predecessor's partials (double-buffered), write own
        const int par = (int)(v[1] != 0.0);  // stand-in for a parity known at capture
        if (threadIdx.x < 32) {
            double s = 0;
            for (int b = threadIdx.x; b < gridDim.x; b += 32) s += part[2048 * par + b];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (threadIdx.x == 0) part[2048 * (par ^ 1) + blockIdx.x] = x + s * 1e-30;
        }
    }
    if (mode == 3) {  // release/acquire ticket
        __shared__ bool last;
        if (threadIdx.x == 0) {
            part[blockIdx.x] = x;
            last = atom_add_acqrel(ticket, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last && threadIdx.x == 0) {
            double s = 0;
            for (int b = 0; b < gridDim.x; ++b) s += __ldcg(part + b);
            v[0] = s * 1e-30;
            *ticket = 0;
        }
    }
}

int main() {
    const int N = 1 << 20;
    int* chain;
    unsigned* cnt;
    double* buf;
    long long* out;
    cudaMalloc(&chain, N * sizeof(int));
    cudaMalloc(&cnt, 64);
    cudaMalloc(&buf, 1 << 20);
    cudaMalloc(&out, 16 * sizeof(long long));
    int* h = new int[N];
    for (int k = 0; k < N; ++k) h[k] = (int)((k * 2654435761u + 12345u) % N) & ~31;  // 128B-separated
    cudaMemcpy(chain, h, N * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemset(cnt, 0, 64);
    k_lat<<<1, 32>>>(chain, cnt, buf, out, 64);
    k_lat<<<1, 32>>>(chain, cnt, buf, out, 2000);
    cudaDeviceSynchronize();
    long long r[16];
    cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
    const char* nm[] = {"dep ld.cg (L2)", "st+__threadfence", "st+fence.acq_rel", "atomicAdd ret", "st+fence+atomic",
                        "st+atom.release", "st+atom.acq_rel", "ld.acquire dep", "fence+dep ld"};
    for (int k = 0; k < 9; ++k) printf("%-20s %6lld cycles\n", nm[k], r[k]);
    printf("dadd chain %.2f  dmul chain %.2f  fadd chain %.2f cycles/op\n", r[10] / 100.0, r[11] / 100.0, r[12] / 100.0);
    // kernel chains
    cudaStream_t s;
    cudaStreamCreate(&s);
    double* v;
    double* part;
    cudaMalloc(&v, 148 * 1024 * 8);
    cudaMalloc(&part, 4096 * 8);
    cudaMemset(v, 0, 148 * 1024 * 8);
    for (int mode = 0; mode < 6; ++mode) {
        for (int grid : {1, 38, 148}) {
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int k = 0; k < 200; ++k) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = mode >= 1 ? 1 : 0;
                cudaLaunchKernelEx(&cfg, k_tiny, v, cnt + 8, part, mode);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, s);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, s);
            for (int rep = 0; rep < 5; ++rep) cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("chain mode %d grid %3d: %.2f us/kernel\n", mode, grid, ms * 1e3 / 1000);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
