// Distributed-shared-memory microbenchmarks for the tail kernel's cluster
// (16 CTAs x 512 threads): dependent remote-load latency, independent-load
// throughput, cluster barrier cost, mapa cost.  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o dsm_bench dsm_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned cta_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ double ld_dsm(unsigned a) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_dsm(long long* out, int iters, int cs) {
    extern __shared__ double buf[];  // 4096 doubles
    const unsigned rank = cta_rank();
    for (int i = threadIdx.x; i < 4096; i += 512) buf[i] = (double)((i * 7 + rank) & 4095);
    csync();
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf);
    long long t0 = clock64();
    double acc = 0.0;
    if (MODE == 0) {  // dependent remote loads, one thread per CTA
        if (threadIdx.x == 0) {
            int j = 0;
            for (int k = 0; k < iters; ++k) {
                const double v = ld_dsm(mapa(base + 8 * j, (rank + 1 + k) % cs));
                j = (int)v;
                acc += v;
            }
        }
    } else if (MODE == 1) {  // all threads: 8 independent remote loads per step
        int j = threadIdx.x;
        for (int k = 0; k < iters; ++k) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = ld_dsm(mapa(base + 8 * ((j + 97 * q) & 4095), (rank + q + 1) % cs));
#pragma unroll
            for (int q = 0; q < 8; ++q) acc += v[q];
            j = (j + (int)v[0]) & 4095;
        }
    } else if (MODE == 2) {  // all threads: 8 independent LOCAL loads via generic smem
        int j = threadIdx.x;
        for (int k = 0; k < iters; ++k) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = buf[(j + 97 * q) & 4095];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc += v[q];
            j = (j + (int)v[0]) & 4095;
        }
    } else if (MODE == 3) {  // cluster barriers
        for (int k = 0; k < iters; ++k) csync();
    } else if (MODE == 4) {  // all threads: 8 independent remote loads, own rank via mapa
        int j = threadIdx.x;
        for (int k = 0; k < iters; ++k) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = ld_dsm(mapa(base + 8 * ((j + 97 * q) & 4095), rank));
#pragma unroll
            for (int q = 0; q < 8; ++q) acc += v[q];
            j = (j + (int)v[0]) & 4095;
        }
    } else if (MODE == 6) {  // all threads: 8 remote loads through generic pointers (map_shared_rank)
        int j = threadIdx.x;
        for (int k = 0; k < iters; ++k) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                v[q] = *static_cast<const double*>(__cluster_map_shared_rank(buf + ((j + 97 * q) & 4095), (rank + q + 1) % cs));
#pragma unroll
            for (int q = 0; q < 8; ++q) acc += v[q];
            j = (j + (int)v[0]) & 4095;
        }
    } else if (MODE == 7) {  // generic pointers to the OWN CTA
        int j = threadIdx.x;
        for (int k = 0; k < iters; ++k) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                v[q] = *static_cast<const double*>(__cluster_map_shared_rank(buf + ((j + 97 * q) & 4095), rank));
#pragma unroll
            for (int q = 0; q < 8; ++q) acc += v[q];
            j = (j + (int)v[0]) & 4095;
        }
    } else if (MODE == 8) {  // one thread: dependent generic remote loads
        if (threadIdx.x == 0) {
            int j = 0;
            for (int k = 0; k < iters; ++k) {
                const double v = *static_cast<const double*>(__cluster_map_shared_rank(buf + j, (rank + 1 + k) % cs));
                j = (int)v;
                acc += v;
            }
        }
    } else if (MODE == 5) {  // one warp per CTA: 8 independent remote loads per lane
        if (threadIdx.x < 32) {
            int j = threadIdx.x;
            for (int k = 0; k < iters; ++k) {
                double v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    v[q] = ld_dsm(mapa(base + 8 * ((j + 97 * q) & 4095), (rank + q + 1) % cs));
#pragma unroll
                for (int q = 0; q < 8; ++q) acc += v[q];
                j = (j + (int)v[0]) & 4095;
            }
        }
    }
    long long t1 = clock64();
    csync();
    if (threadIdx.x == 0) out[rank] = (t1 - t0) / iters;
    if (acc == 12345.678) out[100] = 1;
}

int main() {
    long long* out;
    cudaMalloc(&out, 128 * sizeof(long long));
    const char* nm[] = {"dep remote ld (1 thr)", "8 remote ld x 512 thr", "8 local ld x 512 thr", "cluster barrier",
                        "8 self-mapa ld x 512", "8 remote ld x 1 warp", "8 generic remote x 512", "8 generic self x 512",
                        "dep generic remote (1 thr)"};
    for (int cs : {16, 8, 4}) {
        for (int mode = 0; mode < 9; ++mode) {
            void (*k)(long long*, int, int) = nullptr;
            switch (mode) {
                case 0: k = k_dsm<0>; break;
                case 1: k = k_dsm<1>; break;
                case 2: k = k_dsm<2>; break;
                case 3: k = k_dsm<3>; break;
                case 4: k = k_dsm<4>; break;
                case 5: k = k_dsm<5>; break;
                case 6: k = k_dsm<6>; break;
                case 7: k = k_dsm<7>; break;
                case 8: k = k_dsm<8>; break;
            }
            cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 8);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = 4096 * 8;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k, out, 1000, cs);
            cudaDeviceSynchronize();
            long long r[16];
            cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
            printf("cs %2d %-24s %6lld cycles/iter (cta0)  err %s\n", cs, nm[mode], r[0],
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
