// spmv_bench.cu -- level-0 SpMV microbenchmark (diagnostics, not product):
// 7-point 3D Laplacian n^3 built on the device; times the group kernel and
// the TMA kernel with a vector gather, the TMA kernel with no gather
// (constant source), and a plain copy of the matrix stream as the bandwidth
// reference.  Build: see tools/spmv_bench.sh
#include <cstdio>
#include <vector>

#include "../paper_1302_2547_b200/csrc/csr_group.cuh"
#include "../paper_1302_2547_b200/csrc/csr_tma.cuh"

using namespace uaamg;
namespace uaamg {
std::atomic<uint64_t> g_launches{0};
}

struct SrcConst {
    __device__ void init() {}
    __device__ void pre(int) const {}
    __device__ double operator()(int) const { return 1.0; }
};

__global__ void k_build(int n, int* rp, int* ci, double* av) {
    const int N = n * n * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const int x = i / (n * n), y = (i / n) % n, z = i % n;
        int cnt = 7 * i;  // fixed 7 slots per row (boundary rows padded with explicit zeros: timing only)
        rp[i] = cnt;
        const int nb[7] = {x > 0 ? i - n * n : -1, y > 0 ? i - n : -1, z > 0 ? i - 1 : -1, i,
                           z < n - 1 ? i + 1 : -1, y < n - 1 ? i + n : -1, x < n - 1 ? i + n * n : -1};
        for (int k = 0; k < 7; ++k) {
            ci[cnt + k] = nb[k] >= 0 ? nb[k] : i;
            av[cnt + k] = nb[k] == i ? 6.0 : (nb[k] >= 0 ? -1.0 : 0.0);
        }
        if (i == N - 1) rp[N] = 7 * N;
    }
}

__global__ void k_copy(const int4* a, int4* b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 128;
    const int N = n * n * n;
    const long long nnz = 7ll * N;
    int *rp, *ci;
    double *av, *x, *y;
    cudaMalloc(&rp, sizeof(int) * (N + 1) + 64);
    cudaMalloc(&ci, sizeof(int) * nnz + 64);
    cudaMalloc(&av, sizeof(double) * nnz + 64);
    cudaMalloc(&x, sizeof(double) * N + 64);
    cudaMalloc(&y, sizeof(double) * N + 64);
    k_build<<<1184, 256>>>(n, rp, ci, av);
    cudaMemset(x, 0, sizeof(double) * N);
    Csr A;
    A.n = N; A.nnz = (int)nnz; A.rp = rp; A.ci = ci; A.av = av;
    Groups G = exact_groups(N);
    const double bytes = 12.0 * nnz + 4.0 * (N + 1) + 16.0 * N;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    void* flush;
    cudaMalloc(&flush, 256 << 20);
    auto timeit = [&](const char* name, auto&& launch, double b) {
        float best = 1e9, sum = 0;
        const int reps = 20;
        for (int r = 0; r < reps + 2; ++r) {
            cudaMemsetAsync(flush, r, 256 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 2) { best = std::min(best, ms); sum += ms; }
        }
        printf("%-34s best %8.1f us  mean %8.1f us  %7.1f GB/s (best)\n", name, best * 1e3, sum / reps * 1e3,
               b / (best * 1e-3) / 1e9);
        cudaError_t err = cudaGetLastError();
        if (err) printf("  error %s\n", cudaGetErrorString(err));
    };
    EpiStore ep{};
    ep.y = y;
    timeit("group SrcVec", [&] {
        const int grid = std::min(cdiv(G.units(), kGrpWarps), kNumSMs * kGrpCtasPerSM);
        k_csr_group<SrcVec, EpiStore, false><<<grid, 32 * kGrpWarps>>>(A, G, SrcVec{x}, ep);
    }, bytes);
    for (int cap : {7 * kTmaRows}) {
        const size_t smem = tma_smem_bytes(cap);
        cudaFuncSetAttribute(k_csr_tma<SrcVec, EpiStore, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_csr_tma<SrcConst, EpiStore, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_csr_tma<SrcVec, EpiStore, false>, kTmaRows, smem);
        const int ntiles = cdiv(N, kTmaRows);
        printf("TMA smem %zu occ %d\n", smem, occ);
        for (int mult : {1, 2}) {
            const int grid = std::min(ntiles, kNumSMs * occ * mult);
            char nm[64];
            snprintf(nm, sizeof nm, "tma SrcVec grid x%d", mult);
            timeit(nm, [&] { k_csr_tma<SrcVec, EpiStore, false><<<grid, kTmaRows, smem>>>(A, ntiles, cap, SrcVec{x}, ep); },
                   bytes);
            snprintf(nm, sizeof nm, "tma SrcConst grid x%d", mult);
            timeit(nm, [&] { k_csr_tma<SrcConst, EpiStore, false><<<grid, kTmaRows, smem>>>(A, ntiles, cap, SrcConst{}, ep); },
                   bytes - 8.0 * N);
        }
    }
    const size_t words = (size_t)nnz * 12 / 16;
    void* dst;
    cudaMalloc(&dst, words * 16 + 64);
    timeit("copy col+val stream (r+w)", [&] { k_copy<<<4 * 148 * 8, 256>>>((const int4*)av, (int4*)dst, words); },
           2.0 * words * 16);
    return 0;
}
