// l0_sweep.cu -- level-0 kernel size sweep (diagnostics, not product).
// 3D 7-point (or 27-point) Laplacian n^3 built on the device; times the
// l1-sweep epilogue (out = x + invm (b - A x)) through the TMA tile kernel
// and the group kernel, and a plain streaming copy of the same byte count,
// at several sizes -- to split each kernel's time into a fixed part and a
// bandwidth part (t = t0 + bytes / BW).
// Build + run: tools/l0_sweep.sh [stencil]
#include <cstdio>
#include <type_traits>
#include <vector>

#include "../paper_1302_2547_b200/csrc/csr_group.cuh"
#include "../paper_1302_2547_b200/csrc/csr_tma.cuh"
#include "../paper_1302_2547_b200/csrc/csr_ell.cuh"
#include <cub/cub.cuh>

using namespace uaamg;
namespace uaamg {
std::atomic<uint64_t> g_launches{0};
}

__global__ void k_count(int n, int st, int* rp) {
    const long long N = (long long)n * n * n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i / ((long long)n * n)), y = (int)((i / n) % n), z = (int)(i % n);
        int c = 0;
        for (int dx = -1; dx <= 1; ++dx)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dz = -1; dz <= 1; ++dz) {
                    if (st == 7 && abs(dx) + abs(dy) + abs(dz) > 1) continue;
                    if (x + dx < 0 || x + dx >= n || y + dy < 0 || y + dy >= n || z + dz < 0 || z + dz >= n) continue;
                    ++c;
                }
        rp[i + 1] = c;
        if (i == 0) rp[0] = 0;
    }
}
__global__ void k_fill(int n, int st, const int* rp, int* ci, double* av) {
    const long long N = (long long)n * n * n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i / ((long long)n * n)), y = (int)((i / n) % n), z = (int)(i % n);
        int p = rp[i];
        for (int dx = -1; dx <= 1; ++dx)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dz = -1; dz <= 1; ++dz) {
                    if (st == 7 && abs(dx) + abs(dy) + abs(dz) > 1) continue;
                    if (x + dx < 0 || x + dx >= n || y + dy < 0 || y + dy >= n || z + dz < 0 || z + dz >= n) continue;
                    ci[p] = (int)(i + ((long long)dx * n + dy) * n + dz);
                    av[p] = (dx | dy | dz) ? -1.0 : (double)(st - 1);
                    ++p;
                }
    }
}
__global__ void k_scan_serial(long long N, int* rp) {  // tiny helper, one thread (setup only)
    for (long long i = 1; i <= N; ++i) rp[i] += rp[i - 1];
}
__global__ void k_copy(const int4* a, int4* b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_fillv(long long n, double* v, double x) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) v[i] = x;
}

int main(int argc, char** argv) {
    const int st = argc > 1 ? atoi(argv[1]) : 7;
    std::vector<int> sizes = st == 7 ? std::vector<int>{96, 128, 160, 192, 256} : std::vector<int>{96, 128, 160, 192, 256};
    void* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("stencil %d\n%-6s %10s %10s | %-30s %9s %9s %6s\n", st, "n", "rows", "MB", "kernel", "us", "GB/s", "frac");
    for (int n : sizes) {
        const long long N = (long long)n * n * n;
        int *rp, *ci;
        double *av, *x, *b, *iv, *y;
        cudaMalloc(&rp, sizeof(int) * (N + 1) + 64);
        k_count<<<1184, 256>>>(n, st, rp);
        // prefix sum with cub would be nicer; serial scan on one thread is fine for a tool
        k_scan_serial<<<1, 1>>>(N, rp);
        int nnz = 0;
        cudaMemcpy(&nnz, rp + N, sizeof(int), cudaMemcpyDeviceToHost);
        cudaMalloc(&ci, sizeof(int) * (size_t)nnz + 64);
        cudaMalloc(&av, sizeof(double) * (size_t)nnz + 64);
        k_fill<<<1184, 256>>>(n, st, rp, ci, av);
        cudaMalloc(&x, sizeof(double) * N + 64);
        cudaMalloc(&b, sizeof(double) * N + 64);
        cudaMalloc(&iv, sizeof(double) * N + 64);
        cudaMalloc(&y, sizeof(double) * N + 64);
        k_fillv<<<1184, 256>>>(N, x, 0.5);
        k_fillv<<<1184, 256>>>(N, b, 1.0);
        k_fillv<<<1184, 256>>>(N, iv, 1.0 / 12.0);
        cudaDeviceSynchronize();
        Csr A;
        A.n = (int)N; A.nnz = nnz; A.rp = rp; A.ci = ci; A.av = av;
        Groups G = exact_groups((int)N);
        const double bytes = 12.0 * nnz + 4.0 * (N + 1) + 32.0 * N;  // sweep: x gathered, b, invm in, out
        auto timeit = [&](const char* name, auto&& launch, double by) {
            float best = 1e9;
            for (int r = 0; r < 12; ++r) {
                cudaMemsetAsync(flush, r, 256 << 20);
                cudaEventRecord(e0);
                launch();
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r >= 2) best = std::min(best, ms);
            }
            const double gbs = by / (best * 1e-3) / 1e9;
            printf("%-6d %10lld %10.1f | %-30s %9.1f %9.1f %6.3f\n", n, N, by / 1e6, name, best * 1e3, gbs, gbs / 6555.2);
            cudaError_t err = cudaGetLastError();
            if (err) printf("  error %s\n", cudaGetErrorString(err));
        };
        EpiSweep ep{};
        ep.invm = iv; ep.b = b; ep.out = y; ep.g = nullptr;
        timeit("group sweep", [&] {
            const int grid = std::min(cdiv(G.units(), kGrpWarps), kNumSMs * kGrpCtasPerSM);
            k_csr_group<SrcVec, EpiSweep, false><<<grid, 32 * kGrpWarps>>>(A, G, SrcVec{x}, ep);
        }, bytes);
        // max nonzeros per tile (regular stencil: interior bound), 128- and 64-row tiles
        auto tma = [&](auto rows_tag, auto stages_tag) {
            constexpr int R = decltype(rows_tag)::value;
            constexpr int S = decltype(stages_tag)::value;
            const int cap = st * R;
            if (cap > kTmaMaxCap) return;
            const size_t smem = tma_smem_bytes(cap, R, S);
            auto kfn = k_csr_tma<SrcVec, EpiSweep, false, R, S>;
            cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kTmaThreads, smem);
            const int ntiles = cdiv(N, R);
            const int grid = std::min(ntiles, kNumSMs * occ);
            char nm[64];
            snprintf(nm, sizeof nm, "tma%d s%d (%d CTA/SM, %zu B)", R, S, occ, smem);
            timeit(nm, [&] { kfn<<<grid, kTmaThreads, smem>>>(A, 0, (int)N, ntiles, cap, SrcVec{x}, ep, 0); }, bytes);
        };
        tma(std::integral_constant<int, 128>{}, std::integral_constant<int, 3>{});
        tma(std::integral_constant<int, 64>{}, std::integral_constant<int, 3>{});
        {
            // sliced ELL copy (csr_ell.cuh)
            const int nsl = (int)cdiv(N, 32);
            long long *slab, *off;
            cudaMalloc(&slab, sizeof(long long) * (nsl + 1));
            cudaMalloc(&off, sizeof(long long) * (nsl + 1));
            cudaMemset(slab, 0, sizeof(long long) * (nsl + 1));
            k_ell_width<<<1184, 256>>>((int)N, 0, rp, slab);
            size_t tmp = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tmp, slab, off, nsl + 1);
            void* t;
            cudaMalloc(&t, tmp);
            cub::DeviceScan::ExclusiveSum(t, tmp, slab, off, nsl + 1);
            long long tot = 0;
            cudaMemcpy(&tot, off + nsl, sizeof(long long), cudaMemcpyDeviceToHost);
            int* ecol;
            double* eval;
            cudaMalloc(&ecol, sizeof(int) * tot);
            cudaMalloc(&eval, sizeof(double) * tot);
            k_ell_fill<<<1184, 256>>>((int)N, 0, rp, ci, av, off, ecol, eval);
            cudaDeviceSynchronize();
            Ell E;
            E.off = off; E.col = ecol; E.val = eval;
            for (int mult : {4, 8, 16}) {
                const int grid = std::min(cdiv(nsl, kEllWarps), kNumSMs * mult);
                char nm[64];
                snprintf(nm, sizeof nm, "ell grid %dxSM (pad %.3f)", mult, (double)tot / nnz);
                timeit(nm, [&] { k_ell<SrcVec, EpiSweep, false><<<grid, 32 * kEllWarps>>>(A, 0, (int)N, E, SrcVec{x}, ep); }, bytes);
            }
            cudaFree(slab); cudaFree(off); cudaFree(t); cudaFree(ecol); cudaFree(eval);
        }
        auto tmar = [&](auto rows_tag, auto stages_tag) {
            constexpr int R = decltype(rows_tag)::value;
            constexpr int S = decltype(stages_tag)::value;
            const int cap = st * R;
            if (cap > 4096) return;
            const size_t smem = tma_smem_bytes(cap, R, S);
            auto kfn = k_csr_tma_rows<SrcVec, EpiSweep, false, R, S>;
            cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, R, smem);
            const int ntiles = cdiv(N, R);
            const int grid = std::min(ntiles, kNumSMs * occ);
            char nm[64];
            snprintf(nm, sizeof nm, "rows%d s%d (%d CTA/SM, %zu B)", R, S, occ, smem);
            timeit(nm, [&] { kfn<<<grid, R, smem>>>(A, 0, (int)N, ntiles, cap, SrcVec{x}, ep, 0); }, bytes);
        };
        tmar(std::integral_constant<int, 128>{}, std::integral_constant<int, 3>{});
        tmar(std::integral_constant<int, 128>{}, std::integral_constant<int, 2>{});
        tmar(std::integral_constant<int, 256>{}, std::integral_constant<int, 2>{});
        tmar(std::integral_constant<int, 64>{}, std::integral_constant<int, 3>{});
        const size_t words = (size_t)(bytes / 2) / 16;
        void *src, *dst;
        cudaMalloc(&src, words * 16 + 64);
        cudaMalloc(&dst, words * 16 + 64);
        cudaMemset(src, 1, words * 16);
        timeit("copy (same bytes, r+w)", [&] { k_copy<<<4 * 148 * 8, 256>>>((const int4*)src, (int4*)dst, words); },
               2.0 * words * 16);
        cudaFree(src);
        cudaFree(dst);
        cudaFree(rp); cudaFree(ci); cudaFree(av); cudaFree(x); cudaFree(b); cudaFree(iv); cudaFree(y);
    }
    return 0;
}
