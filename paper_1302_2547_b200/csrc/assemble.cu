// assemble.cu -- on-device canonical sparse assembly.
//
// from_coo (U/sparse.py:56-74): stable lexicographic sort of the triplets
// by (row, col), duplicates summed exactly as np.add.reduceat does -- a
// length-1 segment is copied, a longer one is a0 + pairwise_sum(a1..) with
// numpy's pairwise summation (8 accumulators up to 128 elements, halving at
// multiples of 8 above) -- then exact zeros dropped and row_ptr counted.
// assemble_laplacian (U/graph.py:63-82): the triplet list the reference
// builds (both directions of every edge with -w, boundary weights on the
// diagonal, then the diagonal of accumulated edge weights -- each vertex's
// weights added in edge-list order, as the reference's Python loop does)
// fed to from_coo.  Bit-identical to the host builders for any weights.
#include <cub/cub.cuh>

#include "kernels.h"

namespace uaamg {

namespace {

// numpy pairwise_sum_DOUBLE over a[0..n) with an index indirection
__device__ double np_pairwise(const double* v, const int* idx, long long n) {
    // pw(a, n) = pw(a, n2) + pw(a + n2, n - n2) evaluated post-order with an
    // explicit work stack (depth ~3 log2(n / 128)) and a result stack
    double parts[40];
    int np_ = 0;
    int op[80];  // 0: evaluate the range, 1: add the top two results
    long long oo[80], on[80];
    int ns = 0;
    op[ns] = 0; oo[ns] = 0; on[ns] = n; ++ns;
    while (ns > 0) {
        --ns;
        const int kind = op[ns];
        if (kind == 1) {
            const double b = parts[--np_];
            const double a = parts[--np_];
            parts[np_++] = __dadd_rn(a, b);
            continue;
        }
        const long long o = oo[ns], m = on[ns];
        if (m < 8) {
            double r = 0.0;
            for (long long i = 0; i < m; ++i) r = __dadd_rn(r, v[idx[o + i]]);
            parts[np_++] = r;
        } else if (m <= 128) {
            double r[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = v[idx[o + j]];
            long long i = 8;
            for (; i < m - (m % 8); i += 8)
#pragma unroll
                for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v[idx[o + i + j]]);
            double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
            for (; i < m; ++i) res = __dadd_rn(res, v[idx[o + i]]);
            parts[np_++] = res;
        } else {
            long long n2 = m / 2;
            n2 -= n2 % 8;
            // post-order: left, right, then combine
            op[ns] = 1; ++ns;
            op[ns] = 0; oo[ns] = o + n2; on[ns] = m - n2; ++ns;
            op[ns] = 0; oo[ns] = o; on[ns] = n2; ++ns;
        }
    }
    return parts[0];
}

__global__ void k_coo_check(long long m, const long long* r, const long long* c, long long nr, long long nc,
                            int* bad) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m; k += (long long)gridDim.x * blockDim.x)
        if (r[k] < 0 || r[k] >= nr || c[k] < 0 || c[k] >= nc) atomicOr(bad, 1);
}
__global__ void k_coo_keys(long long m, const long long* r, const long long* c, long long nc,
                           unsigned long long* key, int* idx) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m; k += (long long)gridDim.x * blockDim.x) {
        key[k] = (unsigned long long)r[k] * (unsigned long long)nc + (unsigned long long)c[k];
        idx[k] = (int)k;
    }
}
__global__ void k_seg_heads(long long m, const unsigned long long* key, int* head) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m; k += (long long)gridDim.x * blockDim.x)
        head[k] = (k == 0 || key[k] != key[k - 1]) ? 1 : 0;
}
// one thread per duplicate segment: numpy reduceat semantics
__global__ void k_seg_sums(int S, long long m, const int* start, const int* idx, const double* v,
                           double* sum, int* keep) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
        const long long a = start[s], b = (s + 1 < S) ? start[s + 1] : m;
        double t = v[idx[a]];
        if (b - a > 1) t = __dadd_rn(t, np_pairwise(v, idx + a + 1, b - a - 1));
        sum[s] = t;
        keep[s] = (t != 0.0) ? 1 : 0;
    }
}
__global__ void k_coo_emit(int S, const int* start, const unsigned long long* key, const double* sum,
                           const int* keep, const int* pos, long long nc, int* rowcnt, int* ci, double* av) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
        if (!keep[s]) continue;
        const unsigned long long k = key[start[s]];
        const long long r = (long long)(k / (unsigned long long)nc), c = (long long)(k % (unsigned long long)nc);
        const int p = pos[s];
        ci[p] = (int)c;
        av[p] = sum[s];
        atomicAdd(rowcnt + r + 1, 1);
    }
}
// Laplacian: the reference's triplet list (U/graph.py:66-81)
__global__ void k_lap_triplets(long long m, long long nb, int n, const long long* ei, const long long* ej,
                               const double* w, const long long* bj, const double* bw, long long* r, long long* c,
                               double* v) {
    const long long tot = 2 * m + nb;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot; k += (long long)gridDim.x * blockDim.x) {
        if (k < 2 * m) {
            const long long e = k >> 1;
            const bool second = k & 1;
            r[k] = second ? ej[e] : ei[e];
            c[k] = second ? ei[e] : ej[e];
            v[k] = -w[e];
        } else {
            const long long q = k - 2 * m;
            r[k] = bj[q];
            c[k] = bj[q];
            v[k] = bw[q];
        }
    }
    (void)n;
}
// incidence list for the diagonal: edge e adds w to its i (first) then its
// j (second) endpoint -- key = vertex, stable sort keeps edge order
__global__ void k_lap_incid(long long m, const long long* ei, const long long* ej, unsigned long long* key,
                            int* idx) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < 2 * m; k += (long long)gridDim.x * blockDim.x) {
        const long long e = k >> 1;
        key[k] = (unsigned long long)((k & 1) ? ej[e] : ei[e]);
        idx[k] = (int)k;
    }
}
__global__ void k_lap_diag(long long m, int n, const unsigned long long* key, const int* idx, const double* w,
                           const int* vstart, double* diag) {
    // one thread per vertex: weights in edge order from 0.0 (diag[i] += w)
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        double d = 0.0;
        for (int k = vstart[u]; k < vstart[u + 1]; ++k) d = __dadd_rn(d, w[idx[k] >> 1]);
        diag[u] = d;
    }
    (void)m;
    (void)key;
}
__global__ void k_vertex_bounds(long long M, int n, const unsigned long long* key, int* vstart) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k <= M; k += (long long)gridDim.x * blockDim.x) {
        const long long prev = k == 0 ? -1 : (long long)key[k - 1];
        const long long cur = k == M ? n : (long long)key[k];
        for (long long u = prev + 1; u <= cur && u <= n; ++u) vstart[u] = (int)k;
    }
}
__global__ void k_lap_diag_triplets(int n, long long base, const double* diag, long long* r, long long* c,
                                    double* v) {
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        r[base + u] = u;
        c[base + u] = u;
        v[base + u] = diag[u];
    }
}

int g256(long long n) { return (int)std::max(1ll, std::min((n + 255) / 256, (long long)kNumSMs * 16)); }

}  // namespace

// canonical CSR from device triplets; out arrays allocated here (DBuf)
long long device_from_coo(long long nr, long long nc, long long m, const long long* r, const long long* c,
                          const double* v, DBuf<int>& rp, DBuf<int>& ci, DBuf<double>& av, cudaStream_t s) {
    if (nr <= 0 || nr >= 0x7fffffffll || nc <= 0 || nc >= 0x7fffffffll || m >= 0x7fffffffll)
        throw Error(UAAMG_EINVAL, "from_coo: dimensions out of the int32 range");
    rp.alloc(nr + 1, s);
    UA_CK(cudaMemsetAsync(rp.p, 0, sizeof(int) * (nr + 1), s));
    if (m == 0) {
        ci.alloc(1, s);
        av.alloc(1, s);
        return 0;
    }
    DBuf<int> bad(1, s);
    UA_CK(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    UA_LAUNCH(k_coo_check, g256(m), 256, 0, s, m, r, c, nr, nc, bad.p);
    DBuf<unsigned long long> key(m, s), keys(m, s);
    DBuf<int> idx(m, s), idxs(m, s);
    UA_LAUNCH(k_coo_keys, g256(m), 256, 0, s, m, r, c, nc, key.p, idx.p);
    int bits = 1;
    while (bits < 64 && ((unsigned long long)(nr) * (unsigned long long)nc) >> bits) ++bits;
    size_t tmp = 0;
    UA_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, keys.p, idx.p, idxs.p, (int)m, 0, bits, s));
    DBuf<char> t(tmp, s);
    UA_CK(cub::DeviceRadixSort::SortPairs(t.p, tmp, key.p, keys.p, idx.p, idxs.p, (int)m, 0, bits, s));
    DBuf<int> head(m, s), start(m, s), nsel(1, s);
    UA_LAUNCH(k_seg_heads, g256(m), 256, 0, s, m, keys.p, head.p);
    cub::CountingInputIterator<int> it(0);
    size_t t2 = 0;
    UA_CK(cub::DeviceSelect::Flagged(nullptr, t2, it, head.p, start.p, nsel.p, (int)m, s));
    DBuf<char> tt(t2, s);
    UA_CK(cub::DeviceSelect::Flagged(tt.p, t2, it, head.p, start.p, nsel.p, (int)m, s));
    int h[2] = {0, 0};
    UA_CK(cudaMemcpyAsync(h, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaMemcpyAsync(h + 1, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    if (h[1]) throw Error(UAAMG_EINVAL, "coordinate out of range");
    const int S = h[0];
    DBuf<double> sum(S, s);
    DBuf<int> keep(S + 1, s), pos(S + 1, s);
    UA_LAUNCH(k_seg_sums, g256(S), 256, 0, s, S, m, start.p, idxs.p, v, sum.p, keep.p);
    UA_CK(cudaMemsetAsync(keep.p + S, 0, sizeof(int), s));
    size_t t3 = 0;
    UA_CK(cub::DeviceScan::ExclusiveSum(nullptr, t3, keep.p, pos.p, S + 1, s));
    DBuf<char> t3b(t3, s);
    UA_CK(cub::DeviceScan::ExclusiveSum(t3b.p, t3, keep.p, pos.p, S + 1, s));
    int nnz = 0;
    UA_CK(cudaMemcpyAsync(&nnz, pos.p + S, sizeof(int), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    ci.alloc(std::max(nnz, 1), s);
    av.alloc(std::max(nnz, 1), s);
    UA_LAUNCH(k_coo_emit, g256(S), 256, 0, s, S, start.p, keys.p, sum.p, keep.p, pos.p, nc, rp.p, ci.p, av.p);
    size_t t4 = 0;
    UA_CK(cub::DeviceScan::InclusiveSum(nullptr, t4, rp.p + 1, rp.p + 1, (int)nr, s));
    DBuf<char> t4b(t4, s);
    UA_CK(cub::DeviceScan::InclusiveSum(t4b.p, t4, rp.p + 1, rp.p + 1, (int)nr, s));
    UA_CK(cudaStreamSynchronize(s));
    return nnz;
}

long long device_assemble_laplacian(int n, long long m, const long long* ei, const long long* ej, const double* w,
                                    long long nb, const long long* bj, const double* bw, DBuf<int>& rp,
                                    DBuf<int>& ci, DBuf<double>& av, cudaStream_t s) {
    const long long M = 2 * m + nb + n;
    DBuf<long long> r(M, s), c(M, s);
    DBuf<double> v(M, s), diag(n, s);
    if (m + nb > 0)
        UA_LAUNCH(k_lap_triplets, g256(2 * m + nb), 256, 0, s, m, nb, n, ei, ej, w, bj, bw, r.p, c.p, v.p);
    // diagonal: per vertex, its edge weights in edge order (U/graph.py:70-73)
    DBuf<int> vstart(n + 1, s);
    if (m > 0) {
        DBuf<unsigned long long> key(2 * m, s), keys(2 * m, s);
        DBuf<int> idx(2 * m, s), idxs(2 * m, s);
        UA_LAUNCH(k_lap_incid, g256(2 * m), 256, 0, s, m, ei, ej, key.p, idx.p);
        int bits = 1;
        while (bits < 64 && ((unsigned long long)n >> bits)) ++bits;
        size_t tmp = 0;
        UA_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, keys.p, idx.p, idxs.p, (int)(2 * m), 0, bits, s));
        DBuf<char> t(tmp, s);
        UA_CK(cub::DeviceRadixSort::SortPairs(t.p, tmp, key.p, keys.p, idx.p, idxs.p, (int)(2 * m), 0, bits, s));
        UA_LAUNCH(k_vertex_bounds, g256(2 * m + 1), 256, 0, s, 2 * m, n, keys.p, vstart.p);
        UA_LAUNCH(k_lap_diag, g256(n), 256, 0, s, m, n, keys.p, idxs.p, w, vstart.p, diag.p);
        UA_CK(cudaStreamSynchronize(s));
    } else {
        UA_CK(cudaMemsetAsync(diag.p, 0, sizeof(double) * n, s));
    }
    UA_LAUNCH(k_lap_diag_triplets, g256(n), 256, 0, s, n, 2 * m + nb, diag.p, r.p, c.p, v.p);
    return device_from_coo(n, n, M, r.p, c.p, v.p, rp, ci, av, s);
}

}  // namespace uaamg

// ====================================================================== C ABI
struct uaamg_csr {
    int n_rows = 0, n_cols = 0;
    long long nnz = 0;
    uaamg::DBuf<int> rp, ci;
    uaamg::DBuf<double> av;
};

namespace uaamg {
extern thread_local std::string g_last_error;
cudaStream_t library_stream();
}

using namespace uaamg;

#define UA_ATRY(...)                                                                                    \
    try {                                                                                               \
        __VA_ARGS__;                                                                                    \
        const cudaError_t pe = cudaGetLastError();                                                      \
        if (pe != cudaSuccess) throw Error(UAAMG_ECUDA, std::string("pending CUDA error: ") + cudaGetErrorString(pe)); \
        return UAAMG_OK;                                                                                \
    } catch (const Error& e) {                                                                          \
        g_last_error = e.what();                                                                        \
        return e.code;                                                                                  \
    } catch (const std::exception& e) {                                                                 \
        g_last_error = e.what();                                                                        \
        return UAAMG_ECUDA;                                                                             \
    }

extern "C" {

int uaamg_from_coo(int64_t n_rows, int64_t n_cols, int64_t m, const int64_t* rows, const int64_t* cols,
                   const double* vals, uaamg_csr** out, void* stream) {
    UA_ATRY({
        auto c = std::make_unique<uaamg_csr>();
        cudaStream_t s = (cudaStream_t)stream;
        c->n_rows = (int)n_rows;
        c->n_cols = (int)n_cols;
        c->nnz = device_from_coo(n_rows, n_cols, m, (const long long*)rows, (const long long*)cols, vals, c->rp,
                                 c->ci, c->av, s);
        UA_CK(cudaStreamSynchronize(s));
        *out = c.release();
    })
}

int uaamg_assemble_laplacian(int n, int64_t m, const int64_t* ei, const int64_t* ej, const double* w, int64_t nb,
                             const int64_t* bj, const double* bw, uaamg_csr** out, void* stream) {
    UA_ATRY({
        auto c = std::make_unique<uaamg_csr>();
        cudaStream_t s = (cudaStream_t)stream;
        c->n_rows = c->n_cols = n;
        c->nnz = device_assemble_laplacian(n, m, (const long long*)ei, (const long long*)ej, w, nb,
                                           (const long long*)bj, bw, c->rp, c->ci, c->av, s);
        UA_CK(cudaStreamSynchronize(s));
        *out = c.release();
    })
}

int uaamg_csr_view(const uaamg_csr* c, int* n_rows, int* n_cols, int64_t* nnz, int** row_ptr, int** col,
                   double** val) {
    *n_rows = c->n_rows;
    *n_cols = c->n_cols;
    *nnz = c->nnz;
    *row_ptr = c->rp.p;
    *col = c->ci.p;
    *val = c->av.p;
    return UAAMG_OK;
}

void uaamg_csr_free(uaamg_csr* c) { delete c; }

}  // extern "C"
