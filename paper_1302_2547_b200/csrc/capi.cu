// capi.cu -- kernel-table entry points (replacing K/__init__.py:39-54).
// Device pointers in, device pointers out, caller's stream.
#include <cstring>
#include <string>

#include "setup.h"

namespace uaamg {
extern thread_local std::string g_last_error;

static Csr make_csr(int n, const int* rp, const int* ci, const double* av) {
    Csr c;
    c.n = n; c.rp = rp; c.ci = ci; c.av = av;
    return c;
}

__global__ void k_copy_i(int n, const int* a, int* b) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}
}  // namespace uaamg

using namespace uaamg;

#define UA_GUARD(...)                                                                        \
    try {                                                                                    \
        __VA_ARGS__;                                                                         \
        const cudaError_t pe_ = cudaGetLastError();                                          \
        if (pe_ != cudaSuccess)                                                              \
            throw Error(UAAMG_ECUDA, std::string("pending CUDA error after ") + __func__ + ": " + \
                                         cudaGetErrorString(pe_));                           \
        return UAAMG_OK;                                                                     \
    } catch (const Error& e) {                                                               \
        g_last_error = e.what();                                                             \
        return e.code;                                                                       \
    } catch (const std::exception& e) {                                                      \
        g_last_error = e.what();                                                             \
        return UAAMG_ECUDA;                                                                  \
    }

extern "C" {

int uaamg_gen_grid3d(int nx, int ny, int nz, int stencil, int neumann, int* row_ptr, int* col, double* val,
                     int64_t* nnz, void* stream) {
    UA_GUARD({
        const long long r = gen_grid3d(nx, ny, nz, stencil, neumann, row_ptr, col, val, (cudaStream_t)stream);
        if (nnz && r >= 0) *nnz = r;
    })
}

int uaamg_reshape_sweep(int n, int64_t nnz, const int* row_ptr, const int* col, const double* val, int nc, int* v2a,
                        int* seeds, int smoother_l1, double omega, int sweeps, int pair_cap, int* skipped,
                        void* stream) {
    UA_GUARD({
        Csr A = make_csr(n, row_ptr, col, val);
        A.nnz = (int)nnz;
        const int k = device_reshape_sweep(A, nc, v2a, seeds, smoother_l1, omega, sweeps, pair_cap,
                                           (cudaStream_t)stream);
        if (skipped) *skipped = k;
    })
}

int uaamg_gen_grid3d_rows(int nx, int ny, int nz, int stencil, int neumann, int row_begin, int row_end,
                          int* row_ptr, int* col, double* val, int64_t* nnz, void* stream) {
    UA_GUARD({
        const long long r = gen_grid3d(nx, ny, nz, stencil, neumann, row_ptr, col, val, (cudaStream_t)stream,
                                       row_begin, row_end);
        if (nnz && r >= 0) *nnz = r;
    })
}

int uaamg_k_hash_u01(uint64_t seed, int64_t pass_idx, const int64_t* idx, int64_t m, double* out, void* stream) {
    UA_GUARD(launch_hash_u01(seed, pass_idx, idx, m, out, (cudaStream_t)stream))
}

int uaamg_k_spmv(int n, const int* row_ptr, const int* col, const double* val, const double* x, double* y,
                 void* stream) {
    UA_GUARD({
        cudaStream_t s = (cudaStream_t)stream;
        launch_spmv(make_csr(n, row_ptr, col, val), exact_groups(n), x, y, s);
    })
}

int uaamg_k_diag_of(int n, const int* row_ptr, const int* col, const double* val, double* out, void* stream) {
    UA_GUARD(launch_diag(make_csr(n, row_ptr, col, val), 0, out, (cudaStream_t)stream))
}

int uaamg_k_l1_diag(int n, const int* row_ptr, const int* col, const double* val, double* out, void* stream) {
    UA_GUARD(launch_diag(make_csr(n, row_ptr, col, val), 1, out, (cudaStream_t)stream))
}

int uaamg_k_degrees(int n, const int* row_ptr, const int* col, int* out, void* stream) {
    UA_GUARD(launch_degrees(make_csr(n, row_ptr, col, nullptr), out, (cudaStream_t)stream))
}

int uaamg_k_quasi_random_scores(int n, const int* row_ptr, const int* col, uint64_t seed, int64_t pass_idx,
                                double* out, void* stream) {
    UA_GUARD({
        cudaStream_t s = (cudaStream_t)stream;
        DBuf<int> deg(std::max(n, 1), s);
        Csr A = make_csr(n, row_ptr, col, nullptr);
        launch_degrees(A, deg.p, s);
        launch_scores(A, deg.p, seed, pass_idx, out, s);
    })
}

int uaamg_k_squared_pattern(int n, const int* row_ptr, const int* col, int* out_ptr, int* out_idx, int64_t* nnz2,
                            void* stream) {
    UA_GUARD({
        cudaStream_t s = (cudaStream_t)stream;
        Csr A = make_csr(n, row_ptr, col, nullptr);
        *nnz2 = squared_pattern(A, out_ptr, out_idx, s);
        UA_CK(cudaStreamSynchronize(s));
    })
}

int uaamg_k_select_centers(int n, const int* p_ptr, const int* p_idx, const double* scores,
                           const uint8_t* processed, uint8_t* is_center, void* stream) {
    UA_GUARD(launch_select_pattern(make_csr(n, p_ptr, p_idx, nullptr), scores, processed, is_center,
                                   (cudaStream_t)stream))
}

int uaamg_k_select_centers_2hop(int n, const int* row_ptr, const int* col, const double* scores,
                                const uint8_t* processed, uint8_t* is_center, void* stream) {
    UA_GUARD(select_2hop(make_csr(n, row_ptr, col, nullptr), scores, processed, is_center, (cudaStream_t)stream))
}

int uaamg_k_claim_owners(int n, const int* p_ptr, const int* p_idx, const double* scores, const uint8_t* processed,
                         const uint8_t* is_center, int* owner, void* stream) {
    UA_GUARD(launch_claim_pattern(make_csr(n, p_ptr, p_idx, nullptr), scores, processed, is_center, owner,
                                  (cudaStream_t)stream))
}

int uaamg_k_claim_owners_2hop(int n, const int* row_ptr, const int* col, const double* scores,
                              const uint8_t* processed, const uint8_t* is_center, int* owner, void* stream) {
    UA_GUARD(claim_2hop(make_csr(n, row_ptr, col, nullptr), scores, processed, is_center, owner,
                        (cudaStream_t)stream))
}

int uaamg_k_admit_members(int n, const int* row_ptr, const int* col, const double* val, int n_centers,
                          const int* centers, const int* bucket_ptr, const int* bucket_js, int64_t cap,
                          uint8_t* processed, int* vertex_to_agg, int agg_base, void* stream) {
    UA_GUARD({
        cudaStream_t s = (cudaStream_t)stream;
        int total = 0;
        UA_CK(cudaMemcpyAsync(&total, bucket_ptr + n_centers, sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        admit_table(make_csr(n, row_ptr, col, val), n_centers, centers, bucket_ptr, bucket_js,
                    cap <= 0 ? (1ll << 62) : cap, processed, vertex_to_agg, agg_base, total, s);
    })
}

int uaamg_k_galerkin(int n, const int* row_ptr, const int* col, const double* val, const int* v2a, int nc,
                     int* out_ptr, int* out_col, double* out_val, int64_t* nnz_c, void* stream) {
    UA_GUARD({
        long long m = 0;
        int nnz = 0;
        cudaStream_t s = (cudaStream_t)stream;
        UA_CK(cudaMemcpyAsync(&nnz, row_ptr + n, sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        Csr A = make_csr(n, row_ptr, col, val);
        A.nnz = nnz;
        galerkin_table(A, v2a, nc, out_ptr, out_col, out_val, &m, s);
        *nnz_c = m;
    })
}

int uaamg_k_restrict(int nc, const int* agg_ptr, const int* members, const double* r, double* out, void* stream) {
    UA_GUARD({
        cudaStream_t s = (cudaStream_t)stream;
        launch_restrict_exact(nc, agg_ptr, members, exact_groups(nc), r, out, s);
    })
}

int uaamg_k_prolongate_add(int n, const int* v2a, const double* e_coarse, const double* x, double* out,
                           void* stream) {
    UA_GUARD(launch_prolongate(n, 2, nullptr, nullptr, x, v2a, e_coarse, nullptr, out, nullptr,
                               (cudaStream_t)stream))
}

int uaamg_k_smooth_sweeps(int n, const int* row_ptr, const int* col, const double* val, const double* inv_m,
                          const double* x, const double* b, int sweeps, double* out, void* stream) {
    UA_GUARD({
        cudaStream_t s = (cudaStream_t)stream;
        if (sweeps <= 0) {
            UA_CK(cudaMemcpyAsync(out, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        } else {
            Csr A = make_csr(n, row_ptr, col, val);
            DBuf<double> t0(std::max(n, 1), s), t1(std::max(n, 1), s);
            const double* cur = x;
            for (int k = 0; k < sweeps; ++k) {
                double* nx = (k == sweeps - 1) ? out : ((cur == t0.p) ? t1.p : t0.p);
                launch_sweep_exact(A, exact_groups(n), inv_m, b, cur, nx, s);
                cur = nx;
            }
            UA_CK(cudaStreamSynchronize(s));
        }
    })
}

int uaamg_aggregate(int n, const int* row_ptr, const int* col, const double* val, uint64_t seed, int max_passes,
                    int64_t size_cap, int* vertex_to_agg, int* seeds, int* n_coarse, void* stream) {
    UA_GUARD({
        cudaStream_t s = (cudaStream_t)stream;
        if (max_passes < 1) throw Error(UAAMG_EAGG, "max_passes must be >= 1");
        Csr A = make_csr(n, row_ptr, col, val);
        DBuf<int> deg(std::max(n, 1), s);
        launch_degrees(A, deg.p, s);
        *n_coarse = device_aggregate(A, deg.p, seed, max_passes, size_cap, vertex_to_agg, seeds, s, nullptr);
    })
}

}  // extern "C"
