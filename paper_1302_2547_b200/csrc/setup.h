// setup.h -- host-side setup drivers (internal).
#pragma once
#include <functional>

#include "kernels.h"

namespace uaamg {

struct AggStats {
    int passes = 0;
    int leftover = 0;
};

// overlap (optional): host work run while the aggregation kernel executes
// (after its launch, before the host reads the result); capped aggregation
// reads |a_ij|, so there it runs first
int device_aggregate(const Csr& A, const int* deg, uint64_t seed, int max_passes, long long size_cap, int* v2a,
                     int* seeds, cudaStream_t s, AggStats* stats, const std::function<void()>* overlap = nullptr);
void build_members(int n, int nc, const int* v2a, int* agg_ptr, int* members, cudaStream_t s);
long long device_galerkin(const Csr& A, const int* v2a, int nc, const int* agg_ptr, const int* members,
                          DBuf<int>& rp_c, DBuf<int>& ci_c, DBuf<double>& av_c, cudaStream_t s);
int device_coarse_factor(const Csr& A, bool singular, DBuf<double>& Minv, cudaStream_t s);
// subgraph reshaping sweeps (reshape.cu): v2a updated in place, seeds =
// smallest members; returns the number of pairs skipped (> pair_cap)
int device_reshape_sweep(const Csr& A, int nc, int* v2a, int* seeds, int l1, double omega, int sweeps, int pair_cap,
                         cudaStream_t s);

// kernel-table helpers
void launch_select_pattern(const Csr& P, const double* s_, const uint8_t* processed, uint8_t* out, cudaStream_t s);
void launch_claim_pattern(const Csr& P, const double* s_, const uint8_t* processed, const uint8_t* is_center,
                          int* owner, cudaStream_t s);
void select_2hop(const Csr& A, const double* sc, const uint8_t* processed, uint8_t* out, cudaStream_t s);
void claim_2hop(const Csr& A, const double* sc, const uint8_t* processed, const uint8_t* is_center, int* owner,
                cudaStream_t s);
void admit_table(const Csr& A, int nctr, const int* centers, const int* bptr, const int* bjs, long long cap,
                 uint8_t* processed, int* v2a, int agg_base, int total_bucket, cudaStream_t s);
long long squared_pattern(const Csr& A, int* out_ptr, int* out_idx, cudaStream_t s);
void squared_pattern_finish(int n, const unsigned long long* uniq, int m, int* out_ptr, int* out_idx,
                            cudaStream_t s);
void galerkin_table(const Csr& A, const int* v2a, int nc, int* out_ptr, int* out_col, double* out_val,
                    long long* nnz_c, cudaStream_t s);

}  // namespace uaamg
