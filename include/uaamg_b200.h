/*
 * uaamg_b200.h -- C ABI of the B200-native UA-AMG setup/solve path.
 *
 * Drop-in boundary for the reference package /root/reference/pkg/src/uaamg
 * ("U/" below, "K/" = U/kernels/).  Two layers:
 *
 *   1. The kernel table.  The reference selects its hot kernels through a
 *      16-name module table (K/__init__.py:37-54, plugin loader :14-34).  Each
 *      uaamg_k_* entry below replaces one table entry, operating on DEVICE
 *      pointers (int32 indices, float64 values) on the caller's CUDA stream.
 *      Variable-size outputs are two-phase (count, then fill into caller
 *      buffers).  INTEGRATION.md shows the ctypes backend module a maintainer
 *      adds next to K/numba_backend.py to bind these.
 *
 *   2. The drivers.  uaamg_setup replaces U/hierarchy.py:120 setup() and
 *      uaamg_npcg_solve replaces U/solvers.py:190 npcg_solve(); uaamg_cycle
 *      replaces U/solvers.py:128 cycle().  The hierarchy stays device
 *      resident behind an opaque handle.
 *
 * Conventions: every function returns 0 on success or a negative UAAMG_E*
 * code; uaamg_last_error() returns a thread-local message for the last
 * failure.  No C++ exceptions cross the ABI.  `stream` is a cudaStream_t (0 =
 * legacy default stream).  All kernels are deterministic: results do not
 * depend on grid size, stream, or timing (no floating-point atomics).
 * Floating-point sums that the reference performs sequentially (row sums,
 * aggregate sums, Galerkin entry sums) are performed in the same order
 * without FMA contraction, so they are bit-identical to K/numba_backend.py.
 */
#ifndef UAAMG_B200_H
#define UAAMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UAAMG_OK 0
#define UAAMG_EINVAL (-1)      /* bad argument (reference: ValueError)            */
#define UAAMG_ECUDA (-2)       /* CUDA runtime failure                             */
#define UAAMG_ENUMERICAL (-3)  /* reference NumericalError (U/solvers.py:16-21)    */
#define UAAMG_ESETUP (-4)      /* reference SetupError (U/hierarchy.py:18)         */
#define UAAMG_EAGG (-5)        /* reference AggregationError (U/aggregation.py:21) */
#define UAAMG_ENOMEM (-6)
#define UAAMG_EUNSUPPORTED (-7)

typedef struct uaamg_hierarchy uaamg_hierarchy;

/* ------------------------------------------------------------------ */
/* library                                                              */
/* ------------------------------------------------------------------ */
int uaamg_version(void);
const char *uaamg_last_error(void);
/* number of kernel launches issued by this library since load (all threads) */
uint64_t uaamg_launch_count(void);

/* ------------------------------------------------------------------ */
/* kernel table (replaces K/__init__.py:39-54 entries)                  */
/* ------------------------------------------------------------------ */
/* K/numba_backend.py:38-44  hash_u01(seed, pass_idx, idx) */
int uaamg_k_hash_u01(uint64_t seed, int64_t pass_idx, const int64_t *idx, int64_t m, double *out, void *stream);
/* K/numba_backend.py:47-56  spmv(indptr, indices, data, x) */
int uaamg_k_spmv(int n, const int *row_ptr, const int *col, const double *val, const double *x, double *y,
                 void *stream);
/* K/numba_backend.py:59-68  diag_of */
int uaamg_k_diag_of(int n, const int *row_ptr, const int *col, const double *val, double *out, void *stream);
/* K/numba_backend.py:71-84  l1_diag */
int uaamg_k_l1_diag(int n, const int *row_ptr, const int *col, const double *val, double *out, void *stream);
/* K/numba_backend.py:87-97  degrees (int32 output) */
int uaamg_k_degrees(int n, const int *row_ptr, const int *col, int *out, void *stream);
/* K/numba_backend.py:100-111  quasi_random_scores */
int uaamg_k_quasi_random_scores(int n, const int *row_ptr, const int *col, uint64_t seed, int64_t pass_idx,
                                double *out, void *stream);
/* K/numba_backend.py:114-142  squared_pattern: phase 1 counts (out_ptr[n+1]
 * filled, *nnz2 returned), phase 2 (out_idx != NULL) fills sorted rows. */
int uaamg_k_squared_pattern(int n, const int *row_ptr, const int *col, int *out_ptr, int *out_idx, int64_t *nnz2,
                            void *stream);
/* K/numba_backend.py:175-193  select_centers over an explicit pattern P
 * (P = A^2 reproduces the reference exactly; the B200 setup path instead runs
 * the same selection as two max-hops over A, see uaamg_k_select_centers_2hop). */
int uaamg_k_select_centers(int n, const int *p_ptr, const int *p_idx, const double *scores,
                           const uint8_t *processed, uint8_t *is_center, void *stream);
/* same result as uaamg_k_select_centers(A^2 pattern) without forming A^2 */
int uaamg_k_select_centers_2hop(int n, const int *row_ptr, const int *col, const double *scores,
                                const uint8_t *processed, uint8_t *is_center, void *stream);
/* K/numba_backend.py:196-220  claim_owners over an explicit pattern / 2-hop over A */
int uaamg_k_claim_owners(int n, const int *p_ptr, const int *p_idx, const double *scores, const uint8_t *processed,
                         const uint8_t *is_center, int *owner, void *stream);
int uaamg_k_claim_owners_2hop(int n, const int *row_ptr, const int *col, const double *scores,
                              const uint8_t *processed, const uint8_t *is_center, int *owner, void *stream);
/* K/numba_backend.py:223-273  admit_members (in place on processed and
 * vertex_to_agg; centers are listed with their buckets exactly as the
 * reference's host glue builds them, U/aggregation.py:152-168).  cap<=0 means
 * unlimited. */
int uaamg_k_admit_members(int n, const int *row_ptr, const int *col, const double *val, int n_centers,
                          const int *centers, const int *bucket_ptr, const int *bucket_js, int64_t cap,
                          uint8_t *processed, int *vertex_to_agg, int agg_base, void *stream);
/* K/numba_backend.py:145-172  galerkin_coo: phase 1 (out_col == NULL) fills
 * out_ptr[nc+1] and *nnz_c; phase 2 fills out_col/out_val. */
int uaamg_k_galerkin(int n, const int *row_ptr, const int *col, const double *val, const int *v2a, int nc,
                     int *out_ptr, int *out_col, double *out_val, int64_t *nnz_c, void *stream);
/* K/numba_backend.py:276-285  restrict(agg_ptr, members, r) */
int uaamg_k_restrict(int nc, const int *agg_ptr, const int *members, const double *r, double *out, void *stream);
/* K/numba_backend.py:288-294  prolongate_add(v2a, e_coarse, x) */
int uaamg_k_prolongate_add(int n, const int *v2a, const double *e_coarse, const double *x, double *out,
                           void *stream);
/* K/numba_backend.py:297-310  smooth_sweeps (x is not modified; result in out) */
int uaamg_k_smooth_sweeps(int n, const int *row_ptr, const int *col, const double *val, const double *inv_m,
                          const double *x, const double *b, int sweeps, double *out, void *stream);

/* aggregate(A, config) on device (U/aggregation.py:172-203): writes
 * vertex_to_agg[n] and coarse_vertex_of_agg[*n_coarse] (caller buffers of
 * size n).  size_cap <= 0 means unlimited. */
int uaamg_aggregate(int n, const int *row_ptr, const int *col, const double *val, uint64_t seed, int max_passes,
                    int64_t size_cap, int *vertex_to_agg, int *seeds, int *n_coarse, void *stream);

/* ------------------------------------------------------------------ */
/* drivers                                                              */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t size_cap;       /* <= 0: unlimited (AggregationConfig.size_cap=None) */
    uint64_t seed;          /* AggregationConfig.seed                            */
    int max_passes;         /* AggregationConfig.max_passes (20)                 */
    int passes_per_level;   /* AggregationConfig.passes_per_level (1 or 2)       */
    int n0;                 /* setup(n0=100)                                     */
    int max_levels;         /* setup(max_levels=20)                              */
    int singular;           /* -1 auto (detect_singular), 0/1 forced             */
    int reshape_sweeps;     /* setup(reshape_sweeps=0): subgraph reshaping sweeps per level */
    int reshape_pair_cap;   /* setup(reshape_pair_cap=16): largest pair enumerated (<= 16) */
    int borrow;             /* 1: level 0 aliases the caller's arrays (they must
                               outlive the hierarchy, as the reference's Level 0
                               holds the caller's matrix, and each must have
                               64 readable bytes past its last element: the
                               level-0 tile kernel's bulk copies round slices
                               up to 16-byte granules); arrays that are not
                               16-byte aligned are copied anyway; 0: copied */
} uaamg_setup_params;

/* U/hierarchy.py:120-153.  Matrix arrays are device pointers, copied into
 * the hierarchy unless params->borrow.  Returns UAAMG_ESETUP on stagnation
 * (message as the reference's SetupError). */
int uaamg_setup(int n, int64_t nnz, const int *row_ptr, const int *col, const double *val,
                const uaamg_setup_params *params, uaamg_hierarchy **out, void *stream);
/* The same setup from the reference's HOST layout (U/sparse.py SparseMatrix:
 * int64 indptr / indices, float64 data, in host memory) -- the drop-in for a
 * caller that holds the reference's matrix (U/hierarchy.py:120 called on a
 * SparseMatrix).  The library uploads the arrays through pinned staging,
 * narrowing the indices to int32 on the way, and uploads the values WHILE
 * the level-0 aggregation runs (it reads only the pattern).  Level 0 is
 * owned by the hierarchy; params->borrow is ignored.  The host arrays may be
 * reused as soon as the call returns. */
int uaamg_setup_host(int64_t n, int64_t nnz, const int64_t *indptr, const int64_t *indices, const double *data,
                     const uaamg_setup_params *params, uaamg_hierarchy **out, void *stream);
void uaamg_hierarchy_free(uaamg_hierarchy *h);

typedef struct {
    int n_levels;
    int singular;
    double grid_complexity;
    double operator_complexity;
    double setup_seconds;   /* device time of the last setup (CUDA events) */
} uaamg_hierarchy_info;
int uaamg_hierarchy_get_info(const uaamg_hierarchy *h, uaamg_hierarchy_info *info);

/* Device views of level l (valid while h lives).  v2a/seeds/agg_ptr/members
 * are NULL on the coarsest level (n_coarse = 0). */
typedef struct {
    int n;
    int64_t nnz;
    const int *row_ptr;
    const int *col;
    const double *val;
    int n_coarse;
    const int *vertex_to_agg;
    const int *coarse_vertex_of_agg;
    const int *agg_ptr;   /* members_csr (U/aggregation.py:70-77) */
    const int *members;
} uaamg_level_view;
int uaamg_hierarchy_level(const uaamg_hierarchy *h, int level, uaamg_level_view *view);

/* CoarseSolver (U/hierarchy.py:31-65).  uaamg_coarse_factor densifies an
 * n x n CSR matrix on the device and writes into minv (n*n doubles,
 * row-major, caller-owned) its inverse via Cholesky (*mode = 1) or, when
 * `singular` is set or the Cholesky factorisation fails (the reference then
 * sets singular = True), the eigen pseudo-inverse with the reference's
 * cut 1e-12 * max(lambda_max, 0) (*mode = 2).  uaamg_hierarchy_coarse
 * returns the hierarchy's own factor of its coarsest level.
 * uaamg_dense_apply: x = minv b for nrhs right-hand sides (b, x: n x nrhs
 * row-major, i.e. numpy's (n,) or (n, nrhs)) -- CoarseSolver.solve. */
int uaamg_coarse_factor(int n, int64_t nnz, const int *row_ptr, const int *col, const double *val, int singular,
                        double *minv, int *mode, void *stream);
int uaamg_hierarchy_coarse(const uaamg_hierarchy *h, const double **minv, int *n, int *mode);
int uaamg_dense_apply(int n, const double *minv, const double *b, int nrhs, double *x, void *stream);

typedef struct {
    int kcycle;              /* CycleSpec.kind: 1 kcycle, 0 vcycle           */
    int inner_krylov_steps;  /* CycleSpec.inner_krylov_steps (2)            */
    int pre_sweeps;          /* CycleSpec.pre_sweeps (1)                     */
    int post_sweeps;         /* CycleSpec.post_sweeps (1)                    */
    int smoother_l1;         /* Smoother.kind: 1 "l1", 0 "jacobi"            */
    double omega;            /* Smoother.omega (2/3)                         */
    double tol;              /* npcg_solve tol                                */
    int max_iters;           /* npcg_solve max_iters                          */
    int use_graphs;          /* 1: replay one CUDA graph per iteration        */
    int profile_level0;      /* 1: time level-0 smoother kernels (events)     */
} uaamg_solve_params;

typedef struct {
    int iterations;
    int converged;
    int status;              /* 0 ok, UAAMG_ENUMERICAL on breakdown etc.      */
    double solve_seconds;    /* device time (CUDA events)                     */
    /* level-0 hot-kernel timing when profile_level0 = 1 */
    int64_t l0_kernel_launches;
    double l0_kernel_seconds;
    double l0_kernel_bytes;  /* algorithmic bytes over those launches          */
} uaamg_solve_result;

/* U/solvers.py:190-255.  b, x0 (may be NULL), x are device pointers of
 * length n; history (device or host, see history_on_host) receives
 * iterations+1 relative residuals (capacity max_iters+1). */
int uaamg_npcg_solve(uaamg_hierarchy *h, const uaamg_solve_params *p, const double *b, const double *x0, double *x,
                     double *history_host, uaamg_solve_result *res, void *stream);

/* ------------------------------------------------------------------ */
/* Row-partitioned setup and solve over P ranks (
 * paper_1302_2547_b200/csrc/dist_setup.cu, dist_solve.cu).  Level 0 is split
 * into P contiguous row blocks; each rank holds and computes only its rows
 * (global column indices).  Aggregation, renumbering, members and the
 * Galerkin product run per rank, reading halo entries straight from the
 * owning rank's memory; coarse levels keep the inherited partition (rank q
 * owns the aggregates seeded in its rows) until they drop below shard_rows,
 * then they are gathered and replicated on every rank.  The hierarchy is
 * bit-identical to uaamg_setup's for any P; solve histories agree within
 * round-off of the dot products (folded per rank, then in rank order).
 *
 * Communicator: rank >= 0 is one process per GPU -- create, then exchange
 * the 64-byte CUDA IPC handle of every rank's arena (uaamg_comm_handle;
 * e.g. torch.distributed all_gather), then uaamg_comm_connect with the P
 * handles in rank order.  rank = -1 runs all P ranks as VIRTUAL ranks in the
 * calling process on one device (the partition-invariance harness).  Every
 * buffer a peer reads lives in the rank's arena of arena_bytes. */
typedef struct uaamg_comm uaamg_comm;
typedef struct uaamg_dhier uaamg_dhier;
int uaamg_comm_create(int nranks, int rank, int64_t arena_bytes, uaamg_comm **out);
int uaamg_comm_handle(uaamg_comm *c, void *handle64);
int uaamg_comm_connect(uaamg_comm *c, const void *handles);
int uaamg_comm_barrier(uaamg_comm *c);   /* collective host barrier (teardown) */
void uaamg_comm_free(uaamg_comm *c);

/* U/hierarchy.py:120-153, collective.  bounds: P+1 level-0 row bounds.
 * row_ptr/col/val/nnz: one entry per LOCAL rank (1 per process; P for
 * virtual ranks, in rank order): that rank's rows [bounds[r], bounds[r+1])
 * as a CSR with local row offsets and global column indices (device).
 * size_cap must be 0 and passes_per_level 1 (UAAMG_EUNSUPPORTED otherwise).
 * shard_rows: levels with fewer rows are gathered and replicated. */
int uaamg_dsetup(uaamg_comm *c, int n, const int *bounds, const int *const *row_ptr, const int *const *col,
                 const double *const *val, const int64_t *nnz, const uaamg_setup_params *params,
                 int64_t shard_rows, uaamg_dhier **out, void *stream);
void uaamg_dhier_free(uaamg_dhier *d);

typedef struct {
    int n_levels;
    int n_sharded;          /* levels 0 .. n_sharded-1 are row-partitioned */
    int singular;
    double grid_complexity;
    double operator_complexity;
    double setup_seconds;
} uaamg_dhier_info;
int uaamg_dhier_get_info(const uaamg_dhier *d, uaamg_dhier_info *info);

/* Level l as held by local rank `rank` (device views): a sharded level's
 * own rows [row_begin, row_end) (local row offsets, global columns), its
 * v2a (own rows -> global coarse index) and its seeds (own aggregates'
 * seeds, ascending); a replicated level whole. */
typedef struct {
    int n;
    int64_t nnz;            /* global */
    int sharded;
    int row_begin, row_end;
    int64_t local_nnz;
    const int *row_ptr;
    const int *col;
    const double *val;
    int n_coarse;           /* global; 0 on the coarsest level */
    const int *vertex_to_agg;
    const int *seeds;
    int n_seeds;
} uaamg_dlevel_view;
int uaamg_dhier_level(const uaamg_dhier *d, int level, int rank, uaamg_dlevel_view *view);

/* U/solvers.py:190-255 on a row-partitioned hierarchy, collective.  b, x0
 * (NULL or one per local rank), x: per local rank, its own rows (device).
 * Singular (Neumann) hierarchies: the compatibility check and mean
 * projections (U/solvers.py:112-125) are folded across ranks. */
int uaamg_dsolve(uaamg_dhier *d, const uaamg_solve_params *p, const double *const *b, const double *const *x0,
                 double *const *x, double *history_host, uaamg_solve_result *res, void *stream);

/* On-device generator of the 3D lattice Laplacians of the benchmark configs
 * (C2/C4/C5), bit-identical to the host builder
 * problems.grid3d / the reference's assemble_laplacian: box nx*ny*nz,
 * vertex (x*ny + y)*nz + z, stencil 7 or 27, unit weights, Dirichlet by
 * elimination (neumann = 0) or Neumann.  Two passes: col == NULL writes
 * row_ptr (n+1) and returns *nnz; then col/val (nnz each) are filled. */
int uaamg_gen_grid3d(int nx, int ny, int nz, int stencil, int neumann, int *row_ptr, int *col, double *val,
                     int64_t *nnz, void *stream);
/* rows [row_begin, row_end) only (a rank's block of level 0): local row
 * offsets, global column indices; same two passes. */
int uaamg_gen_grid3d_rows(int nx, int ny, int nz, int stencil, int neumann, int row_begin, int row_end,
                          int *row_ptr, int *col, double *val, int64_t *nnz, void *stream);

/* On-device canonical assembly.
 * uaamg_from_coo: U/sparse.py:56-74 SparseMatrix.from_coo on device
 * triplets (int64 rows/cols, float64 vals): stable (row, col) sort,
 * duplicates summed exactly like np.add.reduceat (a0 + numpy pairwise sum of
 * the rest), exact zeros dropped; UAAMG_EINVAL on out-of-range coordinates.
 * uaamg_assemble_laplacian: U/graph.py:63-82 assemble_laplacian on device
 * edge arrays (ei, ej, w: m edges) and boundary arrays (bj, bw: nb entries),
 * diagonal weights accumulated in edge-list order.  Both return a
 * library-owned CSR (int32 row_ptr/col, float64 val on the device). */
typedef struct uaamg_csr uaamg_csr;
int uaamg_from_coo(int64_t n_rows, int64_t n_cols, int64_t m, const int64_t *rows, const int64_t *cols,
                   const double *vals, uaamg_csr **out, void *stream);
int uaamg_assemble_laplacian(int n, int64_t m, const int64_t *ei, const int64_t *ej, const double *w, int64_t nb,
                             const int64_t *bj, const double *bw, uaamg_csr **out, void *stream);
int uaamg_csr_view(const uaamg_csr *c, int *n_rows, int *n_cols, int64_t *nnz, int **row_ptr, int **col,
                   double **val);
void uaamg_csr_free(uaamg_csr *c);

/* U/reshaping.py:215-248 reshape_sweep on a level matrix and its
 * aggregation (device): v2a (n) is updated in place, seeds (nc) receives the
 * smallest member of every aggregate (U/aggregation.py:248-257); *skipped =
 * pairs larger than pair_cap (<= 16).  UAAMG_EINVAL with the reference's
 * message when a pair has no balanced connected split. */
int uaamg_reshape_sweep(int n, int64_t nnz, const int *row_ptr, const int *col, const double *val, int nc, int *v2a,
                        int *seeds, int smoother_l1, double omega, int sweeps, int pair_cap, int *skipped,
                        void *stream);

/* Host <-> device transfers of the reference-layout host arrays (pageable
 * numpy memory): pipelined through a pinned staging ring filled by host
 * threads.  uaamg_h2d copies count elements of src_elem bytes into dst as
 * dst_elem bytes -- equal sizes copy, 8 -> 4 narrows int64 -> int32 (the
 * reference's indices to the device layout).  uaamg_d2h copies bytes.  Both
 * are ordered on `stream` and return when the host buffer may be reused /
 * read. */
int uaamg_h2d(void *dst, const void *src, int64_t count, int src_elem, int dst_elem, void *stream);
int uaamg_d2h(void *dst, const void *src, int64_t bytes, void *stream);

/* Level-0 row partition of the sharded setup (host-only helper): P equal
 * 128-row-aligned blocks. */
int uaamg_partition_rows(int n, int nranks, int *bounds);
/* Coarse-level ranges of the sharded setup's renumbering (host-only):
 * aggregates are numbered by ascending seed, so rank q's aggregates are
 * [bounds[q], bounds[q+1]) = exclusive scan of the per-rank seed counts. */
int uaamg_coarse_bounds(const int64_t *counts, int nranks, int *bounds);

/* Level-0 hot-kernel timing of the last solve run with profile_level0 = 1:
 * device seconds summed over the working iterations (CUDA events captured
 * around the kernels inside the iteration graph) and algorithmic bytes per
 * launch, for [0] residual, [1] fused prolongation + l1/Jacobi post-sweep,
 * [2] direction SpMV (+ dots).  *count = iterations timed. */
int uaamg_solve_profile(const uaamg_hierarchy *h, double *seconds3, double *bytes3, int64_t *count);

/* Which level the last solve ran as one thread-block cluster (the coarse
 * tail kernel: the level above the coarsest, with its coarsest solve); -1
 * when the separate-kernel path ran.  *cluster = CTAs in that cluster.
 * (Diagnostics; UAAMG_NO_TAIL=1 in the environment disables the tail.) */
int uaamg_tail_info(const uaamg_hierarchy *h, int *level, int *cluster);

/* Which row kernel the solve runs on `level` (diagnostics): 0 warp groups
 * (csr_group.cuh), 1 TMA tiles with warp-cooperative gathers, 2 TMA tiles
 * with one thread per row (rows of <= 12 entries), 3 the sliced-ELL copy
 * (csr_ell.cuh: >= 2^20 rows of 13..32 entries; UAAMG_NO_ELL=1 disables). */
int uaamg_level_kernel(const uaamg_hierarchy *h, int level, int *kind);

/* U/solvers.py:128-157: one cycle on level `level` from a zero guess. */
int uaamg_cycle(uaamg_hierarchy *h, const uaamg_solve_params *p, int level, const double *b, double *x,
                void *stream);

/* smooth(a, smoother, x, b, sweeps) for level `level` of h (U/solvers.py:84-91) */
int uaamg_smooth(uaamg_hierarchy *h, const uaamg_solve_params *p, int level, const double *x, const double *b,
                 int sweeps, double *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* UAAMG_B200_H */
