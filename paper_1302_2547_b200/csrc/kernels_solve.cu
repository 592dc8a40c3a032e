// kernels_solve.cu -- solve-phase kernels: staged SpMV family, smoother
// diagonals, transfers, flexible-CG vector updates with fused deterministic
// reductions, dense coarsest solve.
//
// Reference semantics: U/solvers.py (smoother_inverse_diag :69-81, smooth
// :84-91, transfers :94-109, projections :112-125, cycle :128-157,
// _inner_fcg :160-187, npcg_solve :190-255) and K/numba_backend.py kernels.
#include <cstdlib>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "launch.cuh"

namespace uaamg {

std::atomic<uint64_t> g_launches{0};

void launch_spmv(const Csr& A, const Groups& G, const double* x, double* y, cudaStream_t s) {
    EpiStore e{};
    e.y = y;
    run_stream<SrcVec, EpiStore, false>(A, G, SrcVec{x}, e, s);
}

void launch_sweep_exact(const Csr& A, const Groups& G, const double* invm, const double* b, const double* x,
                        double* out, cudaStream_t s) {
    EpiSweep e{};
    e.invm = invm; e.b = b; e.out = out; e.g = nullptr;
    run_stream<SrcVec, EpiSweep, false>(A, G, SrcVec{x}, e, s);
}

void launch_restrict_exact(int nc, const int* agg_ptr, const int* members, const Groups& MG, const double* r,
                           double* rc, cudaStream_t s) {
    Csr P;
    P.n = nc; P.rp = agg_ptr; P.ci = members; P.av = nullptr;
    EpiStoreG e{};
    e.y = rc; e.g = nullptr;
    run_stream<SrcVec, EpiStoreG, true>(P, MG, SrcVec{r}, e, s);
}

void launch_residual(const Csr& A, const Groups& G, int xmode, const double* invm, const double* b,
                     const double* x, double* r, const int* gate, Exec ex) {
    EpiResid e{};
    e.b = b; e.r = r; e.g = gate;
    if (xmode == 1) run_stream<SrcPre1, EpiResid, false>(A, G, SrcPre1{invm, b}, e, ex);
    else if (xmode == 0) run_stream<SrcZero, EpiResid, false>(A, G, SrcZero{}, e, ex);
    else run_stream<SrcVec, EpiResid, false>(A, G, SrcVec{x}, e, ex);
}

static EpiSweepBeta sweep_beta(const double* invm, const double* b, double* out, const int* gate,
                               const BetaReq& br, RedScratch rs) {
    EpiSweepBeta e{};
    e.invm = invm; e.b = b; e.out = out; e.g = gate;
    e.apprev = br.apprev; e.beta = br.beta; e.pap = br.pap; e.have = br.have;
    e.red = {rs.partials, rs.ticket};
    return e;
}

void launch_residual_sum(const Csr& A, const Groups& G, int xmode, const double* invm, const double* b,
                         const double* x, double* r, double* rc, double* ec, const double* minv, const int* gate,
                         RedScratch rs, Exec ex) {
    EpiResidSum e{};
    e.b = b; e.r = r; e.g = gate; e.rc = rc; e.ec = ec; e.minv = minv; e.red = {rs.partials, rs.ticket};
    if (xmode == 1) run_stream<SrcPre1, EpiResidSum, false>(A, G, SrcPre1{invm, b}, e, ex);
    else if (xmode == 0) run_stream<SrcZero, EpiResidSum, false>(A, G, SrcZero{}, e, ex);
    else run_stream<SrcVec, EpiResidSum, false>(A, G, SrcVec{x}, e, ex);
}

void launch_sweep_vec(const Csr& A, const Groups& G, const double* invm, const double* b, const double* x,
                      double* out, const int* gate, Exec ex, const BetaReq* br, RedScratch rs) {
    if (br) {
        run_stream<SrcVec, EpiSweepBeta, false>(A, G, SrcVec{x}, sweep_beta(invm, b, out, gate, *br, rs), ex);
        return;
    }
    EpiSweep e{};
    e.invm = invm; e.b = b; e.out = out; e.g = gate;
    run_stream<SrcVec, EpiSweep, false>(A, G, SrcVec{x}, e, ex);
}

void launch_sweep_up(const Csr& A, const Groups& G, int xmode, const double* invm, const double* b,
                     const double* xpre, const int* v2a, const double* ec, const int* ec_valid, double* out,
                     const int* gate, Exec ex, const BetaReq* br, RedScratch rs) {
    SrcUp src{};
    src.mode = xmode; src.invm = invm; src.b = b; src.xpre = xpre; src.v2a = v2a; src.ec = ec;
    src.ec_valid = ec_valid;
    if (br) {
        run_stream<SrcUp, EpiSweepBeta, false>(A, G, src, sweep_beta(invm, b, out, gate, *br, rs), ex);
        return;
    }
    EpiSweep e{};
    e.invm = invm; e.b = b; e.out = out; e.g = gate;
    run_stream<SrcUp, EpiSweep, false>(A, G, src, e, ex);
}

void launch_restrict(int nc, const int* agg_ptr, const int* members, const Groups& MG, const double* r,
                     double* rc, const int* gate, Exec ex, FcgState* begin_st, RedScratch rs) {
    Csr P;
    P.n = nc; P.rp = agg_ptr; P.ci = members; P.av = nullptr;
    if (begin_st) {
        EpiRestrictBegin e{};
        e.y = rc; e.g = gate; e.st = begin_st; e.red = {rs.partials, rs.ticket};
        run_stream<SrcVec, EpiRestrictBegin, true>(P, MG, SrcVec{r}, e, ex);
        return;
    }
    EpiStoreG e{};
    e.y = rc; e.g = gate;
    run_stream<SrcVec, EpiStoreG, true>(P, MG, SrcVec{r}, e, ex);
}

void launch_dir_fcg(const Csr& A, const Groups& G, const double* z, const double* pprev, int have_prev,
                    const double* r, double* p, double* ap, FcgState* st, int step, RedScratch rs,
                    Exec ex) {
    EpiDirFcg e{};
    e.p = p; e.ap = ap; e.r = r; e.st = st; e.step = step; e.red = {rs.partials, rs.ticket};
    SrcDir src{};
    src.z = z; src.pprev = pprev; src.beta_p = &st->beta; src.have_p = nullptr; src.have_static = have_prev;
    if (G.tma_cap > 0 || G.n >= kTmaMinRows) {
        // large level: p first, then a plain-gather SpMV (same arithmetic;
        // one gathered array instead of z and p_prev)
        BodyDirP bp{};
        bp.src = src; bp.p = p; bp.g = &st->gate[step];
        run_map(A.n, bp, ex);
        e.p = nullptr;
        run_stream<SrcVec, EpiDirFcg, false>(A, G, SrcVec{p}, e, ex);
        return;
    }
    run_stream<SrcDir, EpiDirFcg, false>(A, G, src, e, ex);
}

bool launch_dir_update_fcg(const Csr& A, const Groups& G, const double* z, const double* pprev, int have_prev,
                           const double* r, double* p, double* ap, double* x, double* r_out, FcgState* st, int step,
                           RedScratch rs, double* part, unsigned* bar, Exec ex, bool last, const ParentUp* pu) {
    static const bool no_fuse = getenv("UAAMG_NO_DIR_FUSE") != nullptr;  // A/B diagnostics
    if (G.tma_cap > 0 || G.n >= kTmaMinRows || no_fuse) {
        launch_dir_fcg(A, G, z, pprev, have_prev, r, p, ap, st, step, rs, ex);
        launch_fcg_update(A.n, step, x, p, r, r_out, ap, st, 0, rs, ex, last);
        return false;
    }
    EpiDirFcg e{};
    e.p = p; e.ap = ap; e.r = r; e.st = st; e.step = step; e.red = {rs.partials, rs.ticket};
    SrcDir src{};
    src.z = z; src.pprev = pprev; src.beta_p = &st->beta; src.have_p = nullptr; src.have_static = have_prev;
    BodyFcgUpd u{};
    u.step = step; u.x = x; u.p = p; u.rin = r; u.rout = r_out; u.ap = ap; u.st = st; u.singular = 0;
    u.last = last ? 1 : 0;
    u.red = {rs.partials, rs.ticket};
    if (last && pu) u.pu = *pu;
    static int maxg_dev[kMaxDevices] = {};
    int& maxg = maxg_dev[cur_dev()];
    if (!maxg) {
        int occ = 0;
        UA_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dir_update<SrcDir>, 32 * kGrpWarps, 0));
        maxg = std::max(1, occ) * kNumSMs;
    }
    const int grid = std::max(1, std::min(cdiv(std::max(G.units(), 1), kGrpWarps), std::min(maxg, kNumSMs * 8)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32 * kGrpWarps);
    cfg.stream = ex.s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    UA_CK(cudaLaunchKernelEx(&cfg, k_dir_update<SrcDir>, A, G, src, e, u, part, bar));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return u.pu.n > 0;
}

void launch_dir_npcg(const Csr& A, const Groups& G, const double* z, const double* pprev, const double* r,
                     double* p, double* ap, NpcgState* st, RedScratch rs, cudaStream_t s) {
    EpiDirNpcg e{};
    e.p = p; e.ap = ap; e.r = r; e.st = st; e.red = {rs.partials, rs.ticket};
    SrcDir src{};
    src.z = z; src.pprev = pprev; src.beta_p = &st->beta; src.have_p = &st->have_prev;
    if (G.tma_cap > 0 || G.n >= kTmaMinRows) {
        BodyDirP bp{};
        bp.src = src; bp.p = p; bp.g = &st->active;
        run_map(A.n, bp, s);
        e.p = nullptr;
        run_stream<SrcVec, EpiDirNpcg, false>(A, G, SrcVec{p}, e, s);
        return;
    }
    run_stream<SrcDir, EpiDirNpcg, false>(A, G, src, e, s);
}

// ============================================================ groups
namespace {
struct LongRow {
    const int* rp;
    int lo;
    __device__ bool operator()(int i) const { return rp[i + 1] - rp[i] > lo; }
};
__global__ void k_row_bounds(int m, const int* rows, const int* rp, int2* out) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x)
        out[k] = make_int2(rp[rows[k]], rp[rows[k] + 1]);
}
}  // namespace

__global__ void k_tile_nnz_max(int n, int rows, const int* rp, int* out) {  // rp: first row of the range
    const int nt = (n + rows - 1) / rows;
    int m = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x)
        m = max(m, rp[min((t + 1) * rows, n)] - rp[t * rows]);
    m = block_max(m);
    if (threadIdx.x == 0) atomicMax(out, m);
}

int max_tile_nnz(int n, const int* rp, cudaStream_t s, int base, int rows) {
    rp += base;
    if (n == 0) return 0;
    DBuf<int> m(1, s);
    UA_CK(cudaMemsetAsync(m.p, 0, sizeof(int), s));
    UA_LAUNCH(k_tile_nnz_max, std::min(cdiv(cdiv(n, rows), 256), 4 * kNumSMs), 256, 0, s, n, rows, rp, m.p);
    int h = 0;
    UA_CK(cudaMemcpyAsync(&h, m.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    return h;
}

void set_tma(Groups& g, int n, const int* rp, cudaStream_t s, int base) {
    static const bool no64 = getenv("UAAMG_NO_TMA64") != nullptr;  // A/B diagnostics
    const bool no_rowpar = getenv("UAAMG_NO_ROWPAR") != nullptr;  // (read per setup)
    g.tma_rowpar = 0;
    if (!no_rowpar && max_tile_nnz(n, rp, s, base, 1) <= kTmaRowParMaxRow) {
        // short rows (7-point-like): thread-per-row tiles beat the gather
        // (tools/l0_sweep.cu: 0.75 vs 0.69 of HBM at 128^3)
        const int cap = max_tile_nnz(n, rp, s, base, kTmaRowParRows);
        if (cap <= kTmaMaxCap) {
            g.tma_cap = std::max(cap, 4);
            g.tma_rows = kTmaRowParRows;
            g.tma_rowpar = 1;
            return;
        }
    }
    int cap = max_tile_nnz(n, rp, s, base, kTmaRows);
    if (cap <= kTmaMaxCap) {
        g.tma_cap = std::max(cap, 4);
        g.tma_rows = kTmaRows;
        return;
    }
    if (no64) return;
    cap = max_tile_nnz(n, rp, s, base, 64);
    if (cap <= kTmaMaxCap) {
        g.tma_cap = std::max(cap, 4);
        g.tma_rows = 64;
    }
}

bool set_ell(GroupBuf& gb, const Csr& A, cudaStream_t s, int n, int base) {
    const bool no_ell = getenv("UAAMG_NO_ELL") != nullptr;  // A/B diagnostics (read per setup)
    if (n < 0) n = A.n;
    if (no_ell || n < kEllMinRows || gb.g.np != 0 || gb.g.tma_rowpar) return false;
    const int maxrow = max_tile_nnz(n, A.rp, s, base, 1);
    if (maxrow > kEllMaxRow) return false;
    const int nsl = cdiv(n, 32);
    DBuf<long long> slab(nsl + 1, s);
    UA_CK(cudaMemsetAsync(slab.p, 0, sizeof(long long) * (nsl + 1), s));
    UA_LAUNCH(k_ell_width, std::min(cdiv(nsl * 32, 256), 8 * kNumSMs), 256, 0, s, n, base, A.rp, slab.p);
    gb.ell_off.alloc(nsl + 1, s);
    size_t tmp = 0;
    UA_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, slab.p, gb.ell_off.p, nsl + 1, s));
    DBuf<char> t(tmp, s);
    UA_CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, slab.p, gb.ell_off.p, nsl + 1, s));
    long long tot = 0;
    UA_CK(cudaMemcpyAsync(&tot, gb.ell_off.p + nsl, sizeof(long long), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    static size_t total_mem_dev[kMaxDevices] = {};
    size_t& total_mem = total_mem_dev[cur_dev()];
    if (!total_mem) {
        size_t fr = 0;
        UA_CK(cudaMemGetInfo(&fr, &total_mem));
    }
    // (the copy is 12 B per slab entry: at most a quarter of the device)
    long long nnz = 0;  // this row range's nonzeros
    {
        int e[2];
        UA_CK(cudaMemcpyAsync(&e[0], A.rp + base, sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaMemcpyAsync(&e[1], A.rp + base + n, sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        nnz = (long long)e[1] - e[0];
    }
    if ((double)tot > kEllMaxPad * (double)nnz || (double)tot * 12.0 > 0.25 * (double)total_mem) {
        gb.ell_off.release();
        return false;
    }
    gb.ell_col.alloc((size_t)tot, s);
    gb.ell_val.alloc((size_t)tot, s);
    UA_LAUNCH(k_ell_fill, std::min(cdiv(nsl * 32, 256), 8 * kNumSMs), 256, 0, s, n, base, A.rp, A.ci, A.av,
              gb.ell_off.p, gb.ell_col.p, gb.ell_val.p);
    gb.g.ell_off = gb.ell_off.p;
    gb.g.ell_col = gb.ell_col.p;
    gb.g.ell_val = gb.ell_val.p;
    return true;
}

void build_groups(int n, const int* rp, int long_min, GroupBuf& out, cudaStream_t s, int base) {
    out.g = exact_groups(n, base);
    rp += base;  // local view: row i of the range at rp[i]
    out.g.long_min = long_min;
    if (n == 0 || long_min == 0x7fffffff) return;
    DBuf<int> rows(n, s), cnt(1, s);
    thrust::counting_iterator<int> it(0);
    size_t tmp = 0;
    UA_CK(cub::DeviceSelect::If(nullptr, tmp, it, rows.p, cnt.p, n, LongRow{rp, long_min}, s));
    DBuf<char> t(tmp, s);
    UA_CK(cub::DeviceSelect::If(t.p, tmp, it, rows.p, cnt.p, n, LongRow{rp, long_min}, s));
    int m = 0;
    UA_CK(cudaMemcpyAsync(&m, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    if (m == 0) return;
    DBuf<int2> bnd(m, s);
    UA_LAUNCH(k_row_bounds, cdiv(m, 256), 256, 0, s, m, rows.p, rp, bnd.p);
    std::vector<int> hrows(m);
    std::vector<int2> hb(m);
    UA_CK(cudaMemcpyAsync(hrows.data(), rows.p, sizeof(int) * m, cudaMemcpyDeviceToHost, s));
    UA_CK(cudaMemcpyAsync(hb.data(), bnd.p, sizeof(int2) * m, cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    std::vector<int4> pcs;
    std::vector<int> pbase(m + 1, 0);
    for (int k = 0; k < m; ++k) {
        pbase[k] = (int)pcs.size();
        for (int e = hb[k].x; e < hb[k].y; e += kGrpRound)
            pcs.push_back(make_int4(base + hrows[k], e, std::min(e + kGrpRound, hb[k].y), k));
    }
    pbase[m] = (int)pcs.size();
    out.piece.alloc(pcs.size(), s);
    out.pbase.alloc(m + 1, s);
    out.ticket.alloc(m, s);
    out.part.alloc(pcs.size(), s);
    out.lval.alloc((size_t)kMaxLongK * m, s);
    UA_CK(cudaMemcpyAsync(out.piece.p, pcs.data(), sizeof(int4) * pcs.size(), cudaMemcpyHostToDevice, s));
    UA_CK(cudaMemcpyAsync(out.pbase.p, pbase.data(), sizeof(int) * (m + 1), cudaMemcpyHostToDevice, s));
    UA_CK(cudaMemsetAsync(out.ticket.p, 0, sizeof(unsigned) * m, s));
    UA_CK(cudaStreamSynchronize(s));  // host vectors are temporaries
    out.g.np = (int)pcs.size();
    out.g.piece = out.piece.p;
    out.g.pbase = out.pbase.p;
    out.g.ticket = out.ticket.p;
    out.g.part = out.part.p;
    out.g.nlong = m;
    out.g.lval = out.lval.p;
}

// ---- smoother diagonal (U/solvers.py:69-81, K/numba_backend.py:59-84)
// Rows of at most kSolveLongMin entries: a thread each, |a_ij| summed in
// ascending order (K/numba_backend.py:71-84) with the loads batched 8 at a
// time.  Longer rows (the solve path's piece rows) are skipped here and
// done by k_inv_diag_long, a block per row (fixed block-tree order, like the
// solve's long-row pieces).
__device__ __forceinline__ void inv_diag_fin(int i, double acc, double dii, int l1, double omega, double* invm,
                                             int* bad_row) {
    const double m = l1 ? __dadd_rn(acc, dii) : dii;
    if (m <= 0.0) atomicMin(bad_row, i);
    invm[i] = (l1 ? 1.0 : omega) / m;
}
// rows [base, base + n) (a rank's rows of a sharded level: rp and invm are
// indexed by global row)
__global__ void k_inv_diag(Csr A, int base, int n, int l1, double omega, double* invm, int* bad_row) {
    for (int i = base + blockIdx.x * blockDim.x + threadIdx.x; i < base + n; i += gridDim.x * blockDim.x) {
        const int e0 = A.rp[i], e1 = A.rp[i + 1];
        if (e1 - e0 > kSolveLongMin) continue;
        double acc = 0.0, dii = 0.0;
        bool seen = false;
        for (int k0 = e0; k0 < e1; k0 += 8) {
            int c[8];
            double a[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = k0 + q < e1 ? A.ci[k0 + q] : -1;
                a[q] = k0 + q < e1 ? A.av[k0 + q] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (c[q] < 0) continue;
                if (l1) {
                    if (c[q] == i) dii = a[q];  // l1: the last diagonal entry (loop over k)
                    else acc = __dadd_rn(acc, fabs(a[q]));
                } else if (c[q] == i && !seen) {
                    dii = a[q];  // jacobi: the first diagonal entry (the loop breaks there)
                    seen = true;
                }
            }
        }
        inv_diag_fin(i, acc, dii, l1, omega, invm, bad_row);
    }
}
__global__ void k_inv_diag_long(Csr A, const int4* piece, const int* pbase, int l1, double omega, double* invm,
                                int* bad_row) {
    __shared__ double sm[kThreads / 32 + 1];
    __shared__ double sd[kThreads / 32 + 1];
    const int row = piece[pbase[blockIdx.x]].x;
    const int e0 = A.rp[row], e1 = A.rp[row + 1];
    double acc = 0.0, dii = 0.0;
    for (int k = e0 + threadIdx.x; k < e1; k += blockDim.x) {
        const int c = A.ci[k];
        const double a = A.av[k];
        if (c == row) dii = a;
        else if (l1) acc = __dadd_rn(acc, fabs(a));
    }
    acc = block_sum<kThreads>(acc, sm);
    dii = block_sum<kThreads>(dii, sd);  // the one diagonal entry (zeros elsewhere)
    if (threadIdx.x == 0) inv_diag_fin(row, acc, dii, l1, omega, invm, bad_row);
}

void launch_inv_diag(const Csr& A, const GroupBuf& G, int l1, double omega, double* invm, int* bad_row,
                     cudaStream_t s) {
    UA_LAUNCH(k_inv_diag, map_grid(G.g.n) * 2, kThreads, 0, s, A, G.g.base, G.g.n, l1, omega, invm, bad_row);
    const int nlong = G.pbase.n > 0 ? (int)G.pbase.n - 1 : 0;
    if (nlong > 0 && G.g.long_min == kSolveLongMin)
        UA_LAUNCH(k_inv_diag_long, nlong, kThreads, 0, s, A, G.g.piece, G.g.pbase, l1, omega, invm, bad_row);
}

__global__ void k_diag(Csr A, int l1, double* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
        double acc = 0.0, dii = 0.0;
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            const int c = A.ci[k];
            if (l1) {
                if (c == i) dii = A.av[k];
                else acc = __dadd_rn(acc, fabs(A.av[k]));
            } else if (c == i) {
                dii = A.av[k];
                break;
            }
        }
        out[i] = l1 ? __dadd_rn(acc, dii) : dii;
    }
}

void launch_diag(const Csr& A, int l1, double* out, cudaStream_t s) {
    UA_LAUNCH(k_diag, map_grid(A.n) * 2, kThreads, 0, s, A, l1, out);
}

void launch_xpre1(int n, const double* invm, const double* b, double* x, const int* gate, Exec ex) {
    BodyXpre1 body{};
    body.invm = invm; body.b = b; body.x = x; body.g = gate;
    run_map(n, body, ex);
}

void launch_prolongate(int n, int xmode, const double* invm, const double* b, const double* xpre, const int* v2a,
                       const double* ec, const int* ec_valid, double* out, const int* gate, Exec ex) {
    BodyProl body{};
    body.src.mode = xmode; body.src.invm = invm; body.src.b = b; body.src.xpre = xpre; body.src.v2a = v2a;
    body.src.ec = ec; body.src.ec_valid = ec_valid; body.out = out; body.g = gate;
    run_map(n, body, ex);
}

void launch_fcg_begin(int n, const double* b, const int* parent_gate, FcgState* st, RedScratch rs, Exec ex) {
    BodyFcgBegin body{};
    body.b = b; body.pg = parent_gate; body.st = st; body.red = {rs.partials, rs.ticket};
    run_map(n, body, ex);
}

void launch_beta(int n, const double* z, const double* pprev, const double* apprev, double* beta, const int* gate,
                 const int* gate2, RedScratch rs, Exec ex) {
    BodyBeta body{};
    body.z = z; body.pp = pprev; body.ap = apprev; body.beta = beta; body.g = gate; body.g2 = gate2;
    body.red = {rs.partials, rs.ticket};
    run_map(n, body, ex);
}



void launch_fcg_update(int n, int step, double* x, const double* p, const double* r_in, double* r_out,
                       const double* ap, FcgState* st, int singular, RedScratch rs, Exec ex, bool last) {
    if (last && !singular) {
        BodyFcgUpdLast body{};
        body.step = step; body.x = x; body.p = p; body.st = st;
        run_map(n, body, ex);
        return;
    }
    BodyFcgUpd body{};
    body.step = step; body.x = x; body.p = p; body.rin = r_in; body.rout = r_out; body.ap = ap; body.st = st;
    body.singular = singular; body.red = {rs.partials, rs.ticket};
    run_map(n, body, ex);
    if (singular) {
        BodyFcgProj pj{};
        pj.n = n; pj.step = step; pj.r = r_out; pj.st = st; pj.red = {rs.partials, rs.ticket};
        run_map(n, pj, ex);
    }
}



void launch_npcg_update(int n, double* x, const double* p, double* r, const double* ap, NpcgState* st,
                        double* history, int singular, RedScratch rs, cudaStream_t s) {
    BodyNpcgUpd body{};
    body.x = x; body.p = p; body.r = r; body.ap = ap; body.st = st; body.hist = history; body.singular = singular;
    body.red = {rs.partials, rs.ticket};
    run_map(n, body, s);
    if (singular) {
        BodyNpcgProjX bx{};
        bx.x = x; bx.st = st; bx.red = {rs.partials, rs.ticket};
        run_map(n, bx, s);
        BodyNpcgProj pj{};
        pj.n = n; pj.x = x; pj.r = r; pj.st = st; pj.hist = history; pj.red = {rs.partials, rs.ticket};
        run_map(n, pj, s);
    }
}

void launch_project_mean(int n, double* v, double* sum_slot, const int* gate, RedScratch rs, Exec ex) {
    BodySum bs{};
    bs.v = v; bs.slot = sum_slot; bs.g = gate; bs.red = {rs.partials, rs.ticket};
    run_map(n, bs, ex);
    BodySub sb{};
    sb.n = n; sb.in = v; sb.out = v; sb.slot = sum_slot; sb.g = gate;
    run_map(n, sb, ex);
}

void launch_check_compatible(int n, const double* b, double* out, int* err_flag, double* sum_slot,
                             const int* gate, int level, RedScratch rs, Exec ex) {
    (void)level;
    BodyCompat bc{};
    bc.b = b; bc.slot = sum_slot; bc.err = err_flag; bc.n = n; bc.g = gate; bc.red = {rs.partials, rs.ticket};
    run_map(n, bc, ex);
    BodySub sb{};
    sb.n = n; sb.in = b; sb.out = out; sb.slot = sum_slot; sb.g = gate;
    run_map(n, sb, ex);
}

// ---- dense coarsest solve x = Minv b (warp per row)
__global__ void k_dense_solve(int n, const double* __restrict__ M, const double* __restrict__ b, double* x,
                              const int* gate) {
    pdl_wait();
    pdl_trigger();
    if (gate && !*gate) return;
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= n) return;
    double acc = 0.0;
    for (int j = lane; j < n; j += 32) acc += M[(size_t)row * n + j] * b[j];
    acc = warp_sum(acc);
    if (lane == 0) x[row] = acc;
}
void launch_dense_solve(int n, const double* Minv, const double* b, double* x, const int* gate, Exec ex) {
    if (n == 0) return;
    UA_LAUNCH_PDL(k_dense_solve, cdiv(n, 8), 256, 0, ex.s, n, Minv, b, x, gate);
}

// x = M b for nrhs right-hand sides (row-major n x nrhs): warp per output,
// the same lane-strided dot + shuffle tree as k_dense_solve, so nrhs = 1
// gives the solve path's bits
__global__ void k_dense_apply(int n, const double* __restrict__ M, const double* __restrict__ b, int nrhs,
                              double* x) {
    const int lane = threadIdx.x & 31;
    const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= (long long)n * nrhs) return;
    const int row = (int)(w / nrhs), c = (int)(w % nrhs);
    double acc = 0.0;
    for (int j = lane; j < n; j += 32) acc += M[(size_t)row * n + j] * b[(size_t)j * nrhs + c];
    acc = warp_sum(acc);
    if (lane == 0) x[(size_t)row * nrhs + c] = acc;
}
void launch_dense_apply(int n, const double* Minv, const double* b, int nrhs, double* x, cudaStream_t s) {
    if (n == 0 || nrhs == 0) return;
    UA_LAUNCH(k_dense_apply, cdiv((long long)n * nrhs, 8), 256, 0, s, n, Minv, b, nrhs, x);
}

void launch_norm(int n, const double* v, double* out, RedScratch rs, cudaStream_t s) {
    BodyNorm b{};
    b.v = v; b.out = out; b.red = {rs.partials, rs.ticket};
    run_map(n, b, s);
}

void launch_npcg_init(int n, const double* b, const double* r, NpcgState* st, double* history, RedScratch rs,
                      cudaStream_t s) {
    BodyNpcgInit body{};
    body.b = b; body.r = r; body.st = st; body.hist = history; body.red = {rs.partials, rs.ticket};
    run_map(n, body, s);
}

void launch_copy(int n, const double* src, double* dst, cudaStream_t s) {
    BodyCopy b{};
    b.a = src; b.o = dst;
    run_map(n, b, s);
}
void launch_axpby_init(int n, const double* b, const double* ax, double* r, cudaStream_t s) {
    BodyBmAx body{};
    body.b = b; body.ax = ax; body.r = r;
    run_map(n, body, s);
}

}  // namespace uaamg

// ============================================================ problem generation
// On-device 3D lattice Laplacian: the canonical CSR
// that paper_1302_2547_b200/problems.py:grid3d builds on the host (itself
// bit-identical to the reference's assemble_laplacian(GraphProblem(...)),
// U/graph.py:63-82, U/sparse.py:56-74): vertex i = (x*ny + y)*nz + z, columns
// ascending (offsets dx outer, dz inner), off-diagonals -1, diagonal
// stencil-1 (Dirichlet by elimination) or the degree (Neumann).
namespace uaamg {
namespace {
__device__ __forceinline__ int grid_nbrs(int x, int y, int z, int nx, int ny, int nz, int stencil, int* off,
                                         long long sxy, int sy) {
    int k = 0;
    for (int dx = -1; dx <= 1; ++dx)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dz = -1; dz <= 1; ++dz) {
                if (stencil == 7 && abs(dx) + abs(dy) + abs(dz) > 1) continue;
                if ((dx < 0 && x == 0) || (dx > 0 && x == nx - 1) || (dy < 0 && y == 0) || (dy > 0 && y == ny - 1) ||
                    (dz < 0 && z == 0) || (dz > 0 && z == nz - 1))
                    continue;
                if (off) off[k] = (int)(dx * sxy + dy * sy + dz);
                ++k;
            }
    return k;
}
// rows [r0, r1) of the lattice; row_ptr / cnt local (index i - r0), columns global
__global__ void k_grid_count(int nx, int ny, int nz, int stencil, long long r0, long long r1, int* cnt) {
    for (long long i = r0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < r1; i += (long long)gridDim.x * blockDim.x) {
        const int z = (int)(i % nz), y = (int)((i / nz) % ny), x = (int)(i / ((long long)ny * nz));
        cnt[i - r0 + 1] = grid_nbrs(x, y, z, nx, ny, nz, stencil, nullptr, (long long)ny * nz, nz);
        if (i == r0) cnt[0] = 0;
    }
}
__global__ void k_grid_fill(int nx, int ny, int nz, int stencil, int neumann, long long r0, long long r1, const int* rp,
                            int* ci, double* av) {
    for (long long i = r0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < r1; i += (long long)gridDim.x * blockDim.x) {
        const int z = (int)(i % nz), y = (int)((i / nz) % ny), x = (int)(i / ((long long)ny * nz));
        int off[27];
        const int k = grid_nbrs(x, y, z, nx, ny, nz, stencil, off, (long long)ny * nz, nz);
        const double diag = neumann ? (double)(k - 1) : (double)(stencil - 1);
        int p = rp[i - r0];
        for (int q = 0; q < k; ++q, ++p) {
            ci[p] = (int)(i + off[q]);
            av[p] = off[q] == 0 ? diag : -1.0;
        }
    }
}
}  // namespace

long long gen_grid3d(int nx, int ny, int nz, int stencil, int neumann, int* rp, int* ci, double* av,
                     cudaStream_t s, long long r0, long long r1) {
    const long long N = (long long)nx * ny * nz;
    if (N <= 0 || N > 0x7fffffffll) throw Error(UAAMG_EINVAL, "grid size out of range");
    if (stencil != 7 && stencil != 27) throw Error(UAAMG_EINVAL, "stencil must be 7 or 27");
    if (r1 < 0) r1 = N;
    if (r0 < 0 || r0 > r1 || r1 > N) throw Error(UAAMG_EINVAL, "row range out of the grid");
    const long long n = r1 - r0;
    const int grid = std::max(1, std::min(cdiv(n, 256), 8 * kNumSMs));
    if (!ci) {
        // pass 1: row_ptr (counts + inclusive scan), returns nnz
        if (n == 0) {
            UA_CK(cudaMemsetAsync(rp, 0, sizeof(int), s));
            return 0;
        }
        UA_LAUNCH(k_grid_count, grid, 256, 0, s, nx, ny, nz, stencil, r0, r1, rp);
        size_t tmp = 0;
        UA_CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, rp + 1, rp + 1, (int)n, s));
        DBuf<char> t(tmp, s);
        UA_CK(cub::DeviceScan::InclusiveSum(t.p, tmp, rp + 1, rp + 1, (int)n, s));
        int nnz = 0;
        UA_CK(cudaMemcpyAsync(&nnz, rp + n, sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        return nnz;
    }
    if (n) UA_LAUNCH(k_grid_fill, grid, 256, 0, s, nx, ny, nz, stencil, neumann, r0, r1, rp, ci, av);
    return -1;
}
}  // namespace uaamg
