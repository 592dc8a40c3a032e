// runtime.h -- device-resident hierarchy, solve workspaces and the solve
// plan (internal; shared by runtime.cu and shard.cu).
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "csr_tma.cuh"
#include "setup.h"
#include "tail.h"

namespace uaamg {

extern thread_local std::string g_last_error;

struct Level {
    int n = 0;
    long long nnz = 0;
    DBuf<int> rp, ci;
    DBuf<double> av;
    GroupBuf grp;   // warp work units of A (solve path: long rows split)
    int nc = 0;  // 0 on the coarsest level
    DBuf<int> v2a, seeds, agg_ptr, members;
    GroupBuf mgrp;  // warp work units of members_csr (restriction)
    Csr csr() const {
        Csr c;
        c.n = n; c.nnz = (int)nnz; c.rp = rp.p; c.ci = ci.p; c.av = av.p;
        return c;
    }
    const Groups& groups() const { return grp.g; }
    const Groups& mgroups() const { return mgrp.g; }
};

struct LevelWs {
    DBuf<double> invm, r, rhs, e, tA, tB, bp, xup;           // cycle (xup: large levels, post > 1)
    DBuf<double> xf, rf, z, p0, p1, ap0, ap1;                // inner FCG
};

constexpr int kLookahead = 3;  // iteration graphs queued ahead of the host's flag read
constexpr int kEvRing = 4;
int mapped_slot_acquire(int** host, int** dev);
void mapped_slot_release(int k);
// executable-graph cache keyed by (parity, node count): an update is only
// tried on a graph of the same shape, so it does not fail into a fresh
// instantiation (several ms) inside a timed solve
cudaGraphExec_t graph_cache_take(int par, size_t nodes);
void graph_cache_give(cudaGraphExec_t e, int dev, int par, size_t nodes);

struct SolveWs {
    uaamg_solve_params key{};
    int dev = 0;            // device the workspace (and its graphs) live on
    bool ready = false;
    std::vector<LevelWs> lev;
    DBuf<FcgState> fcg;     // one per level
    DBuf<NpcgState> npcg;
    DBuf<double> partials;
    DBuf<unsigned> ticket;
    DBuf<double> sums;      // per-level scratch sums (singular)
    DBuf<int> err;          // incompatibility flag
    DBuf<int> bad_row;
    // outer vectors
    DBuf<double> r, z, p0, p1, ap0, ap1, hist, bproj;
    TailPlan tail;         // the level above the coarsest in one cluster (tail.cu)
    DBuf<double> fpart;    // fused direction + update: per-CTA partials
    DBuf<unsigned> fbar;   // and its grid barrier
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    size_t graph_nodes[2] = {0, 0};  // node counts (graph cache key)
    uint64_t graph_kernels[2] = {0, 0};  // kernel launches recorded per graph
    // level-0 hot-kernel timing (profile_level0): event pairs per graph parity
    // around the residual, fused up-sweep and direction-SpMV kernels
    cudaEvent_t pev[2][6] = {};
    bool profiled = false;
    double prof_seconds[3] = {0, 0, 0};  // residual, up-sweep, direction SpMV
    int64_t prof_count = 0;
    bool graphs_built = false;
    double* graph_x = nullptr;  // graphs bake in the iterate pointer
    int* h_flags = nullptr;  // pinned, mapped: [0] mirror of NpcgState::active
    int* d_flags = nullptr;  // its device address
    int flag_slot = -1;      // slot in the shared mapped page (mapped_slot_acquire)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaEvent_t evr[4] = {nullptr, nullptr, nullptr, nullptr};  // lookahead ring (kEvRing)
    ~SolveWs() {
        for (int k = 0; k < 2; ++k) graph_cache_give(graph[k], dev, k, graph_nodes[k]);  // its work has completed
        for (auto& row : pev)
            for (auto& e : row) if (e) cudaEventDestroy(e);
        mapped_slot_release(flag_slot);
        for (auto& e : ev) if (e) cudaEventDestroy(e);
        for (auto& e : evr) if (e) cudaEventDestroy(e);
    }
};

}  // namespace uaamg

struct uaamg_hierarchy {
    std::vector<std::unique_ptr<uaamg::Level>> levels;
    bool singular = false;
    int coarse_mode = 0;
    uaamg::DBuf<double> Minv;
    double grid_complexity = 1, operator_complexity = 1, setup_seconds = 0;
    cudaStream_t stream = 0;  // library-owned non-blocking stream (capturable)
    std::unique_ptr<uaamg::SolveWs> ws;
    std::mutex mu;
    ~uaamg_hierarchy() {
        ws.reset();
        levels.clear();
        Minv.release();
        // the library stream is shared by all hierarchies (library_stream)
    }
};

namespace uaamg {

// ------------------------------------------------------------------ helpers
// Orders the library's own stream after the caller's stream on entry and the
// caller's stream after the library's on exit (the caller may pass the legacy
// default stream, which cannot be graph-captured).
struct StreamJoin {
    cudaStream_t caller, own;
    StreamJoin(cudaStream_t c, cudaStream_t o) : caller(c), own(o) {
        if (c == o) return;
        cudaEvent_t ev;
        UA_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        UA_CK(cudaEventRecord(ev, c));
        UA_CK(cudaStreamWaitEvent(o, ev, 0));
        cudaEventDestroy(ev);
    }
    ~StreamJoin() {
        if (caller == own) return;
        cudaEvent_t ev;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return;
        cudaEventRecord(ev, own);
        cudaStreamWaitEvent(caller, ev, 0);
        cudaEventDestroy(ev);
    }
};

// U/solvers.py:128-255 on one device: cycle / _inner_fcg / one NPCG
// iteration as a fixed launch sequence (see runtime.cu)
struct Plan {
    uaamg_hierarchy* h;
    SolveWs* ws;
    uaamg_solve_params p;
    cudaStream_t s;
    int prof = -1;  // >= 0: record level-0 timing events of this parity
    Exec ex() const { return Exec(s); }
    void mark(int k) {
        // External: a real event-record node inside the captured graph (a
        // plain cudaEventRecord during capture only orders nodes)
        if (prof >= 0) UA_CK(cudaEventRecordWithFlags(ws->pev[prof][k], s, cudaEventRecordExternal));
    }
    RedScratch rs() const { return RedScratch{ws->partials.p, ws->ticket.p}; }
    int coarsest() const { return (int)h->levels.size() - 1; }
    bool sing() const { return h->singular; }

    // U/solvers.py:128-157.  br: fuse the beta dot of the flexible CG that
    // consumes `out` into the last sweep; returns whether that happened.
    bool cycle(int l, const double* b, double* out, const int* gate, const BetaReq* br = nullptr) {
        Level& L = *h->levels[l];
        LevelWs& W = ws->lev[l];
        if (sing()) {
            launch_check_compatible(L.n, b, W.bp.p, ws->err.p, ws->sums.p + 4 * l, gate, l, rs(), ex());
            b = W.bp.p;
        }
        if (l == coarsest()) {
            launch_dense_solve(L.n, h->Minv.p, b, out, gate, ex());
            if (sing()) launch_project_mean(L.n, out, ws->sums.p + 4 * l + 2, gate, rs(), ex());
            return false;
        }
        const Csr A = L.csr();
        const Groups& B = L.groups();
        // pre-smoothing from a zero guess.  Large (HBM-bound) levels
        // materialise the pre-smoothed iterate and the prolongated iterate
        // instead of rebuilding them inside every gather: two cheap
        // streaming passes make both SpMVs plain vector gathers (same
        // arithmetic, same bits).
        const bool mat = L.n >= kTmaMinRows;
        int xmode = p.pre_sweeps == 0 ? 0 : (p.pre_sweeps == 1 && !mat ? 1 : 2);
        const double* xpre = nullptr;
        double* cur = W.tA.p;
        if (xmode == 2) {
            launch_xpre1(L.n, W.invm.p, b, W.tA.p, gate, ex());
            for (int k = 1; k < p.pre_sweeps; ++k) {
                double* nx = (cur == W.tA.p) ? W.tB.p : W.tA.p;
                launch_sweep_vec(A, B, W.invm.p, b, cur, nx, gate, ex());
                cur = nx;
            }
            xpre = cur;
        }
        LevelWs& C = ws->lev[l + 1];
        const bool exact = (l + 1 == coarsest());
        // coarsest level = one aggregate: residual, restriction (a sum) and
        // the 1x1 solve in one kernel
        if (exact && L.nc == 1 && !sing() && l > 0) {
            launch_residual_sum(A, B, xmode, W.invm.p, b, xpre, W.r.p, C.rhs.p, C.e.p, h->Minv.p, gate, rs(), ex());
        } else {
            return cycle_tail(l, b, out, gate, br, xmode, xpre);
        }
        return cycle_post(l, b, out, gate, br, xmode, xpre, C.e.p, nullptr);
    }

    bool cycle_tail(int l, const double* b, double* out, const int* gate, const BetaReq* br, int xmode,
                    const double* xpre) {
        Level& L = *h->levels[l];
        LevelWs& W = ws->lev[l];
        const Csr A = L.csr();
        const Groups& B = L.groups();
        // r = b - A x ; r_c = restrict(r)
        if (l == 0) mark(0);
        launch_residual(A, B, xmode, W.invm.p, b, xpre, W.r.p, gate, ex());
        if (l == 0) mark(1);
        LevelWs& C = ws->lev[l + 1];
        const bool exact = (l + 1 == coarsest());
        const bool direct = !p.kcycle || p.inner_krylov_steps == 0 || exact;
        // the coarse flexible CG's ||r_c|| / gate[0] come out of the restriction
        const bool begun = !direct && !sing();
        // the tail kernel restricts, solves and returns the coarse correction
        const bool tail = ws->tail.on && l + 1 == ws->tail.Lt;
        if (!tail) {
            launch_restrict(L.nc, L.agg_ptr.p, L.members.p, L.mgroups(), W.r.p, C.rhs.p, gate, ex(),
                            begun ? ws->fcg.p + l + 1 : nullptr, rs());
            if (sing()) launch_project_mean(L.nc, C.rhs.p, ws->sums.p + 4 * l + 1, gate, rs(), ex());
        }
        const double* ec;
        const int* ec_valid = nullptr;
        if (tail) {
            double* o = direct ? C.e.p : C.xf.p;
            int* u0 = direct ? nullptr : &ws->fcg.p[l + 1].upd[0];
            // the tail also materialises this level's prolongated iterate, so
            // the post-sweep gathers one array (xmode 1, one post-sweep)
            const bool xm = xmode == 1 && p.post_sweeps == 1 && ws->tail.args.xn == L.n;
            launch_tail(ws->tail, W.r.p, gate, o, u0, s, xm ? b : nullptr, xm ? W.tA.p : nullptr);
            ec = o;
            ec_valid = u0;
            if (xm) {
                const BetaReq* fb = sing() ? nullptr : br;
                launch_sweep_vec(A, B, W.invm.p, b, W.tA.p, out, gate, ex(), fb, rs());
                return fb != nullptr;
            }
        } else if (direct) {
            cycle(l + 1, C.rhs.p, C.e.p, gate);
            ec = C.e.p;
        } else {
            // a small child FCG's last step also writes this level's
            // prolongated iterate (xmode 1), so the post-sweep gathers it
            ParentUp pu;
            const bool want = xmode == 1 && p.post_sweeps == 1 && !sing() && L.n < kTmaMinRows &&
                              !getenv("UAAMG_NO_PARENT_UP");
            if (want) {
                pu.n = L.n; pu.invm = W.invm.p; pu.b = b; pu.v2a = L.v2a.p;
                pu.valid = &ws->fcg.p[l + 1].upd[0]; pu.out = W.tA.p;
            }
            const bool xmat = fcg(l + 1, C.rhs.p, C.xf.p, gate, begun, want ? &pu : nullptr);
            if (xmat) {
                const BetaReq* fb = sing() ? nullptr : br;
                launch_sweep_vec(A, B, W.invm.p, b, W.tA.p, out, gate, ex(), fb, rs());
                return fb != nullptr;
            }
            ec = C.xf.p;
            ec_valid = &ws->fcg.p[l + 1].upd[0];
        }
        return cycle_post(l, b, out, gate, br, xmode, xpre, ec, ec_valid);
    }

    // prolongate + post-smoothing (the last sweep may carry the beta dot)
    bool cycle_post(int l, const double* b, double* out, const int* gate, const BetaReq* br, int xmode,
                    const double* xpre, const double* ec, const int* ec_valid) {
        Level& L = *h->levels[l];
        LevelWs& W = ws->lev[l];
        const Csr A = L.csr();
        const Groups& B = L.groups();
        const bool mat = L.n >= kTmaMinRows;
        const BetaReq* fb = sing() ? nullptr : br;
        if (p.post_sweeps == 0) {
            launch_prolongate(L.n, xmode, W.invm.p, b, xpre, L.v2a.p, ec, ec_valid, out, gate, ex());
            fb = nullptr;
        } else {
            double* other = (xpre == W.tA.p) ? W.tB.p : W.tA.p;
            double* dst = p.post_sweeps == 1 ? out : other;
            if (mat) {
                // x = xpre + e_c[v2a] into `other`, then a plain sweep
                launch_prolongate(L.n, xmode, W.invm.p, b, xpre, L.v2a.p, ec, ec_valid, other, gate, ex());
                if (l == 0) mark(2);
                launch_sweep_vec(A, B, W.invm.p, b, other, dst == other ? W.xup.p : dst, gate, ex(),
                                 p.post_sweeps == 1 ? fb : nullptr, rs());
                if (l == 0) mark(3);
                if (dst == other) dst = W.xup.p;
            } else {
                if (l == 0) mark(2);
                launch_sweep_up(A, B, xmode, W.invm.p, b, xpre, L.v2a.p, ec, ec_valid, dst, gate, ex(),
                                p.post_sweeps == 1 ? fb : nullptr, rs());
                if (l == 0) mark(3);
            }
            double* c2 = dst;
            for (int k = 1; k < p.post_sweeps; ++k) {
                double* nx = (k == p.post_sweeps - 1) ? out : ((c2 == W.tA.p) ? W.tB.p : W.tA.p);
                launch_sweep_vec(A, B, W.invm.p, b, c2, nx, gate, ex(), k == p.post_sweeps - 1 ? fb : nullptr, rs());
                c2 = nx;
            }
        }
        if (sing()) launch_project_mean(L.n, out, ws->sums.p + 4 * l + 3, gate, rs(), ex());
        return fb != nullptr;
    }

    // U/solvers.py:160-187
    // begun: ||b|| / gate[0] were produced by the caller's restriction
    // pu: the parent level's prolongated iterate, written by the last step
    // when that step is one cooperative kernel (returns whether it was)
    bool fcg(int l, const double* b, double* x, const int* parent_gate, bool begun = false,
             const ParentUp* pu = nullptr) {
        bool xmat = false;
        Level& L = *h->levels[l];
        LevelWs& W = ws->lev[l];
        FcgState* st = ws->fcg.p + l;
        if (!begun) launch_fcg_begin(L.n, b, parent_gate, st, rs(), ex());
        double* P[2] = {W.p0.p, W.p1.p};
        double* AP[2] = {W.ap0.p, W.ap1.p};
        for (int k = 0; k < p.inner_krylov_steps; ++k) {
            const int* g = &st->gate[k];
            const double* rin = (k == 0) ? b : W.rf.p;
            double* pc = P[k & 1];
            double* pp = P[(k + 1) & 1];
            double* apc = AP[k & 1];
            double* app = AP[(k + 1) & 1];
            const BetaReq br{app, &st->beta, &st->pap, nullptr};
            const bool fused = cycle(l, rin, W.z.p, g, k > 0 ? &br : nullptr);
            if (k > 0 && !fused) launch_beta(L.n, W.z.p, pp, app, &st->beta, g, nullptr, rs(), ex());
            if (!sing()) {
                const bool last = k == p.inner_krylov_steps - 1;
                xmat = launch_dir_update_fcg(L.csr(), L.groups(), W.z.p, pp, k > 0, rin, pc, apc, x, W.rf.p, st, k,
                                             rs(), ws->fpart.p, ws->fbar.p + 2 * l, ex(), last, last ? pu : nullptr);
            } else {
                launch_dir_fcg(L.csr(), L.groups(), W.z.p, pp, k > 0, rin, pc, apc, st, k, rs(), ex());
                launch_fcg_update(L.n, k, x, pc, rin, W.rf.p, apc, st, sing(), rs(), ex());
            }
        }
        return xmat;
    }

    // one NPCG iteration (U/solvers.py:221-254); parity selects p/p_prev roles
    void npcg_iteration(double* x, int parity) {
        Level& L = *h->levels[0];
        NpcgState* st = ws->npcg.p;
        const int* act = &st->active;
        double* P[2] = {ws->p0.p, ws->p1.p};
        double* AP[2] = {ws->ap0.p, ws->ap1.p};
        double* pc = P[parity];
        double* pp = P[parity ^ 1];
        double* apc = AP[parity];
        double* app = AP[parity ^ 1];
        const BetaReq br{app, &st->beta, &st->pap, &st->have_prev};
        const bool fused = cycle(0, ws->r.p, ws->z.p, act, sing() ? nullptr : &br);
        if (sing()) launch_project_mean(L.n, ws->z.p, &st->sum, act, rs(), s);
        if (!fused) launch_beta(L.n, ws->z.p, pp, app, &st->beta, act, &st->have_prev, rs(), s);
        mark(4);
        launch_dir_npcg(L.csr(), L.groups(), ws->z.p, pp, ws->r.p, pc, apc, st, rs(), s);
        mark(5);
        launch_npcg_update(L.n, x, pc, ws->r.p, apc, st, ws->hist.p, sing(), rs(), s);
    }
};

void ensure_ws(uaamg_hierarchy* h, const uaamg_solve_params& p, cudaStream_t s);
cudaStream_t library_stream();
// a fresh solve workspace; levels < mat_levels materialise the
// pre-smoothed / prolongated iterates; inner0: level 0 is itself reached by
// restriction (the replicated part of a sharded hierarchy)
std::unique_ptr<SolveWs> build_ws(uaamg_hierarchy* h, const uaamg_solve_params& p, cudaStream_t s, int mat_levels,
                                  bool inner0 = false);

// level 0 in the reference's host layout (U/sparse.py SparseMatrix)
struct HostCsr {
    const int64_t* rp;
    const int64_t* ci;
    const double* av;
};
uaamg_hierarchy* setup_impl(int n, long long nnz, const int* rp, const int* ci, const double* av,
                            const uaamg_setup_params& P, cudaStream_t s, int level_offset,
                            const HostCsr* hc = nullptr);

}  // namespace uaamg
