// shard.cu -- row-partitioned (multi-rank) NPCG / K-cycle solve.
//
// SURVEY.md §8e.  P ranks share one deterministic hierarchy (every rank
// builds the same bits, so it is replicated rather than communicated).  The
// levels with at least `shard_rows` rows are SHARDED by contiguous row
// ranges: level 0 in equal 128-aligned blocks, level l + 1 by seed ownership
// -- aggregates are numbered by ascending seed (U/aggregation.py:199-203),
// so the aggregates whose seed lies in rank q's rows of level l are a
// contiguous range of level l + 1.  Smaller levels are REPLICATED: every
// rank runs them whole with the single-device plan (no traffic at all).
//
// On a sharded level a rank computes only its own rows.  Its vectors are
// full-length buffers of which it owns one slice; a gather of column k reads
// buffer[owner(k)][k] -- a local load for owned columns and a peer-memory
// load for halo columns (SrcPeer; on an 8xB200 box the table holds the
// NVLink-mapped peer buffers, so the "halo exchange" is the gather itself,
// fused into the SpMV).  Restriction reads the members of the aggregates it
// produces the same way, in ascending member order (bit-exact); the last
// sharded level restricts into the replicated level in full on every rank.
// Dots publish each rank's total into every rank's slot array (xpublish)
// and k_xfin folds the P totals in rank order, so every rank holds the same
// scalars and takes the same gate decisions.
//
// This build runs the P ranks as VIRTUAL ranks on one device (their
// buffers all local, launched rank by rank in one stream, which orders the
// phases): the partition-invariance harness of SURVEY.md §4 item 3.  The
// peer tables, partitions and rank-ordered reductions are the multi-GPU
// code path; what a multi-process run adds is the mapping of peer buffers
// (cudaIpc handles) and a cross-device barrier between phases.
#include "launch.cuh"
#include "runtime.h"

namespace uaamg {

namespace {

constexpr int kSlotK = 2;  // max values per cross-rank reduction (Epi::K)

enum VRole { V_R, V_RHS, V_E, V_TA, V_TB, V_XUP, V_XF, V_RF, V_Z, V_P0, V_P1, V_AP0, V_AP1,
             T_R, T_Z, T_P0, T_P1, T_AP0, T_AP1, T_X, T_B };
struct VRef {
    int l;
    VRole v;
};
// gate: 0 none, 1 NPCG active, 2 FCG gate[step] of level l
struct GRef {
    int kind = 0;
    int l = 0, step = 0;
};

struct SLevel {
    bool sharded = false;
    Part part{};                 // rows of this level per rank
    std::vector<GroupBuf> gA;    // per rank: own rows of A
    std::vector<GroupBuf> gP;    // per rank: restriction rows (owned aggregates, or all of them)
};

struct Sharded {
    uaamg_hierarchy* h;
    uaamg_solve_params p;
    cudaStream_t s;
    int P;
    int rank = -1;          // -1: virtual ranks (all local); else this process's rank
    std::vector<int> mine;  // ranks computed by this process
    int Ls = 0;             // first replicated level
    std::vector<std::unique_ptr<SolveWs>> ws;  // [rank] (null for remote ranks)
    std::vector<SLevel> lv;
    std::vector<DBuf<double>> xr, br;  // per rank: iterate and right-hand side
    DBuf<double> slots;                // virtual: P x (kSlotK * P)
    DBuf<double*> slot_tab;            // P pointers: slot array of every rank
    // multi-process: every vector a peer may read lives in one cudaMalloc
    // arena per rank (same layout everywhere), exported by CUDA IPC
    char* arena = nullptr;
    size_t arena_bytes = 0;
    std::map<std::pair<int, int>, size_t> off;  // (level, role) -> arena offset
    size_t slots_off = 0, flags_off = 0;
    std::vector<char*> peer_base;               // arena base of every rank (own included)
    DBuf<unsigned*> flag_tab;                   // P pointers: barrier flag array of every rank
    unsigned epoch = 0;

    ~Sharded() {
        ws.clear();  // views into the arena go first
        for (int q = 0; q < (int)peer_base.size(); ++q)
            if (q != rank && peer_base[q]) cudaIpcCloseMemHandle(peer_base[q]);
        if (arena) cudaFree(arena);
    }

    Level& L(int l) const { return *h->levels[l]; }
    int a(int r, int l) const { return lv[l].part.b[r]; }
    int nrows(int r, int l) const { return lv[l].part.b[r + 1] - lv[l].part.b[r]; }
    RedScratch rs(int r) const { return RedScratch{ws[r]->partials.p, ws[r]->ticket.p}; }
    const double* slot(int r) const {
        return rank < 0 ? slots.p + (size_t)r * kSlotK * P : reinterpret_cast<const double*>(arena + slots_off);
    }
    // multi-process: cross-device barrier before an op reads what peers wrote
    void sync();

    double* ptr(int r, VRef x) const {
        if (rank >= 0 && r != rank) {
            auto it = off.find({x.v >= T_R ? -1 : x.l, (int)x.v});
            if (it == off.end()) throw Error(UAAMG_EINVAL, "vector is not shared across ranks");
            return reinterpret_cast<double*>(peer_base[r] + it->second);
        }
        SolveWs& W = *ws[r];
        switch (x.v) {
            case T_R: return W.r.p;
            case T_Z: return W.z.p;
            case T_P0: return W.p0.p;
            case T_P1: return W.p1.p;
            case T_AP0: return W.ap0.p;
            case T_AP1: return W.ap1.p;
            case T_X: return xr[r].p;
            case T_B: return br[r].p;
            default: break;
        }
        LevelWs& V = W.lev[x.l];
        switch (x.v) {
            case V_R: return V.r.p;
            case V_RHS: return V.rhs.p;
            case V_E: return V.e.p;
            case V_TA: return V.tA.p;
            case V_TB: return V.tB.p;
            case V_XUP: return V.xup.p;
            case V_XF: return V.xf.p;
            case V_RF: return V.rf.p;
            case V_Z: return V.z.p;
            case V_P0: return V.p0.p;
            case V_P1: return V.p1.p;
            case V_AP0: return V.ap0.p;
            case V_AP1: return V.ap1.p;
            default: break;
        }
        throw Error(UAAMG_EINVAL, "bad vector role");
    }
    const int* gptr(int r, GRef g) const {
        if (g.kind == 1) return &ws[r]->npcg.p->active;
        if (g.kind == 2) return &ws[r]->fcg.p[g.l].gate[g.step];
        return nullptr;
    }
    FcgState* fst(int r, int l) const { return ws[r]->fcg.p + l; }
    NpcgState* nst(int r) const { return ws[r]->npcg.p; }

    // gather of vector x on level l (partitioned like level l's rows)
    SrcPeer peer(VRef x, int l) const {
        SrcPeer sp{};
        sp.pt = lv[l].part;
        for (int q = 0; q < P; ++q) sp.tab[q] = ptr(q, x);
        return sp;
    }
    template <int K>
    void xred(RedSlot<K>& red, int r) const {
        red.xslot = slot_tab.p;
        red.xP = P;
        red.xrank = r;
    }
    Csr csr(int l) const { return L(l).csr(); }

    // ------------------------------------------------------------ sharded cycle
    // U/solvers.py:128-157 on a sharded level; returns whether the beta dot
    // of the consuming flexible CG was fused into the last sweep
    bool cycle(int l, VRef b, VRef out, GRef g, const VRef* apprev, int beta_state /*0 npcg, 1 fcg l*/);
    void fcg(int l, VRef b, VRef x, GRef parent, bool begun);
    void npcg_iteration(int parity);
};

bool Sharded::cycle(int l, VRef b, VRef out, GRef g, const VRef* apprev, int beta_state) {
    Level& Lv = L(l);
    const Csr A = csr(l);
    const int xmode = p.pre_sweeps == 0 ? 0 : 2;
    // pre-smoothing from a zero guess, materialised (x = 0 + inv_m b, then sweeps)
    VRef cur{l, V_TA};
    if (xmode == 2) {
        sync();
        for (int r : mine) {
            BodyXpre1 body{};
            const int o = a(r, l);
            body.invm = ws[r]->lev[l].invm.p + o;
            body.b = ptr(r, b) + o;
            body.x = ptr(r, cur) + o;
            body.g = gptr(r, g);
            run_map(nrows(r, l), body, s);
        }
        for (int k = 1; k < p.pre_sweeps; ++k) {
            VRef nx{l, cur.v == V_TA ? V_TB : V_TA};
            sync();
            for (int r : mine) {
                EpiSweep e{};
                e.invm = ws[r]->lev[l].invm.p; e.b = ptr(r, b); e.out = ptr(r, nx); e.g = gptr(r, g);
                run_stream<SrcPeer, EpiSweep, false>(A, lv[l].gA[r].g, peer(cur, l), e, s);
            }
            cur = nx;
        }
    }
    // r = b - A x
    sync();
    for (int r : mine) {
        EpiResid e{};
        e.b = ptr(r, b); e.r = ptr(r, VRef{l, V_R}); e.g = gptr(r, g);
        if (xmode == 0) run_stream<SrcZero, EpiResid, false>(A, lv[l].gA[r].g, SrcZero{}, e, s);
        else run_stream<SrcPeer, EpiResid, false>(A, lv[l].gA[r].g, peer(cur, l), e, s);
    }
    // r_c = restrict(r): members gathered from their owners, ascending order
    const int lc = l + 1;
    const bool csh = lv[lc].sharded;
    const bool exact = (lc == (int)h->levels.size() - 1);
    const bool direct = !p.kcycle || p.inner_krylov_steps == 0 || exact;
    const bool begun = !direct;
    Csr Pm;
    Pm.n = Lv.nc; Pm.rp = Lv.agg_ptr.p; Pm.ci = Lv.members.p; Pm.av = nullptr;
    sync();
    for (int r : mine) {
        if (begun) {
            EpiRestrictBegin e{};
            e.y = ws[r]->lev[lc].rhs.p; e.g = gptr(r, g); e.st = fst(r, lc);
            e.red = {rs(r).partials, rs(r).ticket};
            if (csh) xred(e.red, r);
            run_stream<SrcPeer, EpiRestrictBegin, true>(Pm, lv[l].gP[r].g, peer(VRef{l, V_R}, l), e, s);
        } else {
            EpiStoreG e{};
            e.y = ws[r]->lev[lc].rhs.p; e.g = gptr(r, g);
            run_stream<SrcPeer, EpiStoreG, true>(Pm, lv[l].gP[r].g, peer(VRef{l, V_R}, l), e, s);
        }
    }
    if (begun && csh) sync();
    if (begun && csh)
        for (int r : mine) {
            EpiRestrictBegin e{};
            e.st = fst(r, lc);
            e.g = gptr(r, g);
            run_xfin(e, slot(r), P, s);
        }
    // coarse correction
    VRef ec{lc, direct ? V_E : V_XF};
    if (csh) {
        if (direct) cycle(lc, VRef{lc, V_RHS}, ec, g, nullptr, 0);
        else fcg(lc, VRef{lc, V_RHS}, ec, g, true);
    } else {
        sync();
        for (int r : mine) {
            Plan pl{h, ws[r].get(), p, s};
            LevelWs& C = ws[r]->lev[lc];
            if (direct) pl.cycle(lc, C.rhs.p, C.e.p, gptr(r, g));
            else pl.fcg(lc, C.rhs.p, C.xf.p, gptr(r, g), true);
        }
    }
    // prolongation on own rows into tB (or tA if the pre-iterate lives in tB)
    VRef other{l, cur.v == V_TA ? V_TB : V_TA};
    sync();
    for (int r : mine) {
        const int o = a(r, l);
        BodyProlPeer body{};
        body.mode = xmode;
        body.xpre = ptr(r, cur) + o;
        body.v2a = Lv.v2a.p + o;
        body.pt = csh ? lv[lc].part : Part{1, {0, L(lc).n}};
        for (int q = 0; q < P; ++q) body.ec[q] = csh ? ptr(q, ec) : ptr(r, ec);
        body.ec_valid = direct ? nullptr : &fst(r, lc)->upd[0];
        body.out = ptr(r, other) + o;
        body.g = gptr(r, g);
        run_map(nrows(r, l), body, s);
    }
    // post-smoothing sweeps; the last may carry the consuming CG's beta dot
    if (p.post_sweeps == 0) {
        sync();
        for (int r : mine) {
            const int o = a(r, l);
            UA_CK(cudaMemcpyAsync(ptr(r, out) + o, ptr(r, other) + o, sizeof(double) * nrows(r, l),
                                  cudaMemcpyDeviceToDevice, s));
        }
        return false;
    }
    VRef src = other;
    for (int k = 0; k < p.post_sweeps; ++k) {
        const bool last = (k == p.post_sweeps - 1);
        VRef dst = last ? out : VRef{l, src.v == V_XUP ? V_TA : V_XUP};
        sync();
        for (int r : mine) {
            if (last && apprev) {
                EpiSweepBeta e{};
                e.invm = ws[r]->lev[l].invm.p; e.b = ptr(r, b); e.out = ptr(r, dst); e.g = gptr(r, g);
                e.apprev = ptr(r, *apprev);
                if (beta_state == 0) {
                    e.beta = &nst(r)->beta; e.pap = &nst(r)->pap; e.have = &nst(r)->have_prev;
                } else {
                    e.beta = &fst(r, l)->beta; e.pap = &fst(r, l)->pap; e.have = nullptr;
                }
                e.red = {rs(r).partials, rs(r).ticket};
                xred(e.red, r);
                run_stream<SrcPeer, EpiSweepBeta, false>(A, lv[l].gA[r].g, peer(src, l), e, s);
            } else {
                EpiSweep e{};
                e.invm = ws[r]->lev[l].invm.p; e.b = ptr(r, b); e.out = ptr(r, dst); e.g = gptr(r, g);
                run_stream<SrcPeer, EpiSweep, false>(A, lv[l].gA[r].g, peer(src, l), e, s);
            }
        }
        src = dst;
    }
    if (apprev) sync();
    if (apprev)
        for (int r : mine) {
            EpiSweepBeta e{};
            if (beta_state == 0) {
                e.beta = &nst(r)->beta; e.pap = &nst(r)->pap; e.have = &nst(r)->have_prev;
            } else {
                e.beta = &fst(r, l)->beta; e.pap = &fst(r, l)->pap; e.have = nullptr;
            }
            e.g = gptr(r, g);
            run_xfin(e, slot(r), P, s);
        }
    return apprev != nullptr;
}

// U/solvers.py:160-187 on a sharded level (begun: ||b|| came from the restriction)
void Sharded::fcg(int l, VRef b, VRef x, GRef parent, bool begun) {
    if (!begun) {
        sync();
        for (int r : mine) {
            BodyFcgBegin body{};
            const int o = a(r, l);
            body.b = ptr(r, b) + o; body.pg = gptr(r, parent); body.st = fst(r, l);
            body.red = {rs(r).partials, rs(r).ticket};
            xred(body.red, r);
            run_map(nrows(r, l), body, s);
        }
        sync();
        for (int r : mine) {
            BodyFcgBegin body{};
            body.st = fst(r, l);
            body.pg = gptr(r, parent);
            run_xfin(body, slot(r), P, s);
        }
    }
    const Csr A = csr(l);
    const VRole PR[2] = {V_P0, V_P1}, APR[2] = {V_AP0, V_AP1};
    for (int k = 0; k < p.inner_krylov_steps; ++k) {
        GRef g{2, l, k};
        VRef rin = (k == 0) ? b : VRef{l, V_RF};
        VRef pc{l, PR[k & 1]}, pp{l, PR[(k + 1) & 1]}, apc{l, APR[k & 1]}, app{l, APR[(k + 1) & 1]};
        cycle(l, rin, VRef{l, V_Z}, g, k > 0 ? &app : nullptr, 1);
        // p = z + beta p_prev on own rows, then Ap (+ p.Ap, p.r)
        sync();
        for (int r : mine) {
            const int o = a(r, l);
            BodyDirP bp{};
            bp.src.z = ws[r]->lev[l].z.p + o; bp.src.pprev = ptr(r, pp) + o; bp.src.beta_p = &fst(r, l)->beta;
            bp.src.have_p = nullptr; bp.src.have_static = k > 0;
            bp.p = ptr(r, pc) + o; bp.g = gptr(r, g);
            run_map(nrows(r, l), bp, s);
        }
        sync();
        for (int r : mine) {
            EpiDirFcg e{};
            e.p = nullptr; e.ap = ptr(r, apc); e.r = ptr(r, rin); e.st = fst(r, l); e.step = k;
            e.red = {rs(r).partials, rs(r).ticket};
            xred(e.red, r);
            run_stream<SrcPeer, EpiDirFcg, false>(A, lv[l].gA[r].g, peer(pc, l), e, s);
        }
        sync();
        for (int r : mine) {
            EpiDirFcg e{};
            e.st = fst(r, l); e.step = k;
            run_xfin(e, slot(r), P, s);
        }
        sync();
        for (int r : mine) {
            const int o = a(r, l);
            BodyFcgUpd body{};
            body.step = k; body.x = ptr(r, x) + o; body.p = ptr(r, pc) + o; body.rin = ptr(r, rin) + o;
            body.rout = ws[r]->lev[l].rf.p + o; body.ap = ptr(r, apc) + o; body.st = fst(r, l); body.singular = 0;
            body.red = {rs(r).partials, rs(r).ticket};
            xred(body.red, r);
            run_map(nrows(r, l), body, s);
        }
        sync();
        for (int r : mine) {
            BodyFcgUpd body{};
            body.step = k; body.st = fst(r, l); body.singular = 0;
            run_xfin(body, slot(r), P, s);
        }
    }
}

// one NPCG iteration (U/solvers.py:221-254) on sharded level 0
void Sharded::npcg_iteration(int parity) {
    const VRole PR[2] = {T_P0, T_P1}, APR[2] = {T_AP0, T_AP1};
    VRef pc{0, PR[parity]}, pp{0, PR[parity ^ 1]}, apc{0, APR[parity]}, app{0, APR[parity ^ 1]};
    GRef act{1, 0, 0};
    cycle(0, VRef{0, T_R}, VRef{0, T_Z}, act, &app, 0);
    const Csr A = csr(0);
    sync();
    for (int r : mine) {
        const int o = a(r, 0);
        BodyDirP bp{};
        bp.src.z = ws[r]->z.p + o; bp.src.pprev = ptr(r, pp) + o; bp.src.beta_p = &nst(r)->beta;
        bp.src.have_p = &nst(r)->have_prev;
        bp.p = ptr(r, pc) + o; bp.g = gptr(r, act);
        run_map(nrows(r, 0), bp, s);
    }
    sync();
    for (int r : mine) {
        EpiDirNpcg e{};
        e.p = nullptr; e.ap = ptr(r, apc); e.r = ws[r]->r.p; e.st = nst(r);
        e.red = {rs(r).partials, rs(r).ticket};
        xred(e.red, r);
        run_stream<SrcPeer, EpiDirNpcg, false>(A, lv[0].gA[r].g, peer(pc, 0), e, s);
    }
    sync();
    for (int r : mine) {
        EpiDirNpcg e{};
        e.st = nst(r);
        run_xfin(e, slot(r), P, s);
    }
    sync();
    for (int r : mine) {
        const int o = a(r, 0);
        BodyNpcgUpd body{};
        body.x = xr[r].p + o; body.p = ptr(r, pc) + o; body.r = ws[r]->r.p + o; body.ap = ptr(r, apc) + o;
        body.st = nst(r); body.hist = ws[r]->hist.p; body.singular = 0;
        body.red = {rs(r).partials, rs(r).ticket};
        xred(body.red, r);
        run_map(nrows(r, 0), body, s);
    }
    sync();
    for (int r : mine) {
        BodyNpcgUpd body{};
        body.st = nst(r); body.hist = ws[r]->hist.p; body.singular = 0;
        run_xfin(body, slot(r), P, s);
    }
}

__global__ void k_set_npcg_sh(NpcgState* st, double tol, int max_iters) {
    st->host_active = nullptr;
    st->tol = tol;
    st->max_iters = max_iters;
}

// contiguous row ranges: level 0 in equal 128-row-aligned blocks
Part level0_part(int n, int P) {
    Part pt{};
    pt.P = P;
    for (int q = 0; q <= P; ++q) {
        long long v = (long long)n * q / P;
        if (q > 0 && q < P) v = std::min<long long>(n, (v + 127) / 128 * 128);
        pt.b[q] = (int)v;
    }
    for (int q = 1; q <= P; ++q) pt.b[q] = std::max(pt.b[q], pt.b[q - 1]);
    pt.b[P] = n;
    return pt;
}

// aggregates are numbered by ascending seed: rank q's coarse rows are the
// aggregates whose seed lies in its fine rows
void coarse_part(const int* seeds, int nc, const int* fine, int P, int* out) {
    for (int q = 0; q <= P; ++q) out[q] = (int)(std::lower_bound(seeds, seeds + nc, fine[q]) - seeds);
    out[P] = nc;
}

// cross-device barrier: publish `epoch` into every rank's flag line, then
// wait until every rank has published it into ours
__global__ void k_dist_barrier(unsigned* const* flags, int P, int rank, unsigned epoch) {
    __threadfence_system();  // this rank's earlier writes (own and peer) first
    for (int q = 0; q < P; ++q) *(volatile unsigned*)(flags[q] + 32 * rank) = epoch;
    __threadfence_system();
    const volatile unsigned* mine = flags[rank];
    const long long t0 = clock64();
    for (int q = 0; q < P; ++q)
        while ((int)(mine[32 * q] - epoch) < 0) {
            __nanosleep(64);
            if (clock64() - t0 > (1ll << 36)) __trap();  // a rank died: fail loudly
        }
    __threadfence_system();
}

void Sharded::sync() {
    if (rank < 0) return;  // virtual ranks: stream order already orders the phases
    ++epoch;
    UA_LAUNCH(k_dist_barrier, 1, 1, 0, s, flag_tab.p, P, rank, epoch);
}

// partitions, workspaces, work-unit groups of the ranks this process runs
std::unique_ptr<Sharded> sharded_build(uaamg_hierarchy* h, const uaamg_solve_params& p, int P, int rank,
                                       long long shard_rows, cudaStream_t s) {
    if (P < 1 || P > kMaxRanks) throw Error(UAAMG_EINVAL, "ranks must be in [1, 8]");
    if (rank >= P) throw Error(UAAMG_EINVAL, "rank out of range");
    if (h->singular) throw Error(UAAMG_EUNSUPPORTED, "sharded solve of a singular (Neumann) hierarchy");
    if (!(p.tol > 0)) throw Error(UAAMG_EINVAL, "tol must be positive");
    const int nl = (int)h->levels.size();
    std::unique_ptr<Sharded> Sp(new Sharded{h, p, s, P});
    Sharded& S = *Sp;
    S.rank = rank;
    if (rank < 0) for (int q = 0; q < P; ++q) S.mine.push_back(q);
    else S.mine.push_back(rank);
    // sharded levels: level 0 always (when it has coarser levels), then every
    // level with >= shard_rows rows, never the coarsest
    S.Ls = 0;
    while (S.Ls < nl - 1 && (S.Ls == 0 || h->levels[S.Ls]->n >= shard_rows)) ++S.Ls;
    if (S.Ls == 0) throw Error(UAAMG_EUNSUPPORTED, "sharded solve needs at least two levels");
    S.lv.resize(nl);
    S.ws.resize(P);
    for (int r : S.mine) S.ws[r] = build_ws(h, p, s, S.Ls);
    S.lv[0].part = level0_part(h->levels[0]->n, P);
    for (int l = 0; l < S.Ls; ++l) {
        S.lv[l].sharded = true;
        Level& Lv = *h->levels[l];
        std::vector<int> seeds(Lv.nc);
        UA_CK(cudaMemcpyAsync(seeds.data(), Lv.seeds.p, sizeof(int) * Lv.nc, cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        Part cp{};
        cp.P = P;
        coarse_part(seeds.data(), Lv.nc, S.lv[l].part.b, P, cp.b);
        if (l + 1 < S.Ls) S.lv[l + 1].part = cp;
        S.lv[l].gA.resize(P);
        S.lv[l].gP.resize(P);
        for (int r : S.mine) {
            const int a = S.lv[l].part.b[r], n = S.lv[l].part.b[r + 1] - a;
            build_groups(n, Lv.rp.p, kSolveLongMin, S.lv[l].gA[r], s, a);
            if (n >= kTmaMinRows / P && S.lv[l].gA[r].g.np == 0) {
                const int cap = max_tile_nnz(n, Lv.rp.p, s, a);
                if (cap <= kTmaMaxCap) S.lv[l].gA[r].g.tma_cap = std::max(cap, 4);
            }
            // restriction rows: this rank's aggregates (coarse level sharded)
            // or all of them (coarse level replicated)
            const int ca = (l + 1 < S.Ls) ? cp.b[r] : 0;
            const int cn = (l + 1 < S.Ls) ? cp.b[r + 1] - cp.b[r] : Lv.nc;
            build_groups(cn, Lv.agg_ptr.p, kSolveLongMin, S.lv[l].gP[r], s, ca);
        }
    }
    const int n = h->levels[0]->n;
    S.xr.resize(P);
    S.br.resize(P);
    for (int r : S.mine) {
        S.xr[r].alloc(n, s);
        S.br[r].alloc(n, s);
    }
    S.slot_tab.alloc(P, s);
    if (rank < 0) {
        S.slots.alloc((size_t)P * kSlotK * P, s);
        std::vector<double*> tab(P);
        for (int q = 0; q < P; ++q) tab[q] = S.slots.p + (size_t)q * kSlotK * P;
        UA_CK(cudaMemcpyAsync(S.slot_tab.p, tab.data(), sizeof(double*) * P, cudaMemcpyHostToDevice, s));
        UA_CK(cudaStreamSynchronize(s));
        return Sp;
    }
    // multi-process: move every peer-readable vector into one arena
    SolveWs& W = *S.ws[rank];
    std::vector<std::pair<std::pair<int, int>, DBuf<double>*>> shared;
    for (int l = 0; l < S.Ls; ++l) {
        LevelWs& V = W.lev[l];
        const std::pair<VRole, DBuf<double>*> roles[] = {{V_R, &V.r},   {V_TA, &V.tA},  {V_TB, &V.tB},
                                                         {V_XUP, &V.xup}, {V_E, &V.e},  {V_XF, &V.xf},
                                                         {V_P0, &V.p0}, {V_P1, &V.p1}};
        for (auto& rb : roles)
            if (rb.second->p) shared.push_back({{l, (int)rb.first}, rb.second});
    }
    shared.push_back({{-1, (int)T_P0}, &W.p0});
    shared.push_back({{-1, (int)T_P1}, &W.p1});
    shared.push_back({{-1, (int)T_X}, &S.xr[rank]});
    size_t bytes = 0;
    auto take = [&](size_t b) {
        const size_t o = bytes;
        bytes += (b + 64 + 255) & ~(size_t)255;
        return o;
    };
    for (auto& e : shared) S.off[e.first] = take(e.second->n * sizeof(double));
    S.slots_off = take(sizeof(double) * kSlotK * P);
    S.flags_off = take(sizeof(unsigned) * 32 * P);
    S.arena_bytes = bytes;
    UA_CK(cudaStreamSynchronize(s));
    UA_CK(cudaMalloc(&S.arena, bytes));
    UA_CK(cudaMemset(S.arena, 0, bytes));
    for (auto& e : shared) e.second->adopt_view(reinterpret_cast<double*>(S.arena + S.off[e.first]), e.second->n);
    return Sp;
}

// initial residual, the NPCG loop (U/solvers.py:202-255), x assembled from
// the owners' slices
void sharded_run(Sharded& S, const double* b, const double* x0, double* x, double* hist_host,
                 uaamg_solve_result* res) {
    uaamg_hierarchy* h = S.h;
    const uaamg_solve_params& p = S.p;
    cudaStream_t s = S.s;
    const int P = S.P;
    const int n = h->levels[0]->n;
    const int me = S.mine[0];
    for (int r : S.mine) UA_CK(cudaMemcpyAsync(S.br[r].p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    cudaEvent_t e0, e1;
    UA_CK(cudaEventCreate(&e0));
    UA_CK(cudaEventCreate(&e1));
    UA_CK(cudaEventRecord(e0, s));
    const Csr A = h->levels[0]->csr();
    for (int r : S.mine) {
        if (x0) UA_CK(cudaMemcpyAsync(S.xr[r].p, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        else UA_CK(cudaMemsetAsync(S.xr[r].p, 0, sizeof(double) * n, s));
    }
    S.sync();
    for (int r : S.mine) {
        EpiResid e{};
        e.b = S.br[r].p; e.r = S.ws[r]->r.p; e.g = nullptr;
        if (x0) run_stream<SrcPeer, EpiResid, false>(A, S.lv[0].gA[r].g, S.peer(VRef{0, T_X}, 0), e, s);
        else run_stream<SrcZero, EpiResid, false>(A, S.lv[0].gA[r].g, SrcZero{}, e, s);
        UA_LAUNCH(k_set_npcg_sh, 1, 1, 0, s, S.nst(r), p.tol, p.max_iters);
    }
    S.sync();
    for (int r : S.mine) {
        const int o = S.a(r, 0);
        BodyNpcgInit body{};
        body.b = S.br[r].p + o; body.r = S.ws[r]->r.p + o; body.st = S.nst(r); body.hist = S.ws[r]->hist.p;
        body.red = {S.rs(r).partials, S.rs(r).ticket};
        S.xred(body.red, r);
        run_map(S.nrows(r, 0), body, s);
    }
    S.sync();
    for (int r : S.mine) {
        BodyNpcgInit body{};
        body.st = S.nst(r); body.hist = S.ws[r]->hist.p;
        run_xfin(body, S.slot(r), P, s);
    }
    NpcgState hst{};
    UA_CK(cudaMemcpyAsync(&hst, S.nst(me), sizeof(NpcgState), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    for (int it = 0; hst.active && it < p.max_iters; ++it) {
        S.npcg_iteration(it & 1);
        UA_CK(cudaMemcpyAsync(&hst, S.nst(me), sizeof(NpcgState), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
    }
    UA_CK(cudaEventRecord(e1, s));
    // assemble x from the owners' slices (peer reads in multi-process mode)
    S.sync();
    for (int q = 0; q < P; ++q) {
        const int o = S.a(q, 0);
        const double* src = S.rank < 0 || q == S.rank ? S.xr[q].p : S.ptr(q, VRef{0, T_X});
        UA_CK(cudaMemcpyAsync(x + o, src + o, sizeof(double) * S.nrows(q, 0), cudaMemcpyDefault, s));
    }
    S.sync();  // peers may not free their iterate before everyone copied it
    UA_CK(cudaMemcpyAsync(&hst, S.nst(me), sizeof(NpcgState), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    float ms = 0;
    UA_CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    res->iterations = hst.iters;
    res->solve_seconds = ms * 1e-3;
    if (hist_host)
        UA_CK(cudaMemcpy(hist_host, S.ws[me]->hist.p, sizeof(double) * (hst.iters + 1), cudaMemcpyDeviceToHost));
    res->converged = (hst.bnorm == 0.0) ? 1 : (hst.last_rel <= p.tol);
    res->status = 0;
    if (hst.status == 1) {
        res->converged = 0;
        res->status = UAAMG_ENUMERICAL;
        throw Error(UAAMG_ENUMERICAL, "conjugate-gradient breakdown (sharded solve)");
    }
}

}  // namespace

}  // namespace uaamg

using namespace uaamg;

struct uaamg_dist {
    std::unique_ptr<uaamg::Sharded> S;
};

#define UA_TRY(...)                                                                                \
    try {                                                                                          \
        __VA_ARGS__;                                                                               \
        const cudaError_t pe = cudaGetLastError();                                                 \
        if (pe != cudaSuccess) throw Error(UAAMG_ECUDA, std::string("pending CUDA error: ") + cudaGetErrorString(pe)); \
        return UAAMG_OK;                                                                           \
    } catch (const Error& e) {                                                                     \
        g_last_error = e.what();                                                                   \
        return e.code;                                                                             \
    } catch (const std::exception& e) {                                                            \
        g_last_error = e.what();                                                                   \
        return UAAMG_ECUDA;                                                                        \
    }

// host-only entry points: no CUDA runtime call (usable without a GPU)
#define UA_HOST_TRY(...)               \
    try {                              \
        __VA_ARGS__;                   \
        return UAAMG_OK;               \
    } catch (const Error& e) {         \
        g_last_error = e.what();       \
        return e.code;                 \
    }

extern "C" {

int uaamg_npcg_solve_sharded(uaamg_hierarchy* h, const uaamg_solve_params* p, int nranks, int64_t shard_rows,
                             const double* b, const double* x0, double* x, double* history_host,
                             uaamg_solve_result* res, void* stream) {
    UA_TRY({
        std::memset(res, 0, sizeof(*res));
        std::lock_guard<std::mutex> lk(h->mu);
        StreamJoin join((cudaStream_t)stream, h->stream);
        auto S = sharded_build(h, *p, nranks, -1, shard_rows, h->stream);
        sharded_run(*S, b, x0, x, history_host, res);
    })
}

int uaamg_dist_create(uaamg_hierarchy* h, const uaamg_solve_params* p, int rank, int nranks, int64_t shard_rows,
                      uaamg_dist** out) {
    UA_TRY({
        if (rank < 0) throw Error(UAAMG_EINVAL, "rank must be >= 0");
        auto d = std::make_unique<uaamg_dist>();
        d->S = sharded_build(h, *p, nranks, rank, shard_rows, h->stream);
        *out = d.release();
    })
}

int uaamg_dist_handle(uaamg_dist* d, void* handle) {
    UA_TRY({
        cudaIpcMemHandle_t hd;
        UA_CK(cudaIpcGetMemHandle(&hd, d->S->arena));
        std::memcpy(handle, &hd, sizeof(hd));
    })
}

int uaamg_dist_connect(uaamg_dist* d, const void* handles) {
    UA_TRY({
        Sharded& S = *d->S;
        S.peer_base.assign(S.P, nullptr);
        const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
        for (int q = 0; q < S.P; ++q) {
            if (q == S.rank) {
                S.peer_base[q] = S.arena;
                continue;
            }
            void* ptr = nullptr;
            UA_CK(cudaIpcOpenMemHandle(&ptr, hs[q], cudaIpcMemLazyEnablePeerAccess));
            S.peer_base[q] = static_cast<char*>(ptr);
        }
        std::vector<double*> st(S.P);
        std::vector<unsigned*> fl(S.P);
        for (int q = 0; q < S.P; ++q) {
            st[q] = reinterpret_cast<double*>(S.peer_base[q] + S.slots_off);
            fl[q] = reinterpret_cast<unsigned*>(S.peer_base[q] + S.flags_off);
        }
        S.flag_tab.alloc(S.P, S.s);
        UA_CK(cudaMemcpyAsync(S.slot_tab.p, st.data(), sizeof(double*) * S.P, cudaMemcpyHostToDevice, S.s));
        UA_CK(cudaMemcpyAsync(S.flag_tab.p, fl.data(), sizeof(unsigned*) * S.P, cudaMemcpyHostToDevice, S.s));
        UA_CK(cudaStreamSynchronize(S.s));
    })
}

int uaamg_dist_solve(uaamg_dist* d, const double* b, const double* x0, double* x, double* history_host,
                     uaamg_solve_result* res, void* stream) {
    UA_TRY({
        Sharded& S = *d->S;
        if (S.peer_base.empty()) throw Error(UAAMG_EINVAL, "uaamg_dist_connect has not run");
        std::memset(res, 0, sizeof(*res));
        std::lock_guard<std::mutex> lk(S.h->mu);
        StreamJoin join((cudaStream_t)stream, S.h->stream);
        sharded_run(S, b, x0, x, history_host, res);
    })
}

void uaamg_dist_free(uaamg_dist* d) { delete d; }

int uaamg_partition_rows(int n, int nranks, int* bounds) {
    UA_HOST_TRY({
        if (nranks < 1 || nranks > kMaxRanks) throw Error(UAAMG_EINVAL, "ranks must be in [1, 8]");
        const Part pt = level0_part(n, nranks);
        for (int q = 0; q <= nranks; ++q) bounds[q] = pt.b[q];
    })
}

int uaamg_partition_coarse(const int* seeds, int nc, const int* fine_bounds, int nranks, int* bounds) {
    UA_HOST_TRY({
        if (nranks < 1 || nranks > kMaxRanks) throw Error(UAAMG_EINVAL, "ranks must be in [1, 8]");
        coarse_part(seeds, nc, fine_bounds, nranks, bounds);
    })
}

}  // extern "C"
