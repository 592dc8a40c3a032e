// dist_solve.cu -- row-partitioned NPCG / K-cycle solve on a DistHier
// (U/solvers.py:128-255).
//
// On a sharded level a rank computes only its own rows; its vectors hold
// only its rows (arena blocks, peer-readable).  A gather of column k reads
// vec[owner(k)][k] -- local for own columns, a peer load for halo columns
// (SrcPeer), so the halo exchange is the SpMV's gather itself.  Restriction
// reads its aggregates' members from their owners in ascending member order
// (bit-exact); prolongation reads e_c of each row's aggregate from the
// aggregate's owner.  The last sharded level restricts into the whole
// replicated level on every rank, which then runs the single-device plan
// (Plan, runtime.h) -- its tail kernel included -- and prolongs back.
// Dot products: each rank publishes its total into every rank's slot array
// (xpublish), k_xfin folds the P totals in rank order, so all ranks hold
// the same bits and take the same branches.  Ranks are ordered by
// Comm::barrier between phases that read what peers wrote.
#include <cstring>

#include "dist.h"

namespace uaamg {

namespace {

enum VRole { V_R, V_RHS, V_E, V_TA, V_TB, V_XUP, V_XF, V_RF, V_Z, V_P0, V_P1, V_AP0, V_AP1, V_INVM, V_BP, kRoles };
// outer (level-0 NPCG) vectors
enum TRole { T_R, T_Z, T_P0, T_P1, T_AP0, T_AP1, T_X, T_B, kTRoles };
struct VRef {
    int l;     // level (-1: outer vector)
    int v;     // VRole or TRole
};
inline VRef O(TRole t) { return VRef{-1, (int)t}; }
inline VRef Lv(int l, VRole v) { return VRef{l, (int)v}; }

// gate: 0 none, 1 NPCG active, 2 FCG gate[step] of level l
struct GRef {
    int kind = 0;
    int l = 0, step = 0;
};

struct RankWs {
    std::vector<GroupBuf> gA, gP;           // per sharded level: own rows, restriction rows
    DBuf<FcgState> fcg;                     // per sharded level
    DBuf<NpcgState> npcg;
    DBuf<double> partials, hist;
    DBuf<unsigned> ticket;
    DBuf<int> bad_row;
    DBuf<double> sums;                      // singular: 4 scratch sums per level (+ 4 spare)
    DBuf<int> err;                          // singular: incompatible right-hand side at a coarse level
    double* slots = nullptr;                // arena: kSlotK * P (peers publish into it)
    std::unique_ptr<SolveWs> rws;           // replicated levels
};

}  // namespace

struct DistSolve {
    DistHier& H;
    Comm& C;
    uaamg_solve_params p;
    cudaStream_t s;
    int P;
    int Ls;
    std::vector<size_t> marks;  // arena persistent bump before this workspace (per rank)
    std::vector<RankWs> ws;                                  // [P] (mine only)
    // vec[role][level][rank]: unshifted local block pointers (all ranks after the exchange)
    std::vector<std::vector<std::vector<double*>>> vec;      // [kRoles][Ls][P]
    std::vector<std::vector<double*>> outer;                 // [kTRoles][P]
    DBuf<double*> slot_tab_v;                                // virtual: per rank slot table
    std::vector<DBuf<double*>> slot_tab;                     // [P] (mine): every rank's slot array

    const DLevel& L(int l) const { return H.lv[l]; }
    const DRank& R(int l, int r) const { return H.lv[l].r[r]; }
    int a(int r, int l) const { return H.lv[l].pt.b[r]; }
    int nrows(int r, int l) const { return H.lv[l].pt.b[r + 1] - H.lv[l].pt.b[r]; }
    RedScratch rs(int r) const { return RedScratch{ws[r].partials.p, ws[r].ticket.p}; }

    double* ptr(int r, VRef x) const { return x.l < 0 ? outer[x.v][r] : vec[x.v][x.l][r]; }
    // global-row-indexed view of rank r's block of x (level l rows)
    double* sh(int r, VRef x) const {
        const int l = x.l < 0 ? 0 : x.l;
        return ptr(r, x) - a(r, l);
    }
    const int* gptr(int r, GRef g) const {
        if (g.kind == 1) return &ws[r].npcg.p->active;
        if (g.kind == 2) return &ws[r].fcg.p[g.l].gate[g.step];
        return nullptr;
    }
    FcgState* fst(int r, int l) const { return ws[r].fcg.p + l; }
    NpcgState* nst(int r) const { return ws[r].npcg.p; }
    // the replicated hierarchy's plan on rank r
    Plan plan(int r) const { return Plan{H.rep.get(), ws[r].rws.get(), p, s}; }

    SrcPeer peer(VRef x, int l) const {
        SrcPeer sp{};
        sp.pt = L(l).pt;
        for (int q = 0; q < P; ++q) sp.tab[q] = ptr(q, x) ? ptr(q, x) - a(q, l) : nullptr;
        return sp;
    }
    template <int K>
    void xred(RedSlot<K>& red, int r) const {
        red.xslot = slot_tab[r].p;
        red.xP = P;
        red.xrank = r;
    }
    Csr csr(int l, int r) const {
        const DRank& Rr = R(l, r);
        Csr c;
        c.n = L(l).n;
        c.nnz = (int)Rr.nnz;
        c.rp = Rr.rps;
        c.ci = Rr.ci;
        c.av = Rr.av;
        return c;
    }
    Csr members(int l, int r) const {
        const DRank& Rr = R(l, r);
        Csr c;
        c.n = L(l).nc;
        c.rp = Rr.mptr - Rr.mbase;
        c.ci = Rr.mem;
        c.av = nullptr;
        return c;
    }
    // barriers inside NPCG iterations are gated by the iteration's `active`
    // flag (identical on every rank), so gated-off look-ahead replays run none
    const int* bgate = nullptr;
    void sync() { C.barrier(bgate); }
    // one CUDA graph per iteration parity (the plain launch sequence of
    // npcg_iteration, barrier kernels included), replayed with look-ahead
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    uint64_t gk[2] = {0, 0};  // kernels per graph (launch accounting)
    int* h_flag = nullptr;
    int* d_flag = nullptr;
    int flag_slot = -1;
    cudaEvent_t evr[kEvRing] = {};
    ~DistSolve() {
        for (auto& g : graph) if (g) cudaGraphExecDestroy(g);
        mapped_slot_release(flag_slot);
        for (auto& e : evr) if (e) cudaEventDestroy(e);
    }

    void build();
    bool cycle(int l, VRef b, VRef out, GRef g, const VRef* apprev, int beta_state);
    // singular (Neumann) hierarchies, U/solvers.py:112-125 across ranks
    bool sing() const { return H.singular; }
    double* sslot(int r, int l, int k) const { return ws[r].sums.p + 4 * l + k; }
    // cross-rank map-reduce: every rank reduces its rows, totals folded in
    // rank order on every rank (make(r) builds the rank's functor)
    template <class Body, class Mk>
    void xmap(int l, Mk&& make) {
        sync();
        for (int r : C.mine) {
            Body b = make(r);
            b.red = {rs(r).partials, rs(r).ticket};
            xred(b.red, r);
            run_map(nrows(r, l), b, s);
        }
        sync();
        for (int r : C.mine) run_xfin(make(r), ws[r].slots, P, s);
    }
    void project_mean(int l, VRef v, GRef g, int k) {
        xmap<BodySum>(l, [&](int r) {
            BodySum b{};
            b.v = ptr(r, v); b.slot = sslot(r, l, k); b.g = gptr(r, g);
            return b;
        });
        for (int r : C.mine) {
            BodySub sb{};
            sb.n = L(l).n; sb.in = ptr(r, v); sb.out = ptr(r, v); sb.slot = sslot(r, l, k); sb.g = gptr(r, g);
            run_map(nrows(r, l), sb, s);
        }
    }
    void check_compatible(int l, VRef b, VRef out, GRef g) {
        xmap<BodyCompat>(l, [&](int r) {
            BodyCompat bc{};
            bc.b = ptr(r, b); bc.slot = sslot(r, l, 0); bc.err = ws[r].err.p; bc.n = L(l).n; bc.g = gptr(r, g);
            return bc;
        });
        for (int r : C.mine) {
            BodySub sb{};
            sb.n = L(l).n; sb.in = ptr(r, b); sb.out = ptr(r, out); sb.slot = sslot(r, l, 0); sb.g = gptr(r, g);
            run_map(nrows(r, l), sb, s);
        }
    }
    void fcg(int l, VRef b, VRef x, GRef parent, bool begun);
    void npcg_iteration(int parity);
    void run(const std::vector<const double*>& b, const std::vector<const double*>& x0,
             const std::vector<double*>& x, double* hist_host, uaamg_solve_result* res);
};

void DistSolve::build() {
    Ls = H.Ls();
    P = C.P;
    ws.clear();
    ws.resize(P);
    vec.assign(kRoles, std::vector<std::vector<double*>>(Ls, std::vector<double*>(P, nullptr)));
    outer.assign(kTRoles, std::vector<double*>(P, nullptr));
    const bool inner = p.kcycle && p.inner_krylov_steps > 0;
    for (int r : C.mine) {
        RankWs& W = ws[r];
        W.fcg.alloc(std::max(Ls, 1), s);
        UA_CK(cudaMemsetAsync(W.fcg.p, 0, sizeof(FcgState) * std::max(Ls, 1), s));
        W.npcg.alloc(1, s);
        UA_CK(cudaMemsetAsync(W.npcg.p, 0, sizeof(NpcgState), s));
        W.partials.alloc(4 * (size_t)kMaxRedBlocks, s);
        W.ticket.alloc(1, s);
        UA_CK(cudaMemsetAsync(W.ticket.p, 0, sizeof(unsigned), s));
        W.hist.alloc((size_t)p.max_iters + 1, s);
        W.bad_row.alloc(std::max(Ls, 1), s);
        {
            std::vector<int> init(std::max(Ls, 1), 0x7fffffff);
            UA_CK(cudaMemcpyAsync(W.bad_row.p, init.data(), sizeof(int) * init.size(), cudaMemcpyHostToDevice, s));
            UA_CK(cudaStreamSynchronize(s));
        }
        W.slots = C.alloc<double>(r, (size_t)kSlotK * P);
        W.sums.alloc(4 * (size_t)Ls + 8, s);
        UA_CK(cudaMemsetAsync(W.sums.p, 0, sizeof(double) * (4 * Ls + 8), s));
        W.err.alloc(1, s);
        UA_CK(cudaMemsetAsync(W.err.p, 0, sizeof(int), s));
        W.gA.resize(Ls);
        W.gP.resize(Ls);
        for (int l = 0; l < Ls; ++l) {
            const DRank& Rr = R(l, r);
            const size_t n = std::max(Rr.n, 1);
            auto take = [&](VRole v) { vec[v][l][r] = C.alloc<double>(r, n); };
            take(V_INVM); take(V_R); take(V_TA); take(V_TB);
            if (sing()) take(V_BP);
            if (p.post_sweeps > 1) take(V_XUP);
            if (l > 0) { take(V_RHS); take(V_E); }
            if (l > 0 && inner) {
                take(V_XF); take(V_RF); take(V_Z); take(V_P0); take(V_P1); take(V_AP0); take(V_AP1);
            }
            build_groups(Rr.n, Rr.rps, kSolveLongMin, W.gA[l], s, Rr.a);
            if (Rr.n >= kTmaMinRows / 8 && W.gA[l].g.np == 0) set_tma(W.gA[l].g, Rr.n, Rr.rps, s, Rr.a);
            set_ell(W.gA[l], csr(l, r), s, Rr.n, Rr.a);
            // restriction rows: own aggregates, or all of them into the
            // replicated level
            const int ca = Rr.mbase, cn = Rr.mcount;
            build_groups(cn, Rr.mptr - Rr.mbase, kSolveLongMin, W.gP[l], s, ca);
            launch_inv_diag(csr(l, r), W.gA[l], p.smoother_l1, p.omega, vec[V_INVM][l][r] - Rr.a, W.bad_row.p + l, s);
        }
        const size_t n0 = std::max(R(0, r).n, 1);
        for (int t = 0; t < kTRoles; ++t) outer[t][r] = C.alloc<double>(r, n0);
        W.rws = build_ws(H.rep.get(), p, s, 0, true);
    }
    // the finest level's bad row first (the reference's smooth() order)
    std::vector<long long> bad(P, 0x7fffffff);
    for (int l = 0; l < Ls; ++l) {
        for (int r : C.mine) {
            int hb = 0;
            UA_CK(cudaMemcpyAsync(&hb, ws[r].bad_row.p + l, sizeof(int), cudaMemcpyDeviceToHost, s));
            UA_CK(cudaStreamSynchronize(s));
            bad[r] = hb;
        }
        long long m = 0x7fffffff;
        for (long long v : C.allgather(bad)) m = std::min(m, v);
        if (m != 0x7fffffff) throw Error(UAAMG_ENUMERICAL, "non-positive smoother diagonal at row " + std::to_string(m));
    }
    // every rank's blocks (one exchange for all roles)
    std::vector<std::vector<void*>> loc;
    for (int v = 0; v < kRoles; ++v)
        for (int l = 0; l < Ls; ++l) loc.emplace_back(vec[v][l].begin(), vec[v][l].end());
    for (int t = 0; t < kTRoles; ++t) loc.emplace_back(outer[t].begin(), outer[t].end());
    {
        std::vector<void*> sl(P, nullptr);
        for (int r : C.mine) sl[r] = ws[r].slots;
        loc.push_back(sl);
    }
    auto T = C.tables(loc);
    size_t k = 0;
    for (int v = 0; v < kRoles; ++v)
        for (int l = 0; l < Ls; ++l, ++k)
            for (int q = 0; q < P; ++q) vec[v][l][q] = static_cast<double*>(T[k][q]);
    for (int t = 0; t < kTRoles; ++t, ++k)
        for (int q = 0; q < P; ++q) outer[t][q] = static_cast<double*>(T[k][q]);
    std::vector<double*> slots(P);
    for (int q = 0; q < P; ++q) slots[q] = static_cast<double*>(T[k][q]);
    slot_tab.clear();
    slot_tab.resize(P);
    for (int r : C.mine) {
        slot_tab[r].alloc(P, s);
        UA_CK(cudaMemcpyAsync(slot_tab[r].p, slots.data(), sizeof(double*) * P, cudaMemcpyHostToDevice, s));
    }
    UA_CK(cudaStreamSynchronize(s));
}

// U/solvers.py:128-157 on a sharded level; returns whether the beta dot of
// the consuming flexible CG was fused into the last sweep
bool DistSolve::cycle(int l, VRef b, VRef out, GRef g, const VRef* apprev, int beta_state) {
    const int xmode = p.pre_sweeps == 0 ? 0 : 2;
    if (sing()) {
        // U/solvers.py:141: b = _check_compatible(b) (drift check + projection)
        check_compatible(l, b, Lv(l, V_BP), g);
        b = Lv(l, V_BP);
        apprev = nullptr;  // the beta dot is not fused: z is projected first (U/solvers.py:157)
    }
    // pre-smoothing from a zero guess, materialised (x = 0 + inv_m b, then sweeps)
    VRef cur = Lv(l, V_TA);
    if (xmode == 2) {
        for (int r : C.mine) {
            BodyXpre1 body{};
            body.invm = ptr(r, Lv(l, V_INVM));
            body.b = ptr(r, b);
            body.x = ptr(r, cur);
            body.g = gptr(r, g);
            run_map(nrows(r, l), body, s);
        }
        for (int k = 1; k < p.pre_sweeps; ++k) {
            VRef nx = Lv(l, cur.v == V_TA ? V_TB : V_TA);
            sync();
            for (int r : C.mine) {
                EpiSweep e{};
                e.invm = sh(r, Lv(l, V_INVM)); e.b = sh(r, b); e.out = sh(r, nx); e.g = gptr(r, g);
                run_stream<SrcPeer, EpiSweep, false>(csr(l, r), ws[r].gA[l].g, peer(cur, l), e, s);
            }
            cur = nx;
        }
    }
    // r = b - A x
    sync();
    for (int r : C.mine) {
        EpiResid e{};
        e.b = sh(r, b); e.r = sh(r, Lv(l, V_R)); e.g = gptr(r, g);
        if (xmode == 0) run_stream<SrcZero, EpiResid, false>(csr(l, r), ws[r].gA[l].g, SrcZero{}, e, s);
        else run_stream<SrcPeer, EpiResid, false>(csr(l, r), ws[r].gA[l].g, peer(cur, l), e, s);
    }
    // r_c = restrict(r): members gathered from their owners, ascending order
    const int lc = l + 1;
    const bool csh = lc < Ls;
    const int nlev = H.nlevels();
    const bool exact = (lc == nlev - 1);
    const bool direct = !p.kcycle || p.inner_krylov_steps == 0 || exact;
    const bool begun = !direct && !sing();  // singular: the coarse FCG begins after the projection
    sync();
    for (int r : C.mine) {
        const int ca = R(l, r).mbase;
        double* y = csh ? sh(r, Lv(lc, V_RHS)) : ws[r].rws->lev[0].rhs.p - ca;
        FcgState* st = csh ? fst(r, lc) : ws[r].rws->fcg.p;
        if (begun) {
            EpiRestrictBegin e{};
            e.y = y; e.g = gptr(r, g); e.st = st;
            e.red = {rs(r).partials, rs(r).ticket};
            if (csh) xred(e.red, r);
            run_stream<SrcPeer, EpiRestrictBegin, true>(members(l, r), ws[r].gP[l].g, peer(Lv(l, V_R), l), e, s);
        } else {
            EpiStoreG e{};
            e.y = y; e.g = gptr(r, g);
            run_stream<SrcPeer, EpiStoreG, true>(members(l, r), ws[r].gP[l].g, peer(Lv(l, V_R), l), e, s);
        }
    }
    if (begun && csh) {
        sync();
        for (int r : C.mine) {
            EpiRestrictBegin e{};
            e.st = fst(r, lc);
            e.g = gptr(r, g);
            run_xfin(e, ws[r].slots, P, s);
        }
    }
    if (sing()) {
        // U/solvers.py:150: r_c = _project_mean(restrict(r))
        if (csh) {
            project_mean(lc, Lv(lc, V_RHS), g, 1);
        } else {
            for (int r : C.mine)
                launch_project_mean(L(l).nc, ws[r].rws->lev[0].rhs.p, sslot(r, Ls, 1), gptr(r, g), rs(r), s);
        }
    }
    // coarse correction
    VRef ec = Lv(lc, direct ? V_E : V_XF);
    if (csh) {
        if (direct) cycle(lc, Lv(lc, V_RHS), ec, g, nullptr, 0);
        else fcg(lc, Lv(lc, V_RHS), ec, g, begun);
    } else {
        for (int r : C.mine) {
            Plan pl = plan(r);
            LevelWs& Cw = ws[r].rws->lev[0];
            if (direct) pl.cycle(0, Cw.rhs.p, Cw.e.p, gptr(r, g));
            else pl.fcg(0, Cw.rhs.p, Cw.xf.p, gptr(r, g), begun);
        }
    }
    // prolongation on own rows into tB (or tA if the pre-iterate lives in tB)
    VRef other = Lv(l, cur.v == V_TA ? V_TB : V_TA);
    sync();
    for (int r : C.mine) {
        BodyProlPeer body{};
        body.mode = xmode;
        body.xpre = ptr(r, cur);
        body.v2a = R(l, r).v2a;
        if (csh) {
            body.pt = L(lc).pt;
            for (int q = 0; q < P; ++q) body.ec[q] = ptr(q, ec) - a(q, lc);
            body.ec_valid = direct ? nullptr : &fst(r, lc)->upd[0];
        } else {
            body.pt = Part{1, {0, L(l).nc}};
            LevelWs& Cw = ws[r].rws->lev[0];
            for (int q = 0; q < P; ++q) body.ec[q] = direct ? Cw.e.p : Cw.xf.p;
            body.ec_valid = direct ? nullptr : &ws[r].rws->fcg.p[0].upd[0];
        }
        body.out = ptr(r, other);
        body.g = gptr(r, g);
        run_map(nrows(r, l), body, s);
    }
    // post-smoothing sweeps; the last may carry the consuming CG's beta dot
    if (p.post_sweeps == 0) {
        for (int r : C.mine)
            UA_CK(cudaMemcpyAsync(ptr(r, out), ptr(r, other), sizeof(double) * nrows(r, l), cudaMemcpyDeviceToDevice,
                                  s));
        return false;
    }
    VRef src = other;
    for (int k = 0; k < p.post_sweeps; ++k) {
        const bool last = (k == p.post_sweeps - 1);
        VRef dst = last ? out : Lv(l, src.v == V_XUP ? V_TA : V_XUP);
        sync();
        for (int r : C.mine) {
            if (last && apprev) {
                EpiSweepBeta e{};
                e.invm = sh(r, Lv(l, V_INVM)); e.b = sh(r, b); e.out = sh(r, dst); e.g = gptr(r, g);
                e.apprev = sh(r, *apprev);
                if (beta_state == 0) {
                    e.beta = &nst(r)->beta; e.pap = &nst(r)->pap; e.have = &nst(r)->have_prev;
                } else {
                    e.beta = &fst(r, l)->beta; e.pap = &fst(r, l)->pap; e.have = nullptr;
                }
                e.red = {rs(r).partials, rs(r).ticket};
                xred(e.red, r);
                run_stream<SrcPeer, EpiSweepBeta, false>(csr(l, r), ws[r].gA[l].g, peer(src, l), e, s);
            } else {
                EpiSweep e{};
                e.invm = sh(r, Lv(l, V_INVM)); e.b = sh(r, b); e.out = sh(r, dst); e.g = gptr(r, g);
                run_stream<SrcPeer, EpiSweep, false>(csr(l, r), ws[r].gA[l].g, peer(src, l), e, s);
            }
        }
        src = dst;
    }
    if (apprev) {
        sync();
        for (int r : C.mine) {
            EpiSweepBeta e{};
            if (beta_state == 0) {
                e.beta = &nst(r)->beta; e.pap = &nst(r)->pap; e.have = &nst(r)->have_prev;
            } else {
                e.beta = &fst(r, l)->beta; e.pap = &fst(r, l)->pap; e.have = nullptr;
            }
            e.g = gptr(r, g);
            run_xfin(e, ws[r].slots, P, s);
        }
    }
    if (sing()) project_mean(l, out, g, 3);  // U/solvers.py:157
    return apprev != nullptr;
}

// U/solvers.py:160-187 on a sharded level (begun: ||b|| came from the restriction)
void DistSolve::fcg(int l, VRef b, VRef x, GRef parent, bool begun) {
    if (!begun) {
        sync();  // every publishing kernel waits for the peers' previous folds of our slots
        for (int r : C.mine) {
            BodyFcgBegin body{};
            body.b = ptr(r, b); body.pg = gptr(r, parent); body.st = fst(r, l);
            body.red = {rs(r).partials, rs(r).ticket};
            xred(body.red, r);
            run_map(nrows(r, l), body, s);
        }
        sync();
        for (int r : C.mine) {
            BodyFcgBegin body{};
            body.st = fst(r, l);
            body.pg = gptr(r, parent);
            run_xfin(body, ws[r].slots, P, s);
        }
    }
    const VRole PR[2] = {V_P0, V_P1}, APR[2] = {V_AP0, V_AP1};
    for (int k = 0; k < p.inner_krylov_steps; ++k) {
        GRef g{2, l, k};
        VRef rin = (k == 0) ? b : Lv(l, V_RF);
        VRef pc = Lv(l, PR[k & 1]), pp = Lv(l, PR[(k + 1) & 1]), apc = Lv(l, APR[k & 1]), app = Lv(l, APR[(k + 1) & 1]);
        const bool fused = cycle(l, rin, Lv(l, V_Z), g, k > 0 ? &app : nullptr, 1);
        if (k > 0 && !fused) {
            xmap<BodyBeta>(l, [&](int r) {
                BodyBeta bb{};
                bb.z = ptr(r, Lv(l, V_Z)); bb.pp = ptr(r, pp); bb.ap = ptr(r, app); bb.beta = &fst(r, l)->beta;
                bb.g = gptr(r, g); bb.g2 = nullptr;
                return bb;
            });
        }
        // p = z + beta p_prev on own rows, then Ap (+ p.Ap, p.r)
        for (int r : C.mine) {
            BodyDirP bp{};
            bp.src.z = ptr(r, Lv(l, V_Z)); bp.src.pprev = ptr(r, pp); bp.src.beta_p = &fst(r, l)->beta;
            bp.src.have_p = nullptr; bp.src.have_static = k > 0;
            bp.p = ptr(r, pc); bp.g = gptr(r, g);
            run_map(nrows(r, l), bp, s);
        }
        sync();
        for (int r : C.mine) {
            EpiDirFcg e{};
            e.p = nullptr; e.ap = sh(r, apc); e.r = sh(r, rin); e.st = fst(r, l); e.step = k;
            e.red = {rs(r).partials, rs(r).ticket};
            xred(e.red, r);
            run_stream<SrcPeer, EpiDirFcg, false>(csr(l, r), ws[r].gA[l].g, peer(pc, l), e, s);
        }
        sync();
        for (int r : C.mine) {
            EpiDirFcg e{};
            e.st = fst(r, l); e.step = k;
            run_xfin(e, ws[r].slots, P, s);
        }
        sync();
        for (int r : C.mine) {
            BodyFcgUpd body{};
            body.step = k; body.x = ptr(r, x); body.p = ptr(r, pc); body.rin = ptr(r, rin);
            body.rout = ptr(r, Lv(l, V_RF)); body.ap = ptr(r, apc); body.st = fst(r, l); body.singular = sing();
            body.red = {rs(r).partials, rs(r).ticket};
            xred(body.red, r);
            run_map(nrows(r, l), body, s);
        }
        sync();
        for (int r : C.mine) {
            BodyFcgUpd body{};
            body.step = k; body.st = fst(r, l); body.singular = sing();
            run_xfin(body, ws[r].slots, P, s);
        }
        if (sing()) {
            // r -= mean(r), gate from the projected norm (U/solvers.py:185-186)
            xmap<BodyFcgProj>(l, [&](int r) {
                BodyFcgProj pj{};
                pj.n = L(l).n; pj.step = k; pj.r = ptr(r, Lv(l, V_RF)); pj.st = fst(r, l);
                return pj;
            });
        }
    }
}

// one NPCG iteration (U/solvers.py:221-254) on sharded level 0
void DistSolve::npcg_iteration(int parity) {
    const TRole PR[2] = {T_P0, T_P1}, APR[2] = {T_AP0, T_AP1};
    VRef pc = O(PR[parity]), pp = O(PR[parity ^ 1]), apc = O(APR[parity]), app = O(APR[parity ^ 1]);
    GRef act{1, 0, 0};
    const bool fused = cycle(0, O(T_R), O(T_Z), act, &app, 0);
    if (sing()) project_mean(0, O(T_Z), act, 2);  // U/solvers.py:224
    if (!fused) {
        xmap<BodyBeta>(0, [&](int r) {
            BodyBeta bb{};
            bb.z = ptr(r, O(T_Z)); bb.pp = ptr(r, pp); bb.ap = ptr(r, app); bb.beta = &nst(r)->beta;
            bb.g = gptr(r, act); bb.g2 = &nst(r)->have_prev;
            return bb;
        });
    }
    for (int r : C.mine) {
        BodyDirP bp{};
        bp.src.z = ptr(r, O(T_Z)); bp.src.pprev = ptr(r, pp); bp.src.beta_p = &nst(r)->beta;
        bp.src.have_p = &nst(r)->have_prev;
        bp.p = ptr(r, pc); bp.g = gptr(r, act);
        run_map(nrows(r, 0), bp, s);
    }
    sync();
    for (int r : C.mine) {
        EpiDirNpcg e{};
        e.p = nullptr; e.ap = sh(r, apc); e.r = sh(r, O(T_R)); e.st = nst(r);
        e.red = {rs(r).partials, rs(r).ticket};
        xred(e.red, r);
        SrcPeer sp{};
        sp.pt = L(0).pt;
        for (int q = 0; q < P; ++q) sp.tab[q] = ptr(q, pc) - a(q, 0);
        run_stream<SrcPeer, EpiDirNpcg, false>(csr(0, r), ws[r].gA[0].g, sp, e, s);
    }
    sync();
    for (int r : C.mine) {
        EpiDirNpcg e{};
        e.st = nst(r);
        run_xfin(e, ws[r].slots, P, s);
    }
    sync();
    for (int r : C.mine) {
        BodyNpcgUpd body{};
        body.x = ptr(r, O(T_X)); body.p = ptr(r, pc); body.r = ptr(r, O(T_R)); body.ap = ptr(r, apc);
        body.st = nst(r); body.hist = ws[r].hist.p; body.singular = sing();
        body.red = {rs(r).partials, rs(r).ticket};
        xred(body.red, r);
        run_map(nrows(r, 0), body, s);
    }
    sync();
    for (int r : C.mine) {
        BodyNpcgUpd body{};
        body.st = nst(r); body.hist = ws[r].hist.p; body.singular = sing();
        run_xfin(body, ws[r].slots, P, s);
    }
    if (sing()) {
        // x and r projected, then the norm and the bookkeeping (U/solvers.py:238-240)
        xmap<BodyNpcgProjX>(0, [&](int r) {
            BodyNpcgProjX bx{};
            bx.x = ptr(r, O(T_X)); bx.st = nst(r);
            return bx;
        });
        xmap<BodyNpcgProj>(0, [&](int r) {
            BodyNpcgProj pj{};
            pj.n = L(0).n; pj.x = ptr(r, O(T_X)); pj.r = ptr(r, O(T_R)); pj.st = nst(r); pj.hist = ws[r].hist.p;
            return pj;
        });
    }
}

__global__ void k_set_npcg_d(NpcgState* st, double tol, int max_iters, int* host_active) {
    st->host_active = host_active;
    st->tol = tol;
    st->max_iters = max_iters;
}

// b, x0, x: per local rank, own rows (device)
void DistSolve::run(const std::vector<const double*>& b, const std::vector<const double*>& x0,
                    const std::vector<double*>& x, double* hist_host, uaamg_solve_result* res) {
    const int me = C.mine[0];
    const bool have_x0 = !x0.empty() && x0[0] != nullptr;
    bgate = nullptr;
    if (flag_slot < 0) {
        flag_slot = mapped_slot_acquire(&h_flag, &d_flag);
        for (auto& e : evr) UA_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    *(volatile int*)h_flag = 1;
    cudaEvent_t e0, e1;
    UA_CK(cudaEventCreate(&e0));
    UA_CK(cudaEventCreate(&e1));
    UA_CK(cudaEventRecord(e0, s));
    for (size_t k = 0; k < C.mine.size(); ++k) {
        const int r = C.mine[k];
        const size_t n = nrows(r, 0);
        UA_CK(cudaMemcpyAsync(ptr(r, O(T_B)), b[k], sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        if (have_x0) UA_CK(cudaMemcpyAsync(ptr(r, O(T_X)), x0[k], sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        else UA_CK(cudaMemsetAsync(ptr(r, O(T_X)), 0, sizeof(double) * n, s));
        UA_CK(cudaMemsetAsync(ws[r].npcg.p, 0, sizeof(NpcgState), s));
        UA_CK(cudaMemsetAsync(ws[r].fcg.p, 0, sizeof(FcgState) * std::max(Ls, 1), s));
        UA_CK(cudaMemsetAsync(ws[r].err.p, 0, sizeof(int), s));
        if (ws[r].rws) UA_CK(cudaMemsetAsync(ws[r].rws->err.p, 0, sizeof(int), s));
    }
    if (sing()) {
        // U/solvers.py:203-204, 211-215: b projected (error if incompatible), x0 projected
        check_compatible(0, O(T_B), O(T_B), GRef{});
        int herr = 0;
        for (int r : C.mine) {
            int h = 0;
            UA_CK(cudaMemcpyAsync(&h, ws[r].err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            UA_CK(cudaStreamSynchronize(s));
            herr |= h;
        }
        if (herr) throw Error(UAAMG_ENUMERICAL, "right-hand side at the finest level has a null-space component");
        if (have_x0) project_mean(0, O(T_X), GRef{}, 2);
    }
    sync();
    for (int r : C.mine) {
        EpiResid e{};
        e.b = sh(r, O(T_B)); e.r = sh(r, O(T_R)); e.g = nullptr;
        if (have_x0) run_stream<SrcPeer, EpiResid, false>(csr(0, r), ws[r].gA[0].g, peer(O(T_X), 0), e, s);
        else run_stream<SrcZero, EpiResid, false>(csr(0, r), ws[r].gA[0].g, SrcZero{}, e, s);
        UA_LAUNCH(k_set_npcg_d, 1, 1, 0, s, nst(r), p.tol, p.max_iters, r == me ? d_flag : nullptr);
    }
    sync();
    for (int r : C.mine) {
        BodyNpcgInit body{};
        body.b = ptr(r, O(T_B)); body.r = ptr(r, O(T_R)); body.st = nst(r); body.hist = ws[r].hist.p;
        body.red = {rs(r).partials, rs(r).ticket};
        xred(body.red, r);
        run_map(nrows(r, 0), body, s);
    }
    sync();
    for (int r : C.mine) {
        BodyNpcgInit body{};
        body.st = nst(r); body.hist = ws[r].hist.p;
        run_xfin(body, ws[r].slots, P, s);
    }
    NpcgState hst{};
    UA_CK(cudaMemcpyAsync(&hst, nst(me), sizeof(NpcgState), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    bgate = &nst(me)->active;
    if (hst.active && p.use_graphs) {
        if (!graph[0]) {
            for (int par = 0; par < 2; ++par) {
                cudaGraph_t g;
                const uint64_t before = g_launches.load();
                UA_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
                npcg_iteration(par);
                UA_CK(cudaStreamEndCapture(s, &g));
                gk[par] = g_launches.load() - before;
                g_launches.fetch_sub(gk[par]);  // captured, not executed: counted per replay
                UA_CK(cudaGraphInstantiate(&graph[par], g, 0));
                cudaGraphDestroy(g);
            }
        }
        // pipelined kLookahead iterations deep; gated-off replays past the
        // end skip every kernel body and every barrier on all ranks alike
        for (int it = 0; it < p.max_iters; ++it) {
            UA_CK(cudaGraphLaunch(graph[it & 1], s));
            g_launches.fetch_add(gk[it & 1]);
            UA_CK(cudaEventRecord(evr[it % kEvRing], s));
            if (it >= kLookahead) {
                UA_CK(cudaEventSynchronize(evr[(it - kLookahead) % kEvRing]));
                if (*(volatile int*)h_flag == 0) break;
            }
        }
        UA_CK(cudaMemcpyAsync(&hst, nst(me), sizeof(NpcgState), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
    } else {
        for (int it = 0; hst.active && it < p.max_iters; ++it) {
            npcg_iteration(it & 1);
            UA_CK(cudaMemcpyAsync(&hst, nst(me), sizeof(NpcgState), cudaMemcpyDeviceToHost, s));
            UA_CK(cudaStreamSynchronize(s));
        }
    }
    bgate = nullptr;
    UA_CK(cudaEventRecord(e1, s));
    for (size_t k = 0; k < C.mine.size(); ++k) {
        const int r = C.mine[k];
        UA_CK(cudaMemcpyAsync(x[k], ptr(r, O(T_X)), sizeof(double) * nrows(r, 0), cudaMemcpyDeviceToDevice, s));
    }
    UA_CK(cudaStreamSynchronize(s));
    float ms = 0;
    UA_CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    res->iterations = hst.iters;
    res->solve_seconds = ms * 1e-3;
    if (hist_host)
        UA_CK(cudaMemcpy(hist_host, ws[me].hist.p, sizeof(double) * (hst.iters + 1), cudaMemcpyDeviceToHost));
    res->converged = (hst.bnorm == 0.0) ? 1 : (hst.last_rel <= p.tol);
    res->status = 0;
    if (sing()) {
        int herr = 0;
        for (int r : C.mine) {
            int h = 0, h2 = 0;
            UA_CK(cudaMemcpy(&h, ws[r].err.p, sizeof(int), cudaMemcpyDeviceToHost));
            UA_CK(cudaMemcpy(&h2, ws[r].rws->err.p, sizeof(int), cudaMemcpyDeviceToHost));
            herr |= h | h2;
        }
        if (herr) {
            res->converged = 0;
            res->status = UAAMG_ENUMERICAL;
            throw Error(UAAMG_ENUMERICAL,
                        "right-hand side at a coarse level has a null-space component (relative size > 1e-10)");
        }
    }
    if (hst.status == 1) {
        res->converged = 0;
        res->status = UAAMG_ENUMERICAL;
        throw Error(UAAMG_ENUMERICAL, "conjugate-gradient breakdown (sharded solve)");
    }
}

}  // namespace uaamg

// ====================================================================== C ABI
using namespace uaamg;

struct uaamg_comm {
    std::shared_ptr<Comm> c;
};
struct uaamg_dhier {
    std::unique_ptr<DistHier> H;
    std::unique_ptr<DistSolve> S;
    uaamg_solve_params key{};
    std::mutex mu;
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

int uaamg_comm_create(int nranks, int rank, int64_t arena_bytes, uaamg_comm** out) {
    UA_TRY({
        auto c = std::make_unique<uaamg_comm>();
        c->c = std::make_shared<Comm>();
        c->c->create(nranks, rank, (size_t)arena_bytes, library_stream());
        if (rank < 0) c->c->connect_virtual();
        *out = c.release();
    })
}

int uaamg_comm_handle(uaamg_comm* c, void* handle) {
    UA_TRY({
        if (c->c->virt()) throw Error(UAAMG_EINVAL, "virtual ranks have no IPC handle");
        cudaIpcMemHandle_t hd;
        UA_CK(cudaIpcGetMemHandle(&hd, c->c->base[c->c->rank]));
        std::memcpy(handle, &hd, sizeof(hd));
    })
}

int uaamg_comm_connect(uaamg_comm* c, const void* handles) {
    UA_TRY({
        if (c->c->virt()) throw Error(UAAMG_EINVAL, "virtual ranks need no connection");
        c->c->connect(handles);
    })
}

int uaamg_comm_barrier(uaamg_comm* c) {
    UA_TRY({ c->c->host_barrier(); })
}

void uaamg_comm_free(uaamg_comm* c) { delete c; }

int uaamg_dsetup(uaamg_comm* c, int n, const int* bounds, const int* const* row_ptr, const int* const* col,
                 const double* const* val, const int64_t* nnz, const uaamg_setup_params* params, int64_t shard_rows,
                 uaamg_dhier** out, void* stream) {
    UA_TRY({
        Comm& C = *c->c;
        const size_t m = C.mine.size();
        std::vector<const int*> rp(row_ptr, row_ptr + m), ci(col, col + m);
        std::vector<const double*> av(val, val + m);
        std::vector<long long> nz(nnz, nnz + m);
        StreamJoin join((cudaStream_t)stream, C.s);
        auto d = std::make_unique<uaamg_dhier>();
        d->H = dist_setup(c->c, n, bounds, rp, ci, av, nz, *params, shard_rows);
        *out = d.release();
    })
}

void uaamg_dhier_free(uaamg_dhier* d) {
    if (!d) return;
    delete d;
}

int uaamg_dhier_get_info(const uaamg_dhier* d, uaamg_dhier_info* info) {
    UA_TRY({
        const DistHier& H = *d->H;
        info->n_levels = H.nlevels();
        info->n_sharded = H.Ls();
        info->singular = H.singular;
        info->grid_complexity = H.grid_complexity;
        info->operator_complexity = H.operator_complexity;
        info->setup_seconds = H.setup_seconds;
    })
}

int uaamg_dhier_level(const uaamg_dhier* d, int level, int rank, uaamg_dlevel_view* v) {
    UA_TRY({
        const DistHier& H = *d->H;
        if (level < 0 || level >= H.nlevels()) throw Error(UAAMG_EINVAL, "level out of range");
        std::memset(v, 0, sizeof(*v));
        v->n = H.level_n(level);
        v->nnz = H.level_nnz(level);
        if (level < H.Ls()) {
            const DLevel& L = H.lv[level];
            if (rank < 0 || rank >= H.C->P || !(H.C->virt() || rank == H.C->rank))
                throw Error(UAAMG_EINVAL, "rank is not local to this process");
            const DRank& R = L.r[rank];
            v->sharded = 1;
            v->row_begin = R.a;
            v->row_end = R.a + R.n;
            v->local_nnz = R.nnz;
            v->row_ptr = R.rp;
            v->col = R.ci;
            v->val = R.av;
            v->n_coarse = L.nc;
            v->vertex_to_agg = R.v2a;
            v->seeds = R.seeds;
            v->n_seeds = R.nseeds;
        } else {
            const Level& Lr = *H.rep->levels[level - H.Ls()];
            v->sharded = 0;
            v->row_begin = 0;
            v->row_end = Lr.n;
            v->local_nnz = Lr.nnz;
            v->row_ptr = Lr.rp.p;
            v->col = Lr.ci.p;
            v->val = Lr.av.p;
            v->n_coarse = Lr.nc;
            v->vertex_to_agg = Lr.nc ? Lr.v2a.p : nullptr;
            v->seeds = Lr.nc ? Lr.seeds.p : nullptr;
            v->n_seeds = Lr.nc;
        }
    })
}

int uaamg_dsolve(uaamg_dhier* d, const uaamg_solve_params* p, const double* const* b, const double* const* x0,
                 double* const* x, double* history_host, uaamg_solve_result* res, void* stream) {
    UA_TRY({
        std::memset(res, 0, sizeof(*res));
        if (!(p->tol > 0)) throw Error(UAAMG_EINVAL, "tol must be positive");
        DistHier& H = *d->H;
        if (H.Ls() == 0) throw Error(UAAMG_EUNSUPPORTED, "no sharded level (the whole hierarchy is replicated)");
        if (p->inner_krylov_steps > kMaxInner) throw Error(UAAMG_EUNSUPPORTED, "inner_krylov_steps > 16");
        std::lock_guard<std::mutex> lk(d->mu);
        Comm& C = *H.C;
        StreamJoin join((cudaStream_t)stream, C.s);
        const uaamg_solve_params& k = d->key;
        const bool same = d->S && k.kcycle == p->kcycle && k.inner_krylov_steps == p->inner_krylov_steps &&
                          k.pre_sweeps == p->pre_sweeps && k.post_sweeps == p->post_sweeps &&
                          k.smoother_l1 == p->smoother_l1 && k.omega == p->omega && k.max_iters >= p->max_iters;
        if (!same) {
            std::vector<size_t> marks = C.lo;
            if (d->S) marks = d->S->marks;  // a new workspace reuses the old one's arena region
            d->S.reset();
            for (int r : C.mine) C.lo[r] = marks[r];
            d->S.reset(new DistSolve{H, C, *p, C.s});
            d->S->marks = marks;
            d->S->build();
            d->key = *p;
        }
        d->S->p = *p;
        d->S->p.max_iters = p->max_iters;
        const size_t m = C.mine.size();
        std::vector<const double*> bb(b, b + m), xx0;
        if (x0) xx0.assign(x0, x0 + m);
        std::vector<double*> xx(x, x + m);
        d->S->run(bb, xx0, xx, history_host, res);
    })
}

int uaamg_coarse_bounds(const int64_t* counts, int nranks, int* bounds) {
    UA_HOST_TRY({
        if (nranks < 1 || nranks > kMaxRanks) throw Error(UAAMG_EINVAL, "ranks must be in [1, 8]");
        std::vector<long long> c(counts, counts + nranks);
        const Part pt = coarse_bounds(c.data(), nranks);
        for (int q = 0; q <= nranks; ++q) bounds[q] = pt.b[q];
    })
}

int uaamg_partition_rows(int n, int nranks, int* bounds) {
    UA_HOST_TRY({
        if (nranks < 1 || nranks > kMaxRanks) throw Error(UAAMG_EINVAL, "ranks must be in [1, 8]");
        const Part pt = level0_part(n, nranks);
        for (int q = 0; q <= nranks; ++q) bounds[q] = pt.b[q];
    })
}

}  // extern "C"

namespace uaamg {
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
    for (int q = P + 1; q <= kMaxRanks; ++q) pt.b[q] = n;
    return pt;
}
Part coarse_bounds(const long long* counts, int P) {
    Part pt{};
    pt.P = P;
    long long t = 0;
    for (int q = 0; q < P; ++q) {
        if (counts[q] < 0) throw Error(UAAMG_EINVAL, "negative seed count");
        pt.b[q] = (int)t;
        t += counts[q];
    }
    if (t > 0x7fffffffll) throw Error(UAAMG_EINVAL, "coarse level exceeds int32 indices");
    for (int q = P; q <= kMaxRanks; ++q) pt.b[q] = (int)t;
    return pt;
}
}  // namespace uaamg
