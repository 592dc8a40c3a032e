"""Parity of the B200 path (through the C ABI) with the reference.

Golden fixtures come from the reference package itself
(tests/golden/make_golden.py); the CPU oracle (oracle/) supplies live
comparisons on extra random inputs.  Bar (north star): kernels, MIS sets,
aggregate maps, coarse patterns and values bit-exact; residual histories
within 1e-10 relative, iteration counts +-1.
"""

import numpy as np
import pytest
import torch

from golden_util import (CASE_CFG, HIERARCHY_CASES, SOLVE_VARIANTS, assert_hierarchy_equal,
                         assert_history_close, load, problem_for)

pytestmark = pytest.mark.gpu

RTOL = 1e-10   # relative residual-history tolerance (BASELINE.json north star)


@pytest.fixture(scope="module")
def U():
    import paper_1302_2547_b200 as U
    assert torch.cuda.is_available()
    return U


@pytest.fixture(scope="module")
def K():
    from paper_1302_2547_b200 import kernel_table as K
    return K


@pytest.fixture(scope="module")
def kern():
    return load("kernels")


def _smat(U, ip, ix, a):
    return U.SparseMatrix(ip.shape[0] - 1, ip.shape[0] - 1, ip, ix, a)


def test_kernel_table_bitexact(K, kern):
    k = kern
    ip, ix, a = k["indptr"], k["indices"], k["data"]
    assert np.array_equal(K.spmv(ip, ix, a, k["x"]), k["spmv"])
    assert np.array_equal(K.diag_of(ip, ix, a), k["diag_of"])
    assert np.array_equal(K.l1_diag(ip, ix, a), k["l1_diag"])
    assert np.array_equal(K.degrees(ip, ix), k["degrees"])
    assert np.array_equal(K.hash_u01(0xDEADBEEF12345678, 5, k["hash_idx"]), k["hash_u01"])
    assert np.array_equal(K.quasi_random_scores(ip, ix, 0, 0), k["scores_p0"])
    assert np.array_equal(K.quasi_random_scores(ip, ix, 7, 3), k["scores_s7_p3"])
    p2, x2 = K.squared_pattern(ip.shape[0] - 1, ip, ix)
    assert np.array_equal(p2, k["a2_indptr"]) and np.array_equal(x2, k["a2_indices"])
    ctr = K.select_centers(p2, x2, k["scores_s7_p3"], k["processed"])
    assert np.array_equal(ctr, k["select"])
    assert np.array_equal(K.select_centers_2hop(ip, ix, k["scores_s7_p3"], k["processed"]), k["select"])
    own = K.claim_owners(p2, x2, k["scores_s7_p3"], k["processed"], ctr)
    assert np.array_equal(own, k["claim"])
    assert np.array_equal(K.claim_owners_2hop(ip, ix, k["scores_s7_p3"], k["processed"], ctr), k["claim"])
    for tag, cap in (("cap3", 3), ("uncapped", 1 << 62)):
        pr = k["processed"].copy()
        v2a = np.full(ip.shape[0] - 1, -1, dtype=np.int64)
        K.admit_members(ip, ix, a, k["centers"], k["bucket_ptr"], k["bucket_js"], cap, pr, v2a, 17)
        assert np.array_equal(pr, k[f"admit_{tag}_processed"]), tag
        assert np.array_equal(v2a, k[f"admit_{tag}_v2a"]), tag
    gp, gi, gv = K.galerkin_coo(ip, ix, a, k["agg_v2a"], k["agg_seeds"].shape[0])
    assert np.array_equal(gp, k["gal_indptr"]) and np.array_equal(gi, k["gal_indices"])
    assert np.array_equal(gv, k["gal_data"]), "Galerkin values not bit-exact"
    nc = k["agg_seeds"].shape[0]
    order = np.argsort(k["agg_v2a"], kind="stable")
    mptr = np.zeros(nc + 1, dtype=np.int64)
    mptr[1:] = np.cumsum(np.bincount(k["agg_v2a"], minlength=nc))
    assert np.array_equal(K.restrict(mptr, order, k["x"]), k["restrict"])
    assert np.array_equal(K.prolongate_add(k["agg_v2a"], k["e_coarse"], k["x"]), k["prolongate"])
    inv_m = 1.0 / k["l1_diag"]
    assert np.array_equal(K.smooth_sweeps(ip, ix, a, inv_m, k["x"], k["b"], 3), k["smooth3"])


def test_aggregate_bitexact(U, kern):
    k = kern
    A = _smat(U, k["indptr"], k["indices"], k["data"])
    agg = U.aggregate(A, U.AggregationConfig(seed=3))
    assert np.array_equal(agg.vertex_to_agg, k["agg_v2a"])
    assert np.array_equal(agg.coarse_vertex_of_agg, k["agg_seeds"])
    agg = U.aggregate(A, U.AggregationConfig(seed=9, size_cap=4))
    assert np.array_equal(agg.vertex_to_agg, k["aggcap4_v2a"])
    assert np.array_equal(agg.coarse_vertex_of_agg, k["aggcap4_seeds"])
    agg.validate(A, size_cap=4)


def _gpu_levels(h):
    out = []
    for lev in h.levels:
        m = lev.matrix
        ag = lev.aggregation
        out.append(dict(n=m.n_rows, indptr=m.indptr, indices=m.indices, data=m.data,
                        v2a=None if ag is None else ag.vertex_to_agg,
                        seeds=None if ag is None else ag.coarse_vertex_of_agg))
    return out


def _setup(U, case):
    ip, ix, a, g = problem_for(case)
    cfg = dict(CASE_CFG.get(case, {}))
    setup_kw = {k: cfg.pop(k) for k in ("n0", "max_levels") if k in cfg}
    h = U.setup(_smat(U, ip, ix, a), U.AggregationConfig(**cfg), **setup_kw)
    return h, g, ip


@pytest.mark.parametrize("case", HIERARCHY_CASES)
def test_hierarchy_bitexact(U, case):
    h, g, _ = _setup(U, case)
    assert h.singular == bool(g["singular"])
    assert_hierarchy_equal(g, _gpu_levels(h))
    assert abs(h.grid_complexity - float(g["grid_complexity"])) < 1e-12
    assert abs(h.operator_complexity - float(g["operator_complexity"])) < 1e-12


@pytest.mark.parametrize("case", HIERARCHY_CASES)
def test_solve_history(U, case):
    h, g, ip = _setup(U, case)
    b = g["b"] if g["b"].shape[0] else np.ones(ip.shape[0] - 1)
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=float(g["tol"]), max_iters=500)
    assert_history_close(rep.residual_history, g, rtol=RTOL)
    assert rep.converged == bool(g["converged"])
    if g["x"].shape[0]:
        np.testing.assert_allclose(x, g["x"], rtol=1e-7, atol=1e-9 * np.abs(g["x"]).max())


@pytest.mark.parametrize("prefix", list(SOLVE_VARIANTS))
def test_solve_variants(U, prefix):
    h, g, _ = _setup(U, "g2d_dir_64")
    kw = dict(SOLVE_VARIANTS[prefix])
    tol = kw.pop("tol", 1e-8)
    max_iters = kw.pop("max_iters", 500)
    spec = U.CycleSpec(**{k: v for k, v in kw.items() if k in ("kind", "inner_krylov_steps", "pre_sweeps",
                                                                  "post_sweeps")})
    sm = U.Smoother(kind=kw.get("smoother", "l1"), **({"omega": kw["omega"]} if "omega" in kw else {}))
    x0 = g[prefix + "x0"] if prefix + "x0" in g else None
    x, rep = U.npcg_solve(h, spec, sm, g["b"], tol=tol, max_iters=max_iters, x0=x0)
    assert_history_close(rep.residual_history, g, prefix=prefix, rtol=RTOL)


def test_graphs_match_stream_launches(U):
    h, g, _ = _setup(U, "g3d7_16")
    b = np.ones(16 ** 3)
    x1, r1 = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8, use_graphs=True)
    x2, r2 = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8, use_graphs=False)
    assert r1.residual_history == r2.residual_history
    assert np.array_equal(x1, x2)


def test_deterministic_repeat(U):
    h, g, _ = _setup(U, "rgg_20000")
    b = np.ones(20000)
    x1, r1 = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
    x2, r2 = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
    assert np.array_equal(x1, x2) and r1.residual_history == r2.residual_history


@pytest.mark.parametrize("seed,cap,ppl", [(0, None, 1), (11, 3, 1), (5, None, 2), (7, 7, 2)])
def test_random_graphs_vs_oracle(U, oracle, seed, cap, ppl):
    """Extra cases checked live against the CPU oracle (itself pinned to the
    reference): non-integer weights make every float sum order-sensitive."""
    rng = np.random.default_rng(seed)
    n = 1500
    from scipy.spatial import cKDTree
    Pt = rng.random((n, 2))
    pairs = cKDTree(Pt).query_pairs(np.sqrt(9.0 / (np.pi * n)), output_type="ndarray")
    w = rng.uniform(0.1, 3.0, pairs.shape[0])
    rows = np.concatenate([pairs[:, 0], pairs[:, 1]])
    cols = np.concatenate([pairs[:, 1], pairs[:, 0]])
    vals = np.concatenate([-w, -w])
    deg = np.bincount(rows, weights=-vals, minlength=n)
    diag = deg + rng.uniform(0.05, 0.5, n)
    A = U.SparseMatrix.from_coo(n, n, np.r_[rows, np.arange(n)], np.r_[cols, np.arange(n)], np.r_[vals, diag])
    kw = dict(seed=seed, size_cap=cap, passes_per_level=ppl)
    ho = oracle.setup(A.indptr, A.indices, A.data, **kw)
    hg = U.setup(A, U.AggregationConfig(**kw))
    assert hg.n_levels == ho.n_levels
    for Lg, Lo in zip(hg.levels, ho.levels):
        m = Lg.matrix
        assert np.array_equal(m.indptr, Lo.indptr) and np.array_equal(m.indices, Lo.indices)
        assert np.array_equal(m.data, Lo.data)
        if Lo.vertex_to_agg is not None:
            assert np.array_equal(Lg.aggregation.vertex_to_agg, Lo.vertex_to_agg)
            assert np.array_equal(Lg.aggregation.coarse_vertex_of_agg, Lo.coarse_vertex_of_agg)
    b = rng.standard_normal(n)
    xo, ro = oracle.npcg_solve(ho, b, tol=1e-10, max_iters=300)
    xg, rg = U.npcg_solve(hg, U.CycleSpec(), U.Smoother(), b, tol=1e-10, max_iters=300)
    assert abs(rg.iterations - ro.iterations) <= 1
    m = min(len(rg.residual_history), len(ro.residual_history))
    h1, h2 = np.array(rg.residual_history[:m]), np.array(ro.residual_history[:m])
    err = np.where(np.abs(h1 - h2) <= 1e-13, 0, np.abs(h1 - h2) / h2)
    assert err.max() <= 1e-10


@pytest.mark.parametrize("seed,weights,nhub,n", [(1, "int", 4, 4000), (2, "bigint", 4, 4000), (3, "float", 4, 4000),
                                                 (4, "bigint", 0, 4000), (5, "int", 12, 40000)])
def test_hub_graphs_vs_oracle(U, oracle, seed, weights, nhub, n):
    """Graphs with hub vertices (rows of 100-400 entries) checked live
    against the CPU oracle: the long-row team paths of the aggregation, the
    chunked global-table Galerkin (integer weights), the int64 shared-table
    Galerkin (weights ~2^24, no hubs) and the reference-ordered float path."""
    rng = np.random.default_rng(seed)
    from scipy.spatial import cKDTree
    Pt = rng.random((n, 2))
    pairs = cKDTree(Pt).query_pairs(np.sqrt(8.0 / (np.pi * n)), output_type="ndarray")
    hubs = rng.choice(n, nhub, replace=False)
    extra = [np.stack([np.full(k, h), rng.choice(n, k, replace=False)], 1)
             for h, k in zip(hubs, rng.integers(100, 400, hubs.size))]
    pairs = np.concatenate([pairs] + extra)
    pairs = pairs[pairs[:, 0] != pairs[:, 1]]
    pairs = np.unique(np.sort(pairs, 1), axis=0)
    if weights == "int":
        w = rng.integers(1, 4, pairs.shape[0]).astype(np.float64)
    elif weights == "bigint":
        w = rng.integers(1 << 23, 1 << 24, pairs.shape[0]).astype(np.float64)
    else:
        w = rng.uniform(0.1, 3.0, pairs.shape[0])
    rows = np.concatenate([pairs[:, 0], pairs[:, 1]])
    cols = np.concatenate([pairs[:, 1], pairs[:, 0]])
    vals = np.concatenate([-w, -w])
    deg = np.bincount(rows, weights=w[np.r_[np.arange(w.size), np.arange(w.size)]], minlength=n)
    diag = (deg + 1.0 if weights == "int" else np.floor(deg * 1.0625) + 1.0 if weights == "bigint"
            else deg + rng.uniform(0.05, 0.5, n))
    A = U.SparseMatrix.from_coo(n, n, np.r_[rows, np.arange(n)], np.r_[cols, np.arange(n)], np.r_[vals, diag])
    assert nhub == 0 or np.diff(A.indptr).max() > 64
    ho = oracle.setup(A.indptr, A.indices, A.data, seed=seed)
    hg = U.setup(A, U.AggregationConfig(seed=seed))
    assert hg.n_levels == ho.n_levels
    for Lg, Lo in zip(hg.levels, ho.levels):
        m = Lg.matrix
        assert np.array_equal(m.indptr, Lo.indptr) and np.array_equal(m.indices, Lo.indices)
        assert np.array_equal(m.data, Lo.data)
        if Lo.vertex_to_agg is not None:
            assert np.array_equal(Lg.aggregation.vertex_to_agg, Lo.vertex_to_agg)
    b = rng.standard_normal(n)
    xo, ro = oracle.npcg_solve(ho, b, tol=1e-10, max_iters=300)
    xg, rg = U.npcg_solve(hg, U.CycleSpec(), U.Smoother(), b, tol=1e-10, max_iters=300)
    assert abs(rg.iterations - ro.iterations) <= 1
    m = min(len(rg.residual_history), len(ro.residual_history))
    h1, h2 = np.array(rg.residual_history[:m]), np.array(ro.residual_history[:m])
    err = np.where(np.abs(h1 - h2) <= 1e-13, 0, np.abs(h1 - h2) / h2)
    assert err.max() <= 1e-10


def test_edge_cases(U):
    from paper_1302_2547_b200 import problems as P
    # n0 >= n: single level, direct solve
    A = P.grid2d(8)
    h = U.setup(A, n0=100)
    assert h.n_levels == 1
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), np.ones(64), tol=1e-12)
    assert rep.iterations == 1 and rep.converged
    # zero right-hand side
    h = U.setup(P.grid2d(24))
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), np.zeros(576))
    assert rep.iterations == 0 and rep.residual_history == [0.0] and not x.any()
    # max_iters cap
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), np.ones(576), tol=1e-30, max_iters=3)
    assert rep.iterations == 3 and not rep.converged
    # stagnation: no edges -> every vertex its own aggregate -> SetupError
    D = U.SparseMatrix(200, 200, np.arange(201), np.arange(200), np.full(200, 2.0))
    with pytest.raises(U.SetupError):
        U.setup(D)
    # singular hierarchy with an incompatible rhs -> NumericalError
    hn = U.setup(P.grid2d(16, "neumann"))
    assert hn.singular
    with pytest.raises(U.NumericalError):
        U.npcg_solve(hn, U.CycleSpec(), U.Smoother(), np.ones(256))
    # torch device input stays on device
    b = torch.ones(576, dtype=torch.float64, device="cuda")
    xd, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
    assert isinstance(xd, torch.Tensor) and xd.is_cuda


def test_c2_full_size_hierarchy_and_history(U):
    """BASELINE config C2 (3D 7-pt 128^3) at full size: hierarchy hashes and
    the residual history of the reference run."""
    ip, ix, a, g = problem_for("c2_grid3d7_128")
    h = U.setup(_smat(U, ip, ix, a))
    assert_hierarchy_equal(g, _gpu_levels(h))
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), np.ones(ip.shape[0] - 1), tol=1e-8, max_iters=500)
    assert_history_close(rep.residual_history, g, rtol=RTOL)


@pytest.mark.parametrize("dims,stencil,bc", [((5, 5, 5), 7, "dirichlet"), ((6, 4, 5), 27, "dirichlet"),
                                             ((4, 7, 3), 7, "neumann"), ((5, 6, 4), 27, "neumann")])
def test_device_grid_generator_matches_host(U, dims, stencil, bc):
    """On-device 3D lattice builder == host builder (== reference assembly)."""
    from paper_1302_2547_b200 import problems

    h = problems.grid3d(None, stencil, bc, dims=dims)
    d = problems.grid3d_device(None, stencil, bc, dims=dims).to_host()
    assert np.array_equal(h.indptr, d.indptr) and np.array_equal(h.indices, d.indices)
    assert np.array_equal(h.data, d.data)


def test_c2_bit_reproducible(U):
    """Run-to-run determinism at C2 (include/uaamg_b200.h: results do not
    depend on timing): three solves of one hierarchy and a solve of a fresh
    setup give identical residual-history bits and identical x.  Coarse
    levels have hub rows whose long-row pieces finish in arrival order; their
    reduced values are folded in row order (csr_group.cuh)."""
    from paper_1302_2547_b200 import problems
    A = problems.grid3d_device(128, 7)
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    runs = []
    h = U.setup(A)
    for k in range(4):
        if k == 3:
            h = U.setup(A)
        x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8, max_iters=500)
        runs.append((x.cpu().numpy().tobytes(), np.array(rep.residual_history).tobytes(), rep.iterations))
    assert all(r == runs[0] for r in runs[1:])


@pytest.mark.parametrize("level", [0, 1, 2, 3])
def test_cycle_bit_reproducible_without_tail(U, level, monkeypatch):
    """Every level's cycle repeats bit for bit with the separate-kernel coarse
    path too (the tail kernel off: long-row reductions through the group
    kernel's per-row slots)."""
    from paper_1302_2547_b200 import problems
    monkeypatch.setenv("UAAMG_NO_TAIL", "1")
    h = U.setup(problems.grid3d_device(64, 7))
    if level >= h.n_levels - 1:
        pytest.skip("level has no coarser level")
    g = torch.Generator().manual_seed(level)
    b = torch.rand(h.levels[level].n, generator=g, dtype=torch.float64).cuda()
    outs = {U.cycle(h, U.CycleSpec(), U.Smoother(), level, b).cpu().numpy().tobytes() for _ in range(4)}
    assert len(outs) == 1


@pytest.mark.parametrize("seed", [0, 1])
def test_aggregate_nonsymmetric_pattern_vs_oracle(U, oracle, seed):
    """the admission sweeps' neighbour shortcut assumes a
    structurally symmetric pattern; setup checks the pattern and takes the
    plain fixpoint otherwise.  A Laplacian with 15% of its upper entries
    dropped must aggregate exactly like the reference's row-based rule."""
    from paper_1302_2547_b200 import problems
    A = problems.grid2d(48)
    rng = np.random.default_rng(seed)
    r = np.repeat(np.arange(A.n_rows), np.diff(A.indptr))
    drop = (A.indices > r) & (rng.random(A.nnz) < 0.15)
    M = U.SparseMatrix.from_coo(A.n_rows, A.n_rows, r[~drop], A.indices[~drop], A.data[~drop])
    for cfg in (dict(seed=3), dict(seed=9, max_passes=4)):
        agg = U.aggregate(M, U.AggregationConfig(**cfg))
        v2a, seeds = oracle.aggregate(M.indptr, M.indices, M.data, **cfg)
        assert np.array_equal(agg.vertex_to_agg, v2a)
        assert np.array_equal(agg.coarse_vertex_of_agg, seeds)


def test_27pt_tma64_level0_vs_oracle(U, oracle):
    """27-point rows (27 x 128 > the TMA stage) take 64-row TMA tiles; the
    hierarchy and history must still match the oracle (rows folded in
    reference order, bit-exact sums)."""
    from paper_1302_2547_b200 import problems
    A = problems.grid3d(48, 27)
    h = U.setup(A)
    ho = oracle.setup(A.indptr, A.indices, A.data)
    assert h.n_levels == ho.n_levels
    for Lg, Lo in zip(h.levels[1:], ho.levels[1:]):
        m = Lg.matrix
        assert np.array_equal(m.indptr, Lo.indptr) and np.array_equal(m.indices, Lo.indices)
        assert np.array_equal(m.data, Lo.data)
    b = np.ones(A.n_rows)
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-10, max_iters=300)
    xo, ro = oracle.npcg_solve(ho, b, tol=1e-10, max_iters=300)
    assert rep.iterations == ro.iterations
    h1, h2 = np.array(rep.residual_history), np.array(ro.residual_history)
    err = np.where(np.abs(h1 - h2) <= 1e-13, 0, np.abs(h1 - h2) / h2)
    assert err.max() <= 1e-10


def test_ell_level0_matches_tile_kernels(U, oracle):
    """27-point level 0 above 2^20 rows takes the sliced-ELL copy
    (csr_ell.cuh); the solve equals the tile-kernel path (UAAMG_NO_ELL) --
    same row sums (reference order), so the histories differ only by the
    dot products' reduction tree.  (Full size: test_gpu_fullsize C4.)"""
    import ctypes
    import os
    from paper_1302_2547_b200 import _lib, problems

    def kind(h, l):
        k = ctypes.c_int()
        _lib.check(_lib.load().uaamg_level_kernel(h._handle, l, ctypes.byref(k)))
        return k.value
    A = problems.grid3d_device(104, 27)  # 1,124,864 rows
    out = {}
    for mode in ("ell", "tiles"):
        if mode == "tiles":
            os.environ["UAAMG_NO_ELL"] = "1"
        try:
            h = U.setup(A)
            assert kind(h, 0) == (3 if mode == "ell" else 1)
            b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
            x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-10, max_iters=300)
            out[mode] = (x.cpu().numpy(), np.asarray(rep.residual_history), [l.n for l in h.levels])
        finally:
            os.environ.pop("UAAMG_NO_ELL", None)
    assert out["ell"][2] == out["tiles"][2]
    h1, h2 = out["ell"][1], out["tiles"][1]
    assert len(h1) == len(h2)
    assert np.max(np.abs(h1 - h2) / np.abs(h2)) < 1e-12
    np.testing.assert_allclose(out["ell"][0], out["tiles"][0], rtol=1e-9, atol=1e-12)


def test_ell_cycle_bit_identical_float_weights(U):
    """Float-weighted 27-point operator above 2^20 rows (random symmetric
    weights, diagonally dominant): one K-cycle on level 0 through the
    sliced-ELL copy is BIT-identical to the tile-kernel path -- every row is
    folded in CSR order without FMA in both, and the cycle's dots live on the
    coarse levels, which do not change."""
    import ctypes
    import os
    from paper_1302_2547_b200 import _lib, problems
    A0 = problems.grid3d(104, 27)
    n = A0.n_rows
    rows = np.repeat(np.arange(n), np.diff(A0.indptr))
    cols = A0.indices
    lo, hi = np.minimum(rows, cols).astype(np.uint64), np.maximum(rows, cols).astype(np.uint64)
    h64 = (lo * np.uint64(0x9E3779B97F4A7C15) + hi * np.uint64(0xBF58476D1CE4E5B9)) >> np.uint64(11)
    w = 0.5 + h64.astype(np.float64) / float(1 << 53)  # symmetric, in [0.5, 1.5)
    data = np.where(rows == cols, 0.0, -w)
    diag = np.zeros(n)
    np.add.at(diag, rows, np.abs(data))
    data = np.where(rows == cols, diag[rows] + 0.25, data)
    A = U.SparseMatrix(n, n, A0.indptr, A0.indices, data)
    b = np.sin(np.arange(n) * 0.001) + 1.0
    out = {}
    for mode in ("ell", "tiles"):
        if mode == "tiles":
            os.environ["UAAMG_NO_ELL"] = "1"
        try:
            h = U.setup(A.device())
            k = ctypes.c_int()
            _lib.check(_lib.load().uaamg_level_kernel(h._handle, 0, ctypes.byref(k)))
            assert k.value == (3 if mode == "ell" else 1)
            out[mode] = U.cycle(h, U.CycleSpec(), U.Smoother(), 0, b)
        finally:
            os.environ.pop("UAAMG_NO_ELL", None)
    assert np.array_equal(out["ell"], out["tiles"])


def test_rowpar_cycle_bit_identical_float_weights(U):
    """Float-weighted 7-point operator (rows of <= 7 entries): one K-cycle on
    level 0 through the row-parallel TMA kernel is BIT-identical to the
    warp-gather tile kernel (UAAMG_NO_ROWPAR) -- same in-order folds."""
    import ctypes
    import os
    from paper_1302_2547_b200 import _lib, problems
    A0 = problems.grid3d(96, 7)
    n = A0.n_rows
    rows = np.repeat(np.arange(n), np.diff(A0.indptr))
    cols = A0.indices
    lo, hi = np.minimum(rows, cols).astype(np.uint64), np.maximum(rows, cols).astype(np.uint64)
    h64 = (lo * np.uint64(0x9E3779B97F4A7C15) + hi * np.uint64(0xBF58476D1CE4E5B9)) >> np.uint64(11)
    w = 0.5 + h64.astype(np.float64) / float(1 << 53)
    data = np.where(rows == cols, 0.0, -w)
    diag = np.zeros(n)
    np.add.at(diag, rows, np.abs(data))
    data = np.where(rows == cols, diag[rows] + 0.25, data)
    A = U.SparseMatrix(n, n, A0.indptr, A0.indices, data)
    b = np.cos(np.arange(n) * 0.003) + 1.0
    out = {}
    for mode in ("rowpar", "warp"):
        if mode == "warp":
            os.environ["UAAMG_NO_ROWPAR"] = "1"
        try:
            h = U.setup(A.device())
            k = ctypes.c_int()
            _lib.check(_lib.load().uaamg_level_kernel(h._handle, 0, ctypes.byref(k)))
            assert k.value == (2 if mode == "rowpar" else 1)
            out[mode] = U.cycle(h, U.CycleSpec(), U.Smoother(), 0, b)
        finally:
            os.environ.pop("UAAMG_NO_ROWPAR", None)
    assert np.array_equal(out["rowpar"], out["warp"])
