"""Row-partitioned setup and solve, run as P virtual ranks on one GPU
(csrc/dist_setup.cu, csrc/dist_solve.cu).

Partition invariance, the north star's bar:
* the hierarchy -- aggregation maps, seeds, every coarse level's pattern and
  values -- is bit-identical to the reference's (golden fixtures) for every
  rank count, with coarse levels sharded too (small shard_rows);
* residual histories match the reference's within 1e-10 and the
  single-device solve within round-off (only the dot products are folded
  per rank and then across ranks), iterations identical.
"""
import numpy as np
import pytest

from golden_util import assert_hierarchy_equal, assert_history_close, problem_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def U():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1302_2547_b200 as U

    return U


@pytest.fixture(scope="module")
def D():
    from paper_1302_2547_b200 import distributed as D
    return D


def _smat(U, ip, ix, a):
    return U.SparseMatrix(ip.shape[0] - 1, ip.shape[0] - 1, ip, ix, a)


def _levels(dh):
    out = []
    for l in range(dh.n_levels):
        m = dh.level_matrix(l)
        ag = dh.level_aggregation(l)
        out.append(dict(n=m.n_rows, indptr=m.indptr, indices=m.indices, data=m.data,
                        v2a=None if ag is None else ag[0], seeds=None if ag is None else ag[1]))
    return out


@pytest.mark.parametrize("case", ["c1_grid2d_256", "g3d7_16", "rgg_20000", "wgraph_3000", "g2d_aniso_48"])
@pytest.mark.parametrize("ranks", [1, 2, 3, 8])
def test_sharded_setup_bitexact_and_history(U, D, case, ranks):
    from golden_util import CASE_CFG
    ip, ix, a, g = problem_for(case)
    cfg = dict(CASE_CFG.get(case, {}))
    A = _smat(U, ip, ix, a)
    # shard every level with >= 200 rows, so coarse levels are sharded too
    dh = D.setup_distributed(A, ranks=ranks, shard_rows=200, config=U.AggregationConfig(**cfg))
    assert dh.n_sharded >= 1
    assert dh.singular == bool(g["singular"])
    assert_hierarchy_equal(g, _levels(dh))
    assert abs(dh.grid_complexity - float(g["grid_complexity"])) < 1e-12
    assert abs(dh.operator_complexity - float(g["operator_complexity"])) < 1e-12
    b = g["b"] if g["b"].shape[0] else np.ones(ip.shape[0] - 1)
    tol = float(g["tol"])
    h = U.setup(A, U.AggregationConfig(**cfg))
    x1, r1 = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=tol, max_iters=500)
    xs, rs = D.npcg_solve_distributed(dh, U.CycleSpec(), U.Smoother(), b, tol=tol, max_iters=500)
    assert_history_close(rs.residual_history, g, rtol=1e-10)
    assert rs.iterations == r1.iterations
    h1 = np.asarray(r1.residual_history)
    hs = np.asarray(rs.residual_history)
    assert np.all(np.abs(hs - h1) <= 1e-12 * np.abs(h1) + 1e-15)
    np.testing.assert_allclose(xs, x1, rtol=1e-9, atol=1e-12 * np.abs(x1).max())


@pytest.mark.parametrize("kw", [{"kind": "vcycle"}, {"pre_sweeps": 2, "post_sweeps": 2}, {"inner_krylov_steps": 3},
                                {"pre_sweeps": 0}, {"inner_krylov_steps": 0}])
def test_sharded_variants_match_single_device(U, D, kw):
    ip, ix, a, g = problem_for("g2d_dir_64")
    A = _smat(U, ip, ix, a)
    h = U.setup(A)
    dh = D.setup_distributed(A, ranks=4, shard_rows=200)
    b = np.ones(ip.shape[0] - 1)
    spec = U.CycleSpec(**kw)
    x1, r1 = U.npcg_solve(h, spec, U.Smoother(), b, tol=1e-10, max_iters=300)
    xs, rs = D.npcg_solve_distributed(dh, spec, U.Smoother(), b, tol=1e-10, max_iters=300)
    assert rs.iterations == r1.iterations
    h1 = np.asarray(r1.residual_history)
    hs = np.asarray(rs.residual_history)
    assert np.all(np.abs(hs - h1) <= 1e-10 * np.abs(h1) + 1e-15)


def test_sharded_x0_and_jacobi(U, D):
    ip, ix, a, g = problem_for("g3d7_16")
    A = _smat(U, ip, ix, a)
    h = U.setup(A)
    dh = D.setup_distributed(A, ranks=5, shard_rows=100)
    n = ip.shape[0] - 1
    rng = np.random.default_rng(3)
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    sm = U.Smoother(kind="jacobi")
    x1, r1 = U.npcg_solve(h, U.CycleSpec(), sm, b, tol=1e-9, max_iters=200, x0=x0)
    xs, rs = D.npcg_solve_distributed(dh, U.CycleSpec(), sm, b, tol=1e-9, max_iters=200, x0=x0)
    assert rs.iterations == r1.iterations
    np.testing.assert_allclose(rs.residual_history, r1.residual_history, rtol=1e-10, atol=1e-15)


def test_sharded_repeat_is_bit_reproducible(U, D):
    """Repeated solves, and graph replays vs plain launches, give the same bits."""
    ip, ix, a, g = problem_for("rgg_20000")
    dh = D.setup_distributed(_smat(U, ip, ix, a), ranks=3, shard_rows=500)
    b = np.ones(ip.shape[0] - 1)
    r = [D.npcg_solve_distributed(dh, U.CycleSpec(), U.Smoother(), b, tol=1e-8, use_graphs=k != 1)
         for k in range(3)]
    assert r[0][1].residual_history == r[1][1].residual_history == r[2][1].residual_history
    assert np.array_equal(r[0][0], r[1][0]) and np.array_equal(r[0][0], r[2][0])


def test_sharded_c2_full_size(U, D):
    """C2 (128^3) over 8 ranks: level 0 sharded (default shard_rows = 2^20),
    or levels 0 and 1 (shard_rows = 2^18), the rest replicated; hierarchy
    SHA-identical to the reference's, history within 1e-10."""
    ip, ix, a, g = problem_for("c2_grid3d7_128")
    for shard_rows, ns in ((1 << 20, 1), (1 << 18, 2)):
        dh = D.setup_distributed(_smat(U, ip, ix, a), ranks=8, shard_rows=shard_rows)
        assert dh.n_sharded == ns
        assert_hierarchy_equal(g, _levels(dh))
        xs, rs = D.npcg_solve_distributed(dh, U.CycleSpec(), U.Smoother(), np.ones(ip.shape[0] - 1), tol=1e-8,
                                          max_iters=500)
        assert_history_close(rs.residual_history, g, rtol=1e-10)
        assert rs.iterations == int(g["iterations"])
        dh.close()


def test_sharded_errors(U, D):
    from paper_1302_2547_b200 import problems
    A = problems.grid2d(32)
    with pytest.raises(NotImplementedError):
        D.setup_distributed(A, ranks=2, shard_rows=100, config=U.AggregationConfig(size_cap=4))
    # stagnation: the reference's SetupError, with the global level index
    Dg = U.SparseMatrix(400, 400, np.arange(401), np.arange(400), np.full(400, 2.0))
    with pytest.raises(U.SetupError, match="level 0"):
        D.setup_distributed(Dg, ranks=2, shard_rows=100)
    # singular (Neumann): a right-hand side with a null-space component
    dh = D.setup_distributed(problems.grid2d(32, "neumann"), ranks=2, shard_rows=100)
    assert dh.singular
    with pytest.raises(U.NumericalError):
        D.npcg_solve_distributed(dh, U.CycleSpec(), U.Smoother(), np.ones(1024))


@pytest.mark.parametrize("ranks", [2, 3, 8])
@pytest.mark.parametrize("kind", ["kcycle", "vcycle"])
def test_sharded_singular_neumann(U, D, ranks, kind):
    """Neumann (singular) hierarchy: _check_compatible / _project_mean
    (U/solvers.py:112-125) folded across ranks; the reference's history
    within 1e-10, the single-device solve within round-off."""
    ip, ix, a, g = problem_for("g2d_neu_32")
    A = _smat(U, ip, ix, a)
    dh = D.setup_distributed(A, ranks=ranks, shard_rows=100)
    assert dh.singular and dh.n_sharded >= 2
    assert_hierarchy_equal(g, _levels(dh))
    spec = U.CycleSpec(kind=kind)
    prefix = "" if kind == "kcycle" else "vcycle_"
    xs, rs = D.npcg_solve_distributed(dh, spec, U.Smoother(), g["b"], tol=float(g["tol"]), max_iters=500)
    assert_history_close(rs.residual_history, g, prefix=prefix, rtol=1e-10)
    h = U.setup(A)
    x1, r1 = U.npcg_solve(h, spec, U.Smoother(), g["b"], tol=float(g["tol"]), max_iters=500)
    assert rs.iterations == r1.iterations
    np.testing.assert_allclose(rs.residual_history, r1.residual_history, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(xs, x1, rtol=1e-9, atol=1e-12 * np.abs(x1).max())


def test_sharded_ell_shard_matches_single_device(U, D):
    """A 27-point level 0 whose shard has >= 2^20 rows: the shard gets its
    own sliced-ELL copy (csr_ell.cuh, global-row-indexed rows [a, a + n));
    iterations equal and history within round-off of the single-device
    solve (which takes the ELL copy too)."""
    import torch
    from paper_1302_2547_b200 import problems
    A = problems.grid3d_device(104, 27)  # 1,124,864 rows
    h = U.setup(A)
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    x1, r1 = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-9, max_iters=300)
    dh = D.setup_distributed(A, ranks=1)
    xs, rs = D.npcg_solve_distributed(dh, U.CycleSpec(), U.Smoother(), b, tol=1e-9, max_iters=300)
    assert rs.iterations == r1.iterations
    h1 = np.asarray(r1.residual_history)
    hs = np.asarray(rs.residual_history)
    assert np.all(np.abs(hs - h1) <= 1e-12 * np.abs(h1) + 1e-15)
    dh.close()
