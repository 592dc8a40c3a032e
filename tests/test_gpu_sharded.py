"""Row-partitioned (multi-rank) solve, run as P virtual ranks on one GPU
(paper_1302_2547_b200/csrc/shard.cu).

Partition invariance: for P = 1..8 the residual history must match the
reference's (golden fixtures) within the solve's 1e-10 bar and the
single-device solve within round-off -- every SpMV row and restriction sum is
computed in the same order as on one device; only the dot products are
folded per rank and then across ranks.
"""
import numpy as np
import pytest

from golden_util import assert_history_close, problem_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def U():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1302_2547_b200 as U

    return U


def _smat(U, ip, ix, a):
    return U.SparseMatrix(ip.shape[0] - 1, ip.shape[0] - 1, ip, ix, a)


@pytest.mark.parametrize("case", ["c1_grid2d_256", "g3d7_16", "rgg_20000"])
@pytest.mark.parametrize("ranks", [1, 2, 3, 8])
def test_sharded_history_matches_reference(U, case, ranks):
    ip, ix, a, g = problem_for(case)
    h = U.setup(_smat(U, ip, ix, a))
    b = g["b"] if g["b"].shape[0] else np.ones(ip.shape[0] - 1)
    tol = float(g["tol"])
    x1, r1 = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=tol, max_iters=500)
    # shard every level with >= 1000 rows so coarse levels are sharded too
    xs, rs = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=tol, max_iters=500, ranks=ranks,
                          shard_rows=1000)
    assert_history_close(rs.residual_history, g, rtol=1e-10)
    assert rs.iterations == r1.iterations
    h1 = np.asarray(r1.residual_history)
    hs = np.asarray(rs.residual_history)
    assert np.all(np.abs(hs - h1) <= 1e-12 * np.abs(h1) + 1e-15)
    np.testing.assert_allclose(xs, x1, rtol=1e-9, atol=1e-12 * np.abs(x1).max())


@pytest.mark.parametrize("kw", [{"kind": "vcycle"}, {"pre_sweeps": 2, "post_sweeps": 2}, {"inner_krylov_steps": 3},
                                {"pre_sweeps": 0}])
def test_sharded_variants_match_single_device(U, kw):
    ip, ix, a, g = problem_for("g2d_dir_64")
    h = U.setup(_smat(U, ip, ix, a))
    b = np.ones(ip.shape[0] - 1)
    spec = U.CycleSpec(**kw)
    x1, r1 = U.npcg_solve(h, spec, U.Smoother(), b, tol=1e-10, max_iters=300)
    xs, rs = U.npcg_solve(h, spec, U.Smoother(), b, tol=1e-10, max_iters=300, ranks=4, shard_rows=200)
    assert rs.iterations == r1.iterations
    h1 = np.asarray(r1.residual_history)
    hs = np.asarray(rs.residual_history)
    assert np.all(np.abs(hs - h1) <= 1e-10 * np.abs(h1) + 1e-15)


def test_sharded_x0_and_jacobi(U):
    ip, ix, a, g = problem_for("g3d7_16")
    h = U.setup(_smat(U, ip, ix, a))
    n = ip.shape[0] - 1
    rng = np.random.default_rng(3)
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    sm = U.Smoother(kind="jacobi")
    x1, r1 = U.npcg_solve(h, U.CycleSpec(), sm, b, tol=1e-9, max_iters=200, x0=x0)
    xs, rs = U.npcg_solve(h, U.CycleSpec(), sm, b, tol=1e-9, max_iters=200, x0=x0, ranks=5, shard_rows=100)
    assert rs.iterations == r1.iterations
    np.testing.assert_allclose(rs.residual_history, r1.residual_history, rtol=1e-10, atol=1e-15)


def test_sharded_c2_full_size(U):
    """C2 (128^3): levels 0 and 1 sharded over 8 ranks, the rest replicated."""
    ip, ix, a, g = problem_for("c2_grid3d7_128")
    h = U.setup(_smat(U, ip, ix, a))
    b = np.ones(ip.shape[0] - 1)
    xs, rs = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8, max_iters=500, ranks=8)
    assert_history_close(rs.residual_history, g, rtol=1e-10)
