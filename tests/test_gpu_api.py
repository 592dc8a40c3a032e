"""Public-API completeness against the reference (U/__init__.py): the
squared-pattern chain, CoarseSolver(a, singular) with matrix right-hand
sides, and the level-0 aliasing rules of setup()."""

import gc

import numpy as np
import pytest
import scipy.linalg
import torch

from golden_util import load, problem_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def U():
    import paper_1302_2547_b200 as U
    assert torch.cuda.is_available()
    return U


def test_squared_adjacency_pattern_chain(U):
    """U/sparse.py:121-129 + U/aggregation.py:136-141:
    select_coarse_vertices(squared_adjacency_pattern(a), s, processed)."""
    k = load("kernels")
    A = U.SparseMatrix(k["indptr"].shape[0] - 1, k["indptr"].shape[0] - 1, k["indptr"], k["indices"], k["data"])
    A2 = U.squared_adjacency_pattern(A)
    assert np.array_equal(A2.indptr, k["a2_indptr"]) and np.array_equal(A2.indices, k["a2_indices"])
    assert np.all(A2.data == 1.0)
    ctr = U.select_coarse_vertices(A2, k["scores_s7_p3"], k["processed"])
    assert np.array_equal(ctr, np.flatnonzero(k["select"]))
    with pytest.raises(ValueError):
        U.squared_adjacency_pattern(U.SparseMatrix(2, 3, [0, 1, 2], [0, 1], [1.0, 1.0]))


def _spd(U, n, seed):
    from paper_1302_2547_b200 import problems
    return problems.grid2d(n)


@pytest.mark.parametrize("nrhs", [None, 1, 7])
def test_coarse_solver_spd_matches_cholesky(U, nrhs):
    A = _spd(U, 9, 0)  # 81 x 81 Dirichlet Laplacian
    rng = np.random.default_rng(3)
    b = rng.standard_normal(81) if nrhs is None else rng.standard_normal((81, nrhs))
    s = U.CoarseSolver(A, False)
    assert not s.singular
    x = s.solve(b)
    ref = scipy.linalg.cho_solve(scipy.linalg.cho_factor(A.to_dense()), b)
    assert x.shape == b.shape
    np.testing.assert_allclose(x, ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())


def test_coarse_solver_singular_pseudo_inverse(U):
    from paper_1302_2547_b200 import problems
    A = problems.grid2d(6, "neumann")
    dense = A.to_dense()
    rng = np.random.default_rng(4)
    b = rng.standard_normal((36, 3))
    b -= b.mean(axis=0)
    vals, vecs = np.linalg.eigh(dense)
    cut = 1e-12 * max(vals[-1], 0.0)
    inv = np.where(vals > cut, 1.0 / np.where(vals > cut, vals, 1.0), 0.0)
    ref = vecs @ (inv[:, None] * (vecs.T @ b))
    s = U.CoarseSolver(A, True)
    assert s.singular
    np.testing.assert_allclose(s.solve(b), ref, rtol=1e-9, atol=1e-11 * np.abs(ref).max())
    # Cholesky failure (indefinite): the reference flips singular to True and
    # uses the pseudo-inverse, which drops the non-positive eigenvalues
    D = U.SparseMatrix(3, 3, [0, 1, 2, 3], [0, 1, 2], [2.0, -1.0, 4.0])
    s = U.CoarseSolver(D, False)
    assert s.singular
    np.testing.assert_allclose(s.solve(np.array([1.0, 1.0, 1.0])), [0.5, 0.0, 0.25], rtol=1e-14, atol=1e-15)


def test_coarse_solver_empty_and_device(U):
    s = U.CoarseSolver(U.SparseMatrix(0, 0, [0], [], []), False)
    assert s.solve(np.zeros(0)).shape == (0,)
    A = _spd(U, 5, 0)
    s = U.CoarseSolver(A.device(), False)
    bd = torch.ones(25, dtype=torch.float64, device="cuda")
    xd = s.solve(bd)
    assert isinstance(xd, torch.Tensor) and xd.is_cuda
    np.testing.assert_allclose(A.spmv(xd.cpu().numpy()), np.ones(25), rtol=1e-12)


def test_hierarchy_coarsest_solver_outlives_hierarchy(U):
    """`s = setup(A).coarsest_solver; s.solve(b)` must work."""
    from paper_1302_2547_b200 import problems
    A = problems.grid2d(40)
    s = U.setup(A).coarsest_solver
    gc.collect()
    b = np.ones(s.n)
    x = s.solve(b)
    assert x.shape == (s.n,) and np.all(np.isfinite(x))
    h = U.setup(A)
    Ac = h.levels[-1].matrix
    np.testing.assert_allclose(Ac.to_dense() @ x, b, rtol=1e-10, atol=1e-10)


def test_setup_copies_unaligned_or_unpadded_level0(U):
    """setup() aliases a device matrix only when the level-0 tile kernel may
    bulk-copy it in place (aligned, 64 readable bytes past the end); slices
    and exact-size tensors are copied -- same hierarchy either way."""
    ip, ix, a, g = problem_for("g2d_dir_64")
    ref = U.setup(U.SparseMatrix(ip.shape[0] - 1, ip.shape[0] - 1, ip, ix, a))
    dev = torch.device("cuda")
    # exact-size tensors (no slack) and an offset view (misaligned by 4 bytes)
    rp = torch.from_numpy(ip.astype(np.int32)).to(dev)
    big = torch.zeros(ix.shape[0] + 1, dtype=torch.int32, device=dev)
    big[1:] = torch.from_numpy(ix.astype(np.int32)).to(dev)
    ci = big[1:]
    av = torch.from_numpy(a).to(dev)
    d = U.DeviceCSR(ip.shape[0] - 1, ip.shape[0] - 1, rp, ci, av)
    assert not d.borrowable()
    h = U.setup(d)
    for L1, L2 in zip(h.levels, ref.levels):
        assert np.array_equal(L1.matrix.data, L2.matrix.data)
    x1, r1 = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), np.ones(ip.shape[0] - 1), tol=1e-8)
    x2, r2 = U.npcg_solve(ref, U.CycleSpec(), U.Smoother(), np.ones(ip.shape[0] - 1), tol=1e-8)
    assert r1.residual_history == r2.residual_history
    assert U.DeviceCSR.from_host(ref.levels[0].matrix).borrowable()


def _hier_state(h):
    out = []
    for lev in h.levels:
        m = lev.matrix
        ag = lev.aggregation
        out.append((m.indptr.tobytes(), m.indices.tobytes(), m.data.tobytes(),
                    None if ag is None else (ag.vertex_to_agg.tobytes(), ag.coarse_vertex_of_agg.tobytes())))
    return out, h.singular


@pytest.mark.parametrize("case,cfg", [("c1_grid2d_256", {}), ("g2d_neu_32", {}), ("g3d7_16", {"size_cap": 4}),
                                      ("g2d_dir_64", {"passes_per_level": 2}), ("wgraph_3000", {})])
def test_setup_from_host_layout_matches_device_input(U, case, cfg):
    """setup() on the reference's host SparseMatrix goes through
    uaamg_setup_host (int64 arrays staged and narrowed by the library, the
    values uploaded while level 0 aggregates): the same hierarchy bits and
    the same solve bits as setup() on a device CSR."""
    ip, ix, a, g = problem_for(case)
    n = ip.shape[0] - 1
    A = U.SparseMatrix(n, n, ip, ix, a)
    assert A._device is None
    h_host = U.setup(A, U.AggregationConfig(**cfg))
    assert A._device is None  # the host path does not leave a cached device copy
    h_dev = U.setup(U.SparseMatrix(n, n, ip, ix, a).device(), U.AggregationConfig(**cfg))
    assert _hier_state(h_host) == _hier_state(h_dev)
    b = g["b"] if g["b"].shape[0] else np.ones(n)
    x1, r1 = U.npcg_solve(h_host, U.CycleSpec(), U.Smoother(), b, tol=float(g["tol"]), max_iters=500)
    x2, r2 = U.npcg_solve(h_dev, U.CycleSpec(), U.Smoother(), b, tol=float(g["tol"]), max_iters=500)
    assert r1.residual_history == r2.residual_history and np.array_equal(x1, x2)


def test_setup_from_host_layout_single_level_and_errors(U):
    from paper_1302_2547_b200 import problems
    A = problems.grid2d(8)  # 64 rows <= n0: one level, no aggregation to overlap
    h = U.setup(U.SparseMatrix(A.n_rows, A.n_cols, A.indptr, A.indices, A.data))
    assert h.n_levels == 1 and not h.singular
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), np.ones(64), tol=1e-10)
    assert rep.converged
    Dg = U.SparseMatrix(400, 400, np.arange(401), np.arange(400), np.full(400, 2.0))
    with pytest.raises(U.SetupError, match="level 0"):
        U.setup(Dg)
