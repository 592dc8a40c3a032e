"""Pin the CPU oracle (oracle/uaamg_oracle.c) against the reference itself.

Fixtures in tests/golden/ were produced by running the unmodified reference
package (tests/golden/make_golden.py).  Kernels and hierarchies must match
bit-for-bit; residual histories within 1e-10 relative (the reference's dots go
through OpenBLAS, whose summation order is thread-count dependent).
"""

import numpy as np
import pytest

from golden_util import (CASE_CFG, HIERARCHY_CASES, SOLVE_VARIANTS, assert_hierarchy_equal,
                         assert_history_close, load, problem_for)


@pytest.fixture(scope="module")
def kern():
    return load("kernels")


def test_kernel_table_bitexact(oracle, kern):
    k = kern
    ip, ix, a = k["indptr"], k["indices"], k["data"]
    assert np.array_equal(oracle.spmv(ip, ix, a, k["x"]), k["spmv"])
    assert np.array_equal(oracle.diag_of(ip, ix, a), k["diag_of"])
    assert np.array_equal(oracle.l1_diag(ip, ix, a), k["l1_diag"])
    assert np.array_equal(oracle.degrees(ip, ix), k["degrees"])
    assert np.array_equal(oracle.hash_u01(0xDEADBEEF12345678, 5, k["hash_idx"]), k["hash_u01"])
    assert np.array_equal(oracle.quasi_random_scores(ip, ix, 0, 0), k["scores_p0"])
    assert np.array_equal(oracle.quasi_random_scores(ip, ix, 7, 3), k["scores_s7_p3"])
    p2, x2 = oracle.squared_pattern(ip.shape[0] - 1, ip, ix)
    assert np.array_equal(p2, k["a2_indptr"]) and np.array_equal(x2, k["a2_indices"])
    ctr = oracle.select_centers(p2, x2, k["scores_s7_p3"], k["processed"])
    assert np.array_equal(ctr, k["select"])
    own = oracle.claim_owners(p2, x2, k["scores_s7_p3"], k["processed"], ctr)
    assert np.array_equal(own, k["claim"])
    for tag, cap in (("cap3", 3), ("uncapped", 1 << 62)):
        pr = k["processed"].astype(np.uint8)
        v2a = np.full(ip.shape[0] - 1, -1, dtype=np.int64)
        oracle.admit_members(ip, ix, a, k["centers"], k["bucket_ptr"], k["bucket_js"], cap, pr, v2a, 17)
        assert np.array_equal(pr.astype(bool), k[f"admit_{tag}_processed"])
        assert np.array_equal(v2a, k[f"admit_{tag}_v2a"])
    v2a, seeds = oracle.aggregate(ip, ix, a, seed=3)
    assert np.array_equal(v2a, k["agg_v2a"]) and np.array_equal(seeds, k["agg_seeds"])
    v2a, seeds = oracle.aggregate(ip, ix, a, seed=9, size_cap=4)
    assert np.array_equal(v2a, k["aggcap4_v2a"]) and np.array_equal(seeds, k["aggcap4_seeds"])
    gp, gi, gv = oracle.galerkin_coo(ip, ix, a, k["agg_v2a"], k["agg_seeds"].shape[0])
    assert np.array_equal(gp, k["gal_indptr"]) and np.array_equal(gi, k["gal_indices"])
    assert np.array_equal(gv, k["gal_data"])
    nc = k["agg_seeds"].shape[0]
    order = np.argsort(k["agg_v2a"], kind="stable")
    mptr = np.zeros(nc + 1, dtype=np.int64)
    mptr[1:] = np.cumsum(np.bincount(k["agg_v2a"], minlength=nc))
    assert np.array_equal(oracle.restrict(mptr, order, k["x"]), k["restrict"])
    assert np.array_equal(oracle.prolongate_add(k["agg_v2a"], k["e_coarse"], k["x"]), k["prolongate"])
    inv_m = 1.0 / k["l1_diag"]
    assert np.array_equal(oracle.smooth_sweeps(ip, ix, a, inv_m, k["x"], k["b"], 3), k["smooth3"])


def _oracle_levels(h):
    return [dict(n=L.n, indptr=L.indptr, indices=L.indices, data=L.data,
                 v2a=L.vertex_to_agg, seeds=L.coarse_vertex_of_agg) for L in h.levels]


@pytest.mark.parametrize("case", HIERARCHY_CASES)
def test_hierarchy_bitexact(oracle, case):
    ip, ix, a, g = problem_for(case)
    h = oracle.setup(ip, ix, a, **CASE_CFG.get(case, {}))
    assert h.singular == bool(g["singular"])
    assert_hierarchy_equal(g, _oracle_levels(h))


@pytest.mark.parametrize("case", HIERARCHY_CASES)
def test_solve_history(oracle, case):
    ip, ix, a, g = problem_for(case)
    h = oracle.setup(ip, ix, a, **CASE_CFG.get(case, {}))
    b = g["b"] if g["b"].shape[0] else np.ones(ip.shape[0] - 1)
    x, rep = oracle.npcg_solve(h, b, tol=float(g["tol"]), max_iters=500)
    assert_history_close(rep.residual_history, g, rtol=1e-10)
    if g["x"].shape[0]:
        np.testing.assert_allclose(x, g["x"], rtol=1e-7, atol=1e-9 * np.abs(g["x"]).max())


@pytest.mark.parametrize("prefix", list(SOLVE_VARIANTS))
def test_solve_variants(oracle, prefix):
    ip, ix, a, g = problem_for("g2d_dir_64")
    h = oracle.setup(ip, ix, a)
    kw = dict(SOLVE_VARIANTS[prefix])
    tol = kw.pop("tol", 1e-8)
    max_iters = kw.pop("max_iters", 500)
    x0 = g[prefix + "x0"] if prefix + "x0" in g else None
    x, rep = oracle.npcg_solve(h, g["b"], tol=tol, max_iters=max_iters, x0=x0, **kw)
    assert_history_close(rep.residual_history, g, prefix=prefix, rtol=1e-10)


def test_spec_known_answers(oracle):
    """SPEC.md examples the reference satisfies."""
    # path-5, scores [5,1,2,3,4] -> centers {1,5}; A^2 of a path
    n = 5
    rows = [i for i in range(n) for j in (i - 1, i, i + 1) if 0 <= j < n]
    cols = [j for i in range(n) for j in (i - 1, i, i + 1) if 0 <= j < n]
    ip = np.zeros(n + 1, dtype=np.int64)
    ip[1:] = np.cumsum(np.bincount(rows, minlength=n))
    ix = np.array(cols, dtype=np.int64)
    p2, x2 = oracle.squared_pattern(n, ip, ix)
    s = np.array([5.0, 1, 2, 3, 4])
    ctr = oracle.select_centers(p2, x2, s, np.zeros(n, dtype=bool))
    assert np.flatnonzero(ctr).tolist() == [0, 4]
    own = oracle.claim_owners(p2, x2, s, np.zeros(n, dtype=bool), ctr)
    assert own.tolist() == [0, 0, 0, 4, 4]
    # path-4 Laplacian, aggregates {1,2},{3,4} -> [[1,-1],[-1,1]]
    ip4 = np.array([0, 2, 5, 8, 10])
    ix4 = np.array([0, 1, 0, 1, 2, 1, 2, 3, 2, 3])
    a4 = np.array([1.0, -1, -1, 2, -1, -1, 2, -1, -1, 1])
    gp, gi, gv = oracle.galerkin_coo(ip4, ix4, a4, np.array([0, 0, 1, 1]), 2)
    assert gp.tolist() == [0, 2, 4] and gi.tolist() == [0, 1, 0, 1] and gv.tolist() == [1, -1, -1, 1]
    # l1 smoother row (2,-1,-1) -> M_ii = 4
    assert oracle.l1_diag(np.array([0, 3]), np.array([0, 1, 2]), np.array([2.0, -1, -1]))[0] == 4.0
    # path-3 midpoint score with the formula d + ((i mod 12) + u)/12
    sc = oracle.quasi_random_scores(np.array([0, 2, 5, 7]), np.array([0, 1, 0, 1, 2, 1, 2]), 0, 0)
    u = oracle.hash_u01(0, 0, np.array([1]))[0]
    assert sc[1] == 2 + (1 + u) / 12.0


def test_thread_invariance(oracle):
    ip, ix, a, g = problem_for("g3d7_16")
    old = oracle.get_num_threads()
    try:
        oracle.set_num_threads(1)
        h1 = oracle.setup(ip, ix, a)
        oracle.set_num_threads(4)
        h4 = oracle.setup(ip, ix, a)
    finally:
        oracle.set_num_threads(old)
    for L1, L4 in zip(h1.levels, h4.levels):
        assert np.array_equal(L1.data, L4.data) and np.array_equal(L1.indices, L4.indices)
        if L1.vertex_to_agg is not None:
            assert np.array_equal(L1.vertex_to_agg, L4.vertex_to_agg)


def test_c2_full_size(oracle):
    """C2 (3D 7-pt 128^3) at full size: the oracle reproduces the reference's
    hierarchy hashes and its 47-iteration history."""
    ip, ix, a, g = problem_for("c2_grid3d7_128")
    h = oracle.setup(ip, ix, a)
    assert_hierarchy_equal(g, _oracle_levels(h))
    x, rep = oracle.npcg_solve(h, np.ones(ip.shape[0] - 1), tol=float(g["tol"]), max_iters=500)
    assert_history_close(rep.residual_history, g, rtol=1e-10)


@pytest.mark.parametrize("case", HIERARCHY_CASES)
def test_two_hop_selection_matches_pattern(oracle, case):
    """The oracle's A^2-free selection/claim (two maximum hops over A, used
    when A^2 would not fit in memory, e.g. C5's hub levels) gives the
    reference's hierarchy bit for bit, like the A^2-pattern loops."""
    ip, ix, a, g = problem_for(case)
    try:
        oracle.set_select_mode(2)
        h = oracle.setup(ip, ix, a, **CASE_CFG.get(case, {}))
    finally:
        oracle.set_select_mode(0)
    assert_hierarchy_equal(g, _oracle_levels(h))
