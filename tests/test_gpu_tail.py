"""The coarse tail kernel (csrc/tail.cu: the level above the coarsest, its
inner flexible CG / cycle and the coarsest solve in one thread-block cluster)
against the separate-kernel path and the reference histories.

Row sums in the tail follow the group kernel's order exactly; only the dot
products / norms use a different fixed tree, so histories agree with the
separate-kernel path to rounding (<= 1e-12 relative) and with the reference
within the parity tolerance (U/solvers.py:128-255)."""
import ctypes
import os

import numpy as np
import pytest

from golden_util import SOLVE_VARIANTS, assert_history_close, load, problem_for

pytestmark = pytest.mark.gpu

RTOL = 1e-10


@pytest.fixture(scope="module")
def U():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1302_2547_b200 as U
    return U


def tail_info(h):
    from paper_1302_2547_b200 import _lib
    lv, cs = ctypes.c_int(), ctypes.c_int()
    _lib.check(_lib.load().uaamg_tail_info(h._handle, ctypes.byref(lv), ctypes.byref(cs)))
    return lv.value, cs.value


def solve_both(U, A, b, spec, sm=None, **kw):
    """The same solve with the tail kernel and without it (fresh hierarchies)."""
    sm = sm or U.Smoother()
    out = {}
    for mode in ("tail", "plain"):
        if mode == "plain":
            os.environ["UAAMG_NO_TAIL"] = "1"
        try:
            h = U.setup(A)
            try:
                x, rep = U.npcg_solve(h, spec, sm, b, **kw)
            except U.NumericalError as e:
                # a stagnating configuration (no smoothing) may reach an exact
                # p'Ap = 0 breakdown on either path; compare what ran
                x, rep = np.zeros(len(b)), e.report
            out[mode] = (np.asarray(x), np.asarray(rep.residual_history), tail_info(h))
        finally:
            os.environ.pop("UAAMG_NO_TAIL", None)
    return out


def rel(a, b):
    m = min(len(a), len(b))
    return float(np.max(np.abs(a[:m] - b[:m]) / np.maximum(np.abs(b[:m]), 1e-300)))


@pytest.mark.parametrize("n", [24, 40])
def test_tail_matches_separate_kernels_3d(U, n):
    from paper_1302_2547_b200 import problems
    A = problems.grid3d(n, 7).device()
    b = np.ones(n ** 3)
    r = solve_both(U, A, b, U.CycleSpec(), tol=1e-8, max_iters=300)
    lv, cs = r["tail"][2]
    assert lv >= 1 and cs >= 1, "tail kernel not used"
    assert r["plain"][2][0] == -1
    assert len(r["tail"][1]) == len(r["plain"][1])
    assert rel(r["tail"][1], r["plain"][1]) < 1e-12
    np.testing.assert_allclose(r["tail"][0], r["plain"][0], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("prefix", ["", "vcycle_", "jacobi_", "jacobi_w05_", "inner0_", "inner3_", "x0_"])
def test_tail_variants_vs_reference(U, prefix):
    """Golden g2d_dir_64 (dense coarsest level) solve variants, tail on."""
    ip, ix, a, g = problem_for("g2d_dir_64")
    A = U.SparseMatrix(ip.shape[0] - 1, ip.shape[0] - 1, ip, ix, a)
    kw = dict(SOLVE_VARIANTS[prefix])
    spec = U.CycleSpec(**{k: v for k, v in kw.items() if k in ("kind", "inner_krylov_steps")})
    sm = U.Smoother(kind=kw.get("smoother", "l1"), **({"omega": kw["omega"]} if "omega" in kw else {}))
    x0 = g[prefix + "x0"] if prefix + "x0" in g else None
    h = U.setup(A)
    x, rep = U.npcg_solve(h, spec, sm, g["b"], tol=1e-8, max_iters=500, x0=x0)
    assert tail_info(h)[0] >= 1
    assert_history_close(rep.residual_history, g, prefix=prefix, rtol=RTOL)


@pytest.mark.parametrize("pre,post", [(0, 1), (1, 0), (0, 0)])
def test_tail_sweep_variants(U, pre, post):
    from paper_1302_2547_b200 import problems
    A = problems.grid3d(20, 7).device()
    b = np.ones(20 ** 3)
    spec = U.CycleSpec(pre_sweeps=pre, post_sweeps=post)
    n_it = 60 if (pre, post) != (0, 0) else 6
    r = solve_both(U, A, b, spec, tol=1e-8, max_iters=n_it)
    assert r["tail"][2][0] >= 1
    # (0, 0): no smoothing, the preconditioner's range is the coarse space and
    # NPCG stagnates (the reference too); only the first steps are compared
    assert rel(r["tail"][1], r["plain"][1]) < 1e-10


def test_tail_not_used_when_ineligible(U):
    from paper_1302_2547_b200 import problems
    A = problems.grid3d(16, 7).device()
    h = U.setup(A)
    U.npcg_solve(h, U.CycleSpec(pre_sweeps=2, post_sweeps=2), U.Smoother(), np.ones(16 ** 3), tol=1e-8)
    assert tail_info(h)[0] == -1


def test_tail_c2_history_matches_reference(U):
    """The bench configuration (C2, 128^3): the tail runs on level 4 (8512
    rows with two hub rows of 5318 / 3395 entries) on a 16-CTA cluster and
    the history still matches the reference's."""
    import torch
    from paper_1302_2547_b200 import problems
    g = load("c2_grid3d7_128")
    A = problems.grid3d_device(128, 7)
    h = U.setup(A)
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
    lv, cs = tail_info(h)
    assert lv == h.n_levels - 2 and cs == 16
    assert_history_close(rep.residual_history, g, rtol=RTOL)
