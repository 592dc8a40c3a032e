"""Quality metrics (paper_1302_2547_b200/analysis.py, U/analysis.py) against
values computed by the reference itself (tests/golden/analysis.npz, made by
tests/golden/make_analysis_golden.py)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "analysis.npz"))


@pytest.fixture(scope="module")
def U():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1302_2547_b200 as U

    return U


def test_hierarchy_report_dense_path(U):
    from paper_1302_2547_b200 import analysis, problems

    h = U.setup(problems.grid2d(24))
    reps = analysis.hierarchy_report(h)
    assert [r.fine_level for r in reps] == list(G["rep_fine"])
    assert [r.coarse_level for r in reps] == list(G["rep_coarse"])
    np.testing.assert_array_equal([r.coarsening_ratio for r in reps], G["rep_ratio"])
    np.testing.assert_allclose([r.q_energy_sq for r in reps], G["rep_q"], rtol=1e-10)
    e = np.array([np.nan if r.e_norm is None else r.e_norm for r in reps])
    np.testing.assert_allclose(e, G["rep_e"], rtol=1e-10)
    csv = analysis.reports_to_csv(reps, {"case": "g2d_24"})
    assert csv.splitlines()[0] == str(G["rep_csv"]).splitlines()[0]


def test_power_iteration_path_on_device(U):
    """4,900 unknowns > DENSE_CAP: device power iterations (inner K-cycle
    NPCG on the GPU) agree with the reference's host iterations to the
    power-iteration tolerance."""
    from paper_1302_2547_b200 import analysis, problems

    A = problems.grid2d(70)
    h = U.setup(A)
    agg = h.levels[0].aggregation
    q = analysis.q_energy_norm(A, agg)
    rate = analysis.two_level_rate(A, agg)
    assert abs(q - float(G["big_q"])) <= 1e-4 * abs(float(G["big_q"]))
    assert abs(rate - float(G["big_rate"])) <= 1e-4 * abs(float(G["big_rate"]))
