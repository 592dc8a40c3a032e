"""Golden values for the quality metrics (paper_1302_2547_b200/analysis.py),
made by running the REFERENCE's uaamg.analysis in this container:

    python tests/golden/make_analysis_golden.py

(1) hierarchy_report of a 2D 24x24 Dirichlet grid (dense path, every level
pair, with two-level rates); (2) q_energy_norm and two_level_rate of the
level-0 aggregation of a 2D 70x70 grid (4,900 unknowns > DENSE_CAP: power
iterations, the reference's own multigrid as inner solver)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import load_reference, save  # noqa: E402


def main():
    U, _ = load_reference()
    from uaamg import analysis
    from uaamg.graph import assemble_laplacian, generate_structured_grid

    out = {}
    A = assemble_laplacian(generate_structured_grid(24, "dirichlet"))
    h = U.setup(A)
    reps = analysis.hierarchy_report(h)
    out["rep_fine"] = np.array([r.fine_level for r in reps])
    out["rep_coarse"] = np.array([r.coarse_level for r in reps])
    out["rep_ratio"] = np.array([r.coarsening_ratio for r in reps])
    out["rep_q"] = np.array([r.q_energy_sq for r in reps])
    out["rep_e"] = np.array([np.nan if r.e_norm is None else r.e_norm for r in reps])
    out["rep_csv"] = np.array(analysis.reports_to_csv(reps, {"case": "g2d_24"}))
    B = assemble_laplacian(generate_structured_grid(70, "dirichlet"))
    hb = U.setup(B)
    agg = hb.levels[0].aggregation
    t = time.time()
    out["big_q"] = np.array(analysis.q_energy_norm(B, agg))
    out["big_rate"] = np.array(analysis.two_level_rate(B, agg))
    print("large path", time.time() - t, float(out["big_q"]), float(out["big_rate"]))
    save("analysis", **out)


if __name__ == "__main__":
    main()
