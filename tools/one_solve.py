"""One C2 setup + solve (for ncu launch lists / captures)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

n = int(os.environ.get("ONE_SOLVE_N", "128"))
st = int(os.environ.get("ONE_SOLVE_STENCIL", "7"))
d = problems.grid3d_device(n, st)
h = U.setup(d)
b = torch.ones(d.n_rows, dtype=torch.float64, device="cuda")
x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
torch.cuda.synchronize()
print("levels", [l.n for l in h.levels], "iterations", rep.iterations, "final", rep.residual_history[-1])
