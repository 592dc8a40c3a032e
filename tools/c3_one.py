"""One C3 setup + solve (the largest component of the 2^23-point random
geometric graph) for ncu captures (diagnostics)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

A = problems.random_geometric(1 << 23, 12.0, 0, largest_component=True).device()
h = U.setup(A)
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
torch.cuda.synchronize()
print("levels", [l.n for l in h.levels], "iterations", rep.iterations)
