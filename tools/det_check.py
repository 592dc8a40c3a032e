"""Determinism check (diagnostics): hashes of x and the residual history of
C2 solves -- fresh hierarchies (mode 'fresh') or one hierarchy solved
repeatedly (mode 'same').  Usage: python tools/det_check.py [fresh|same]"""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fresh"
A = problems.grid3d_device(128, 7)
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
h = U.setup(A)
hists = []
for k in range(3):
    if mode == "fresh":
        h = U.setup(A)
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
    xh = x.cpu().numpy()
    hists.append(np.array(rep.residual_history))
    print(mode, k, rep.iterations, hashlib.sha1(xh.tobytes()).hexdigest()[:12],
          hashlib.sha1(np.array(rep.residual_history).tobytes()).hexdigest()[:12])
m = min(len(hh) for hh in hists)
d = max(float(np.max(np.abs(hh[:m] - hists[0][:m]) / np.abs(hists[0][:m]))) for hh in hists)
print("max relative history difference between repeats: %.3e" % d)
