"""A/B of the coarse tail kernel (tail.cu) against the separate-kernel path
on one problem: histories, iterations, solve time.  Usage:
python tools/ab_tail.py [n] [kind] [steps] [pre] [post]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
kind = sys.argv[2] if len(sys.argv) > 2 else "kcycle"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
pre = int(sys.argv[4]) if len(sys.argv) > 4 else 1
post = int(sys.argv[5]) if len(sys.argv) > 5 else 1
A = problems.grid3d_device(n, 7)
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
spec = U.CycleSpec(kind=kind, inner_krylov_steps=steps, pre_sweeps=pre, post_sweeps=post)
out = {}
for mode in ["tail", "notail"]:
    if mode == "notail":
        os.environ["UAAMG_NO_TAIL"] = "1"
    else:
        os.environ.pop("UAAMG_NO_TAIL", None)
    h = U.setup(A)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = U.npcg_solve(h, spec, U.Smoother(), b, tol=1e-8, max_iters=300)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out[mode] = np.array(rep.residual_history)
    print(mode, "levels", [l.n for l in h.levels], "iters", rep.iterations, "solve s", [round(t, 4) for t in ts],
          flush=True)
a, c = out["tail"], out["notail"]
m = min(len(a), len(c))
print("len", len(a), len(c), "max |rel diff| of histories", float(np.max(np.abs(a[:m] - c[:m]) / np.abs(c[:m]))))
