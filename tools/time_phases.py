"""Time setup and solve separately (CUDA events) for a config.  Usage: python tools/time_phases.py [n] [stencil]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402
from paper_1302_2547_b200.device import DeviceCSR  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
st = int(sys.argv[2]) if len(sys.argv) > 2 else 7
A = problems.grid3d(n, st)
Ad = DeviceCSR.from_host(A)
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")


def ev_time(fn, reps=3):
    ts = []
    out = None
    for _ in range(reps):
        out = None  # free the previous result first (as bench.py does between steps)
        import gc
        gc.collect()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1) * 1e-3, time.perf_counter() - t0))
    return out, ts


h, ts = ev_time(lambda: U.setup(Ad), reps=int(os.environ.get("SETUP_REPS", "3")))
print("setup (event s, wall s):", [(round(a, 4), round(b_, 4)) for a, b_ in ts], flush=True)
print("levels", [(l.n, l.matrix.nnz if hasattr(l.matrix, "nnz") else None) for l in h.levels], flush=True)
if True:
    res, ts = ev_time(lambda: U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8, max_iters=500), reps=3)
    x, rep = res
    print(f"iters={rep.iterations} solve(event s, wall s)=",
          [(round(a, 4), round(b_, 4)) for a, b_ in ts], "device solve_seconds", rep.timings.get("solve_seconds"),
          flush=True)
