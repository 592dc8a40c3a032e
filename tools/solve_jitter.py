"""Distribution of C2 solve times (CUDA events + wall clock) over repeated
solves: (a) one hierarchy solved N times, (b) setup+solve with a fresh
hierarchy each time (the bench step).  Diagnostics for step-time outliers.
Usage: python tools/solve_jitter.py [N]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
A = problems.grid3d_device(128, 7)
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(s)
    out = fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3, time.perf_counter() - w0, out


h = U.setup(A)
for mode in ("solve-only", "setup+solve"):
    ts = []
    for k in range(N):
        if mode == "solve-only":
            ev, wl, _ = timed(lambda: U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8))
        else:
            def f():
                hh = U.setup(A)
                return U.npcg_solve(hh, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
            ev, wl, _ = timed(f)
        ts.append((round(ev * 1e3, 2), round(wl * 1e3, 2)))
    print(mode, "event/wall ms:", ts)
