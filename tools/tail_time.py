"""Average duration of the tail kernel (CUPTI timeline of one warm C2 solve)
and the solve time.  Usage: python tools/tail_time.py [n]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
A = problems.grid3d_device(n, 7)
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
h = U.setup(A)
for _ in range(2):
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/tt.json")
ev = json.load(open("/tmp/tt.json"))
ev = ev["traceEvents"] if isinstance(ev, dict) else ev
k = sorted([e for e in ev if e.get("cat") == "kernel"], key=lambda e: e["ts"])
tail = [e for e in k if "k_tail" in e["name"]]
# own time: end minus max(start, previous kernel end)
own = []
for i, e in enumerate(k):
    if "k_tail" in e["name"] and i > 0:
        pe = max(p["ts"] + p["dur"] for p in k[max(0, i - 3):i])
        own.append(e["ts"] + e["dur"] - max(e["ts"], pe))
import statistics  # noqa: E402
print(f"iters {rep.iterations} tail launches {len(tail)} own us median {statistics.median(own):.2f} "
      f"dur median {statistics.median([e['dur'] for e in tail]):.2f}; span {(k[-1]['ts'] + k[-1]['dur'] - k[0]['ts']) / 1e3:.2f} ms")
