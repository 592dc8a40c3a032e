"""Kernel timeline of one warm C2 solve (CUPTI via torch.profiler): per-kernel
start/end inside the graph replays, so PDL overlap and inter-kernel gaps are
visible.  Usage: python tools/timeline.py [n] [out.json]"""
import json
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline.json"
A = problems.grid3d_device(n, 7)
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
h = U.setup(A)
for _ in range(2):
    U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8)
    torch.cuda.synchronize()
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
trace = out.replace(".json", "_chrome.json")
prof.export_chrome_trace(trace)
ev = json.load(open(trace))
ev = ev["traceEvents"] if isinstance(ev, dict) else ev
k = [e for e in ev if e.get("cat") == "kernel"]
k.sort(key=lambda e: e["ts"])
rows = [{"name": e["name"][:90], "ts": e["ts"], "dur": e["dur"], "grid": e.get("args", {}).get("grid"),
         "block": e.get("args", {}).get("block")} for e in k]
json.dump(rows, open(out, "w"))
t0, t1 = rows[0]["ts"], rows[-1]["ts"] + rows[-1]["dur"]
print("levels", [l.n for l in h.levels], "iters", rep.iterations, "kernels", len(rows), "span us", round(t1 - t0, 1))
# aggregate by (name, grid): count, sum dur, sum of (start - previous end) gaps
agg = defaultdict(lambda: [0, 0.0, 0.0])
prev_end = rows[0]["ts"]
for r in rows:
    key = (r["name"][:70], str(r["grid"]))
    a = agg[key]
    a[0] += 1
    a[1] += r["dur"]
    a[2] += r["ts"] - prev_end
    prev_end = max(prev_end, r["ts"] + r["dur"])
tot = sum(a[1] for a in agg.values())
gaps = sum(a[2] for a in agg.values())
print(f"sum dur {tot:.1f} us, sum gaps {gaps:.1f} us")
for key, a in sorted(agg.items(), key=lambda kv: -(kv[1][1] + kv[1][2]))[:45]:
    print(f"{a[0]:5d} x {a[1] / a[0]:7.2f} us dur {a[1]:8.1f} gap {a[2]:8.1f}  {key[1]:>14s} {key[0]}")
# one middle iteration in order
mid = [i for i, r in enumerate(rows) if "NpcgUpd" in r["name"]]
if len(mid) > 3:
    lo, hi = mid[len(mid) // 2 - 1] + 1, mid[len(mid) // 2] + 1
    print(f"--- one iteration: {hi - lo} kernels, {rows[hi - 1]['ts'] + rows[hi - 1]['dur'] - rows[lo]['ts']:.1f} us")
    pe = rows[lo - 1]["ts"] + rows[lo - 1]["dur"]
    for r in rows[lo:hi]:
        print(f"  +{r['ts'] - pe:7.2f} {r['dur']:7.2f}  {str(r['grid']):>14s} {r['name'][:80]}")
        pe = max(pe, r["ts"] + r["dur"])
