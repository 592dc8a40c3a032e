"""Determinism bisection (diagnostics): repeat cycle() per level and short
NPCG solves on one C2 hierarchy and report which ones are not bit-repeatable.
Usage: python tools/det_bisect.py [n=128] [reps=4]"""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
A = problems.grid3d_device(n, 7)
h = U.setup(A)
print("levels", [L.n for L in h.levels], "env", {k: v for k, v in os.environ.items() if k.startswith("UAAMG")})


def hsh(t):
    return hashlib.sha1(t.cpu().numpy().tobytes()).hexdigest()[:10]


g = torch.Generator(device="cpu").manual_seed(1)
for lev in range(h.n_levels - 1):
    b = torch.rand(h.levels[lev].n, generator=g, dtype=torch.float64).cuda()
    hs = [hsh(U.cycle(h, U.CycleSpec(), U.Smoother(), lev, b)) for _ in range(reps)]
    print(f"cycle level {lev}: {'OK ' if len(set(hs)) == 1 else 'DRIFT'} {hs}")
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
for graphs in (True, False):
    for k in (1, 2, 3, 5, 10, 47):
        hs = []
        for _ in range(reps):
            x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8, max_iters=k, use_graphs=graphs)
            hs.append(hsh(x))
        print(f"npcg graphs={graphs} max_iters={k}: {'OK ' if len(set(hs)) == 1 else 'DRIFT'} {hs}")
