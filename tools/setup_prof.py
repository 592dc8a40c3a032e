"""Setup phase profile (diagnostics): warm setups, then one with
UAAMG_SETUP_PROF / UAAMG_AGG_PROF output.  Usage: python tools/setup_prof.py [n] [stencil]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
st = int(sys.argv[2]) if len(sys.argv) > 2 else 7
A = problems.grid3d_device(n, st)
for _ in range(3):
    h = U.setup(A)
    del h
torch.cuda.synchronize()
print("=== profiled setup", n, st, flush=True)
h = U.setup(A)
print("levels", [l.n for l in h.levels], "setup_s", h.setup_seconds, flush=True)
