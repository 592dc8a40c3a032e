"""Median device setup time of a 3D grid (diagnostics; A/B of setup
switches via the environment).  Usage: python tools/setup_time.py [n] [stencil]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
st = int(sys.argv[2]) if len(sys.argv) > 2 else 7
A = problems.grid3d_device(n, st)
t = []
for k in range(12):
    h = U.setup(A)
    t.append(h.setup_seconds)
    del h
print(f"setup n={n} st={st} median {1e3 * float(np.median(t[2:])):.3f} ms  min {1e3 * min(t[2:]):.3f} ms")
