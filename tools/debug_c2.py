"""Diagnose CUDA errors on the C2 bench path: check cudaGetLastError after each step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from cuda.bindings import runtime as rt
import paper_1302_2547_b200 as U
from paper_1302_2547_b200 import problems
from paper_1302_2547_b200.device import DeviceCSR

def chk(tag):
    torch.cuda.synchronize()
    e = rt.cudaGetLastError()
    print(tag, e, flush=True)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
A = problems.grid3d(n, 7)
Ad = DeviceCSR.from_host(A); chk("upload")
h = U.setup(Ad); chk("setup")
print([l.n for l in h.levels])
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8); chk("solve")
print(rep.iterations, rep.residual_history[-1], rep.timings)
x, rep = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b, tol=1e-8); chk("solve2")
print(rep.iterations, rep.timings)
del h
import gc; gc.collect(); chk("free")
h = U.setup(Ad); chk("setup2")
print("setup2", h.setup_seconds)
