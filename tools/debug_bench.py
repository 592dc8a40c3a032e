"""Replicate bench.py's step sequence with cudaGetLastError checks."""
import ctypes, gc, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from cuda.bindings import runtime as rt
import paper_1302_2547_b200 as U
from paper_1302_2547_b200 import _lib, problems
from paper_1302_2547_b200.device import DeviceCSR
from paper_1302_2547_b200.solvers import _params

def chk(tag):
    torch.cuda.synchronize()
    print(tag, rt.cudaGetLastError()[0], flush=True)

dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
A = problems.grid3d(int(sys.argv[1]) if len(sys.argv) > 1 else 128, 7)
n = A.n_rows
Ad = DeviceCSR.from_host(A); b = torch.ones(n, dtype=torch.float64, device=dev)
stream = torch.cuda.current_stream()
chk("init")

def solve(h, profile, max_iters=500):
    P = _params(U.CycleSpec(), U.Smoother(), 1e-8, max_iters, True)
    P.profile_level0 = int(profile)
    res = _lib.SolveResult()
    x = torch.empty(n, dtype=torch.float64, device=dev)
    hist = np.zeros(max_iters + 1)
    rc = _lib.load().uaamg_npcg_solve(h._handle, ctypes.byref(P), b.data_ptr(), None, x.data_ptr(),
                                      hist.ctypes.data_as(ctypes.c_void_p), ctypes.byref(res), stream.cuda_stream)
    print("  rc", rc, _lib.last_error() if rc else "", res.iterations, flush=True)

for k in range(4):
    h = U.setup(Ad); chk(f"setup{k}")
    for mi in (200, 500):
        solve(h, False, mi); chk(f"solve{k} mi={mi}")
    solve(h, True); chk(f"solve{k} prof")
    del h; gc.collect(); chk(f"free{k}")
