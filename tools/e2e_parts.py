import os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1302_2547_b200 as U
from paper_1302_2547_b200 import problems
A = problems.grid3d(128, 7); n = A.n_rows
b_np = np.ones(n)
res = {k: [] for k in ("wrap", "setup", "solve", "free", "total")}
for it in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A2 = U.SparseMatrix(n, n, A.indptr, A.indices, A.data, _validate=False)
    t1 = time.perf_counter()
    h2 = U.setup(A2)
    t2 = time.perf_counter()
    x, rep = U.npcg_solve(h2, U.CycleSpec(), U.Smoother(), b_np, tol=1e-8, max_iters=500)
    t3 = time.perf_counter()
    del h2, rep, x
    t4 = time.perf_counter()
    if it >= 2:
        for k, v in zip(("wrap", "setup", "solve", "free", "total"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
            res[k].append(v * 1e3)
for k, v in res.items():
    print(f"{k:6s} {np.median(v):8.3f} ms")
