"""Where the C2 end-to-end step's extra time goes (diagnostics): setup from
the host SparseMatrix vs from a resident device CSR, and the solve with a
numpy b / numpy x vs device vectors."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

A = problems.grid3d(128, 7)
n = A.n_rows
d = U.SparseMatrix(n, n, A.indptr, A.indices, A.data).device()
b_np = np.ones(n)
b_d = torch.ones(n, dtype=torch.float64, device="cuda")


def t(f, k=6):
    out = []
    for _ in range(k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
        del r
    return 1e3 * float(np.median(out[1:]))


print(f"setup(device CSR)          {t(lambda: U.setup(d)):8.2f} ms")
print(f"setup(host SparseMatrix)   {t(lambda: U.setup(U.SparseMatrix(n, n, A.indptr, A.indices, A.data, _validate=False))):8.2f} ms")
h = U.setup(d)
print(f"solve(device b)            {t(lambda: U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b_d, tol=1e-8)):8.2f} ms")
print(f"solve(numpy b)             {t(lambda: U.npcg_solve(h, U.CycleSpec(), U.Smoother(), b_np, tol=1e-8)):8.2f} ms")


def e2e():
    h2 = U.setup(U.SparseMatrix(n, n, A.indptr, A.indices, A.data, _validate=False))
    return U.npcg_solve(h2, U.CycleSpec(), U.Smoother(), b_np, tol=1e-8)


print(f"e2e                        {t(e2e):8.2f} ms")
os.environ["UAAMG_SETUP_PROF"] = "1"
U.setup(U.SparseMatrix(n, n, A.indptr, A.indices, A.data, _validate=False))
