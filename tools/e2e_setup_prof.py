"""Setup phase profile of the host-layout path (diagnostics; run with
UAAMG_SETUP_PROF=1): three warm setups from a fresh host SparseMatrix."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_2547_b200 as U  # noqa: E402
from paper_1302_2547_b200 import problems  # noqa: E402

A = problems.grid3d(128, 7)
n = A.n_rows
for k in range(3):
    print("=== setup", k, file=sys.stderr, flush=True)
    h = U.setup(U.SparseMatrix(n, n, A.indptr, A.indices, A.data, _validate=False))
    torch.cuda.synchronize()
    del h
