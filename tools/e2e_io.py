"""Host <-> device transfer timing of the reference-layout C2 arrays
(diagnostics): pageable torch copies vs the library's staged pipeline."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1302_2547_b200 import problems  # noqa: E402
from paper_1302_2547_b200.device import to_device, to_device_padded, to_host  # noqa: E402

A = problems.grid3d(128, 7)
torch.cuda.init()
for name, f in [("torch pageable int64->dev int32", lambda: torch.from_numpy(A.indices.copy()).cuda().to(torch.int32)),
                ("staged indices int64->int32", lambda: to_device_padded(A.indices, np.int32)),
                ("staged data f64", lambda: to_device_padded(A.data, np.float64)),
                ("staged indptr", lambda: to_device_padded(A.indptr, np.int32))]:
    for k in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    print(f"{name:36s} {t * 1e3:8.2f} ms")
x = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
for k in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    to_host(x)
    t = time.perf_counter() - t0
print(f"{'staged d2h x':36s} {t * 1e3:8.2f} ms")
for k in range(4):
    t0 = time.perf_counter()
    x.cpu().numpy()
    t = time.perf_counter() - t0
print(f"{'torch d2h x':36s} {t * 1e3:8.2f} ms")
