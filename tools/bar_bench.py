"""Grid-barrier microbenchmark (engine grid): seconds per barrier."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401  (initialises the CUDA context)
from paper_1302_2547_b200 import _lib
L = _lib.load()
torch.zeros(1, device="cuda")
for v in (0, 1):
    for it in (1000, 10000):
        s = ctypes.c_double()
        rc = L.uaamg_dev_barrier_bench(v, it, ctypes.byref(s))
        print(f"variant {v} iters {it}: rc={rc} {s.value * 1e6:.3f} us/barrier", flush=True)
