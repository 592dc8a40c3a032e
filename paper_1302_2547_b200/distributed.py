"""Multi-GPU row-partitioned solve: one process per GPU (torch.distributed).

SURVEY.md §8e.  Every rank runs ``setup`` on its own GPU (the hierarchy is
bit-identical on every rank, so it is replicated rather than communicated)
and then calls :func:`npcg_solve_distributed` collectively.  The C library
(``csrc/shard.cu``) shards the levels with at least ``shard_rows`` rows by
contiguous row ranges; halo columns are gathered directly from the owning
rank's CUDA-IPC-mapped buffers (NVLink peer loads fused into the SpMV), and
dot products are folded per rank and then across ranks in rank order.
torch.distributed (any backend; gloo suffices) only carries the one-time
exchange of the 64-byte IPC handles.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .device import ptr, stream, to_device, to_host
from .solvers import NumericalError, SolveReport, _params

HANDLE_BYTES = 64


def partition_rows(n, ranks):
    """Level-0 row ranges (``ranks + 1`` bounds): equal 128-aligned blocks."""
    out = np.zeros(ranks + 1, dtype=np.int32)
    _lib.check(_lib.load().uaamg_partition_rows(int(n), int(ranks), out.ctypes.data_as(ctypes.c_void_p)))
    return out


def partition_coarse(seeds, fine_bounds):
    """Coarse-level row ranges by seed ownership (aggregates ascend by seed)."""
    seeds = np.ascontiguousarray(seeds, dtype=np.int32)
    fine = np.ascontiguousarray(fine_bounds, dtype=np.int32)
    ranks = fine.shape[0] - 1
    out = np.zeros(ranks + 1, dtype=np.int32)
    _lib.check(_lib.load().uaamg_partition_coarse(seeds.ctypes.data_as(ctypes.c_void_p), int(seeds.shape[0]),
                                                  fine.ctypes.data_as(ctypes.c_void_p), ranks,
                                                  out.ctypes.data_as(ctypes.c_void_p)))
    return out


def exchange_handles(local, group=None):
    """All-gather each rank's ``HANDLE_BYTES`` handle; returns them concatenated in rank order."""
    import torch.distributed as dist

    if len(local) != HANDLE_BYTES:
        raise ValueError("IPC handles are 64 bytes")
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(local), group=group)
    return b"".join(out)


def npcg_solve_distributed(h, cycle_spec, smoother, b, tol=1e-6, max_iters=200, x0=None, shard_rows=262144,
                           group=None):
    """Collective ``npcg_solve`` over the ranks of ``group`` (one GPU each)."""
    import torch.distributed as dist

    rank, size = dist.get_rank(group), dist.get_world_size(group)
    if h._offset != 0:
        raise ValueError("npcg_solve needs the full hierarchy")
    n = h.levels[0].n
    host = not isinstance(b, torch.Tensor)
    bd = to_device(b, np.float64)
    if bd.shape != (n,):
        raise ValueError("right-hand side size mismatch")
    x0d = to_device(x0, np.float64) if x0 is not None else None
    P = _params(cycle_spec, smoother, tol, max_iters, False)
    L = _lib.load()
    d = ctypes.c_void_p()
    _lib.check(L.uaamg_dist_create(h._handle, ctypes.byref(P), rank, size, int(shard_rows), ctypes.byref(d)))
    try:
        hb = (ctypes.c_ubyte * HANDLE_BYTES)()
        _lib.check(L.uaamg_dist_handle(d, hb))
        allh = exchange_handles(bytes(hb), group)
        buf = ctypes.create_string_buffer(allh, len(allh))
        _lib.check(L.uaamg_dist_connect(d, buf))
        x = torch.empty(n, dtype=torch.float64, device=bd.device)
        hist = np.zeros(int(max_iters) + 1)
        res = _lib.SolveResult()
        rc = L.uaamg_dist_solve(d, ptr(bd), ptr(x0d), ptr(x), hist.ctypes.data_as(ctypes.c_void_p),
                                ctypes.byref(res), stream())
        report = SolveReport(int(res.iterations), hist[: int(res.iterations) + 1].tolist(), bool(res.converged),
                             {"solve_seconds": float(res.solve_seconds), "ranks": size})
        if rc == _lib.UAAMG_ENUMERICAL:
            raise NumericalError(_lib.last_error(), report=report)
        _lib.check(rc)
        torch.cuda.current_stream().synchronize()
        dist.barrier(group)  # no rank frees its arena while a peer may still read it
    finally:
        L.uaamg_dist_free(d)
    return (to_host(x) if host else x), report
