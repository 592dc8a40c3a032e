"""Subgraph reshaping of aggregate pairs (Alg. 3, PAPER §3.3) on the GPU.

Mirrors the reference's ``uaamg.reshaping.reshape_sweep``
(/root/reference/pkg/src/uaamg/reshaping.py:215-248) and its hook in setup
(hierarchy.py:141-144).  Per sweep the coarse edges are matched greedily in
(min id, max id) order and every matched pair of at most ``pair_cap``
vertices is solved as one small dense problem on the device
(csrc/reshape.cu): the local Laplacian, the smoother error matrix, the
pseudo-inverse and the rank-one trace |T|^2 of every balanced connected split,
keeping the maximum (earliest split on ties); aggregates are then renumbered
by their smallest member.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .aggregation import Aggregation
from .device import DeviceCSR, ptr, stream, to_device
from .solvers import Smoother

DEFAULT_PAIR_CAP = 16


class PairTooLarge(Exception):
    """Union subgraph exceeds the exhaustive-enumeration cap (pairs are skipped)."""


class DisconnectedPair(ValueError):
    """No balanced connected split of a pair exists."""


def _raise_reshape_error(msg):
    if "balanced connected split" in msg:
        raise DisconnectedPair(msg)
    raise ValueError(msg)


def reshape_sweep(a, agg, smoother=Smoother("l1"), sweeps=1, pair_cap=DEFAULT_PAIR_CAP):
    """Reshape a maximal matching of neighbouring aggregate pairs per sweep
    (reference reshaping.py:215-248); the aggregate count never changes."""
    if pair_cap > 16:
        raise NotImplementedError("pair_cap > 16: the device enumeration handles pairs of at most 16 vertices")
    d = a if isinstance(a, DeviceCSR) else a.device()
    n = d.n_rows
    if agg.n_fine != n:
        raise ValueError("aggregation does not match matrix dimensions")
    v2a = to_device(np.asarray(agg.vertex_to_agg), np.int32).clone()
    seeds = torch.empty(max(agg.n_coarse, 1), dtype=torch.int32, device=v2a.device)
    skipped = ctypes.c_int()
    rc = _lib.load().uaamg_reshape_sweep(n, d.nnz, ptr(d.row_ptr), ptr(d.col), ptr(d.val), int(agg.n_coarse),
                                         ptr(v2a), ptr(seeds), int(smoother.kind == "l1"), float(smoother.omega),
                                         int(sweeps), int(pair_cap), ctypes.byref(skipped), stream())
    if rc == _lib.UAAMG_EINVAL:
        _raise_reshape_error(_lib.last_error())
    _lib.check(rc)
    out = Aggregation(n, device_arrays=(v2a, seeds[: agg.n_coarse]))
    return out
