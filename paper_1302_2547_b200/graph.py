"""Graph Laplacian assembly on the device.

Mirror of the reference's ``GraphProblem`` validation and
``assemble_laplacian`` (U/graph.py:20-82) for edge arrays of any size: the
validation is vectorised (torch, on the device) and the assembly runs in
``csrc/assemble.cu`` -- the same triplet list, diagonal weights accumulated
in edge-list order, and the reference's canonical ``from_coo`` -- so the CSR
is bit-identical to ``assemble_laplacian(GraphProblem(n, edges, boundary))``.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .device import DeviceCSR, ptr, stream, to_device


class GraphError(ValueError):
    pass


def _edges(edges):
    # list of (i, j, w) triples, or a tuple of three arrays (i, j, w)
    if isinstance(edges, tuple):
        return edges
    a = np.asarray(edges, dtype=np.float64).reshape(-1, 3) if len(edges) else np.zeros((0, 3))
    return a[:, 0].astype(np.int64), a[:, 1].astype(np.int64), a[:, 2]


def assemble_laplacian_device(n, edges, boundary=()):
    """DeviceCSR of the graph Laplacian.  ``edges``: list of (i, j, w)
    triples or a TUPLE of three arrays (i, j, w); ``boundary``: list of
    (j, w) pairs or a tuple of two arrays (j, w).
    Raises GraphError on the reference's validation failures."""
    n = int(n)
    ei, ej, w = _edges(edges)
    ei = to_device(ei, np.int64)
    ej = to_device(ej, np.int64)
    w = to_device(w, np.float64)
    if isinstance(boundary, tuple) and len(boundary) == 2 and not np.isscalar(boundary[0]):
        bj, bw = boundary  # arrays (j, w)
    else:
        b = np.asarray(boundary, dtype=np.float64).reshape(-1, 2) if len(boundary) else np.zeros((0, 2))
        bj, bw = b[:, 0].astype(np.int64), b[:, 1]
    bj = to_device(bj, np.int64)
    bw = to_device(bw, np.float64)
    # GraphProblem.__post_init__ (U/graph.py:26-56), vectorised
    if ei.numel():
        if bool((ei == ej).any()):
            raise GraphError("self-loop")
        if bool(((ei < 0) | (ei >= n) | (ej < 0) | (ej >= n)).any()):
            raise GraphError("edge out of range")
        if bool((w <= 0).any()):
            raise GraphError("non-positive edge weight")
        lo, hi = torch.minimum(ei, ej), torch.maximum(ei, ej)
        key = torch.sort(lo * n + hi).values
        if key.numel() > 1 and bool((key[1:] == key[:-1]).any()):
            raise GraphError("duplicate edge")
        ei, ej = lo.contiguous(), hi.contiguous()
    if bj.numel():
        if bool(((bj < 0) | (bj >= n)).any()):
            raise GraphError("boundary vertex out of range")
        if bool((bw <= 0).any()):
            raise GraphError("non-positive boundary weight")
        sb = torch.sort(bj).values
        if sb.numel() > 1 and bool((sb[1:] == sb[:-1]).any()):
            raise GraphError("duplicate boundary weight")
    h = ctypes.c_void_p()
    _lib.check(_lib.load().uaamg_assemble_laplacian(n, int(ei.numel()), ptr(ei), ptr(ej), ptr(w), int(bj.numel()),
                                                    ptr(bj), ptr(bw), ctypes.byref(h), stream()))
    return DeviceCSR._from_lib(h)
