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


class GraphProblem:
    """U/graph.py:20-60: n vertices, undirected weighted edges (i, j, w),
    boundary weights (j, wD).  Same validation and normalisation (i < j) as
    the reference, vectorised; ``edges`` / ``boundary`` are the normalised
    lists, the arrays are kept for the device assembly."""

    def __init__(self, n, edges, boundary=()):
        self.n = int(n)
        ei, ej, w = (np.asarray(x) for x in _edges(edges))
        ei, ej, w = ei.astype(np.int64), ej.astype(np.int64), w.astype(np.float64)
        if ei.size:
            if np.any(ei == ej):
                raise GraphError(f"self-loop at vertex {int(ei[np.argmax(ei == ej)])}")
            if np.any((ei < 0) | (ei >= self.n) | (ej < 0) | (ej >= self.n)):
                raise GraphError(f"edge out of range for n={self.n}")
            if np.any(w <= 0):
                raise GraphError("non-positive edge weight")
            lo, hi = np.minimum(ei, ej), np.maximum(ei, ej)
            key = lo * self.n + hi
            if np.unique(key).size != key.size:
                raise GraphError("duplicate edge")
            ei, ej = lo, hi
        if isinstance(boundary, tuple) and len(boundary) == 2 and not np.isscalar(boundary[0]):
            bj, bw = (np.asarray(x) for x in boundary)
        else:
            b = np.asarray(boundary, dtype=np.float64).reshape(-1, 2) if len(boundary) else np.zeros((0, 2))
            bj, bw = b[:, 0], b[:, 1]
        bj, bw = bj.astype(np.int64), bw.astype(np.float64)
        if bj.size:
            if np.any((bj < 0) | (bj >= self.n)):
                raise GraphError("boundary vertex out of range")
            if np.any(bw <= 0):
                raise GraphError("non-positive boundary weight")
            if np.unique(bj).size != bj.size:
                raise GraphError("duplicate boundary weight")
        self.ei, self.ej, self.w, self.bj, self.bw = ei, ej, w, bj, bw

    @property
    def edges(self):
        return [(int(a), int(b), float(c)) for a, b, c in zip(self.ei, self.ej, self.w)]

    @property
    def boundary(self):
        return [(int(a), float(b)) for a, b in zip(self.bj, self.bw)]

    @property
    def singular(self):
        return self.bj.size == 0


def assemble_laplacian(problem):
    """U/graph.py:63-82 on the device; returns the host SparseMatrix like the
    reference (use assemble_laplacian_device to keep it in HBM)."""
    return assemble_laplacian_device(problem.n, (problem.ei, problem.ej, problem.w),
                                     (problem.bj, problem.bw)).to_host()


def generate_structured_grid(n, bc="dirichlet", anisotropy=(1.0, 1.0)):
    """U/graph.py:85-123: n-by-n lattice, edges in the reference's order
    (per vertex: right, then down), Dirichlet boundary weights = sum of the
    missing off-grid edge weights (accumulated in the reference's order)."""
    if n < 2:
        raise GraphError(f"grid size must be >= 2, got {n}")
    if bc not in ("dirichlet", "neumann"):
        raise GraphError(f"unknown boundary condition {bc!r}")
    w_h, w_v = float(anisotropy[0]), float(anisotropy[1])
    if w_h <= 0 or w_v <= 0:
        raise GraphError("anisotropy weights must be positive")
    v = np.arange(n * n, dtype=np.int64)
    r, c = v // n, v % n
    ei = np.stack([v, v], axis=1).reshape(-1)
    ej = np.stack([v + 1, v + n], axis=1).reshape(-1)
    w = np.tile([w_h, w_v], n * n)
    ok = np.stack([c + 1 < n, r + 1 < n], axis=1).reshape(-1)
    ei, ej, w = ei[ok], ej[ok], w[ok]
    if bc == "dirichlet":
        miss = np.zeros(n * n)
        miss = np.where(r == 0, miss + w_v, miss)
        miss = np.where(r == n - 1, miss + w_v, miss)
        miss = np.where(c == 0, miss + w_h, miss)
        miss = np.where(c == n - 1, miss + w_h, miss)
        sel = miss > 0
        return GraphProblem(n * n, (ei, ej, w), (v[sel], miss[sel]))
    return GraphProblem(n * n, (ei, ej, w))


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
