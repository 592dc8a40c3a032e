"""Multilevel hierarchy on the GPU.

Mirrors /root/reference/pkg/src/uaamg/hierarchy.py: ``galerkin_coarse``
(:22-28), ``CoarseSolver`` (:31-65), ``Level``/``Hierarchy`` (:68-109),
``detect_singular`` (:112-117), ``setup`` (:120-153).  ``setup`` runs
entirely on the device (``uaamg_setup``): per level the multi-pass
aggregation, members_csr, and the Galerkin operator A_c = P^T A P as an
exact-order segmented sum by aggregate pair; the coarsest level is factored
densely on the device.  The hierarchy stays device-resident; host mirrors of
level matrices/aggregations are materialised lazily on attribute access.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .aggregation import Aggregation, AggregationConfig
from .device import DeviceCSR, cuda_device, ptr, stream, to_device, to_host, view
from .sparse import SparseMatrix


class SetupError(RuntimeError):
    pass


def galerkin_coarse(a, agg):
    """(A_c)_IJ = sum over s in G_I, t in G_J of a_st; exact zeros dropped."""
    if agg.n_fine != a.n_rows or a.n_rows != a.n_cols:
        raise ValueError("aggregation does not match matrix dimensions")
    from . import kernel_table
    p, i, v = kernel_table.galerkin_coo(a.indptr, a.indices, a.data, agg.vertex_to_agg, agg.n_coarse)
    return SparseMatrix(agg.n_coarse, agg.n_coarse, p, i, v, _validate=False)


class _Native:
    """Owns the native hierarchy handle (and the device matrix level 0
    aliases).  Levels and device views hold this object rather than the
    Hierarchy, so there is no reference cycle and the device memory is
    released as soon as the last user goes away, not at a later cyclic GC
    pass (which would free many hierarchies at once, at an arbitrary point)."""

    __slots__ = ("handle", "matrix_owner", "__weakref__")

    def __init__(self, handle, matrix_owner=None):
        self.handle = handle
        self.matrix_owner = matrix_owner

    def level_view(self, l):
        v = _lib.LevelView()
        _lib.check(_lib.load().uaamg_hierarchy_level(self.handle, l, ctypes.byref(v)))
        return v

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                _lib.load().uaamg_hierarchy_free(self.handle)
            except Exception:
                pass
            self.handle = None


class Level:
    """One hierarchy level: ``matrix`` (host SparseMatrix, lazy) and
    ``aggregation`` (None on the coarsest level); ``device_matrix`` is the
    zero-copy device CSR."""

    __slots__ = ("_h", "_l", "_matrix", "_agg", "_dev")

    def __init__(self, native, l):
        self._h, self._l = native, l  # the native owner (no back-reference to the Hierarchy)
        self._matrix = self._agg = self._dev = None

    def _view(self):
        return self._h.level_view(self._l)

    @property
    def device_matrix(self):
        if self._dev is None:
            v = self._view()
            self._dev = DeviceCSR(v.n, v.n, view(v.row_ptr, v.n + 1, np.int32, self._h),
                                  view(v.col, v.nnz, np.int32, self._h), view(v.val, v.nnz, np.float64, self._h),
                                  lib_owned=True)
        return self._dev

    @property
    def matrix(self):
        if self._matrix is None:
            self._matrix = self.device_matrix.to_host()
        return self._matrix

    @property
    def aggregation(self):
        if self._agg is None:
            v = self._view()
            if v.n_coarse == 0:
                return None
            self._agg = Aggregation(v.n, device_arrays=(view(v.vertex_to_agg, v.n, np.int32, self._h),
                                                        view(v.coarse_vertex_of_agg, v.n_coarse, np.int32, self._h)))
        return self._agg

    @property
    def n(self):
        return self._view().n

    @property
    def nnz(self):
        return int(self._view().nnz)


class CoarseSolver:
    """Dense factorization of the coarsest operator (reference
    hierarchy.py:31-65), held on the device: ``CoarseSolver(a, singular)``
    densifies ``a`` (SparseMatrix or DeviceCSR) and stores its Cholesky-based
    inverse, or -- singular, or Cholesky failed, which then sets
    ``singular = True`` like the reference -- the eigen pseudo-inverse with
    the reference's 1e-12 * lambda_max cut (uaamg_coarse_factor).
    ``solve(b)`` takes one vector or an (n, k) matrix of right-hand-side
    columns (numpy in -> numpy out, CUDA tensor in -> tensor out)."""

    def __init__(self, a, singular):
        self.n = a.n_rows
        self.singular = bool(singular)
        self._owner = None
        if self.n == 0:
            self._minv = None
            return
        d = a if isinstance(a, DeviceCSR) else a.device()
        self._minv = torch.empty(self.n * self.n, dtype=torch.float64, device=cuda_device())
        mode = ctypes.c_int()
        _lib.check(_lib.load().uaamg_coarse_factor(self.n, d.nnz, ptr(d.row_ptr), ptr(d.col), ptr(d.val),
                                                   int(self.singular), ptr(self._minv), ctypes.byref(mode), stream()))
        self.singular = self.singular or mode.value == 2

    @classmethod
    def _of_hierarchy(cls, native):
        """The factor setup() built for the coarsest level.  Holds the
        native owner (not the Hierarchy), so it stays usable on its own."""
        self = cls.__new__(cls)
        minv, n, mode = ctypes.c_void_p(), ctypes.c_int(), ctypes.c_int()
        _lib.check(_lib.load().uaamg_hierarchy_coarse(native.handle, ctypes.byref(minv), ctypes.byref(n),
                                                      ctypes.byref(mode)))
        self.n = n.value
        self.singular = mode.value == 2
        self._owner = native
        self._minv = view(minv.value, self.n * self.n, np.float64, native) if self.n else None
        return self

    def solve(self, b):
        """Solve against one vector or a matrix of right-hand-side columns."""
        host = not isinstance(b, torch.Tensor)
        if self.n == 0:
            return np.zeros_like(b) if host else torch.zeros_like(b)
        bd = to_device(b, np.float64)
        if bd.shape[0] != self.n or bd.dim() not in (1, 2):
            raise ValueError("coarse right-hand side size mismatch")
        nrhs = 1 if bd.dim() == 1 else bd.shape[1]
        x = torch.empty_like(bd)
        _lib.check(_lib.load().uaamg_dense_apply(self.n, ptr(self._minv), ptr(bd), int(nrhs), ptr(x), stream()))
        return to_host(x) if host else x


class Hierarchy:
    """Device-resident multilevel hierarchy (reference hierarchy.py:74-109)."""

    def __init__(self, handle, offset=0, parent=None, matrix_owner=None):
        self._handle = handle
        self._native = parent._native if parent is not None else _Native(handle, matrix_owner)
        self._offset = offset
        self._parent = parent
        L = _lib.load()
        info = _lib.HierarchyInfo()
        _lib.check(L.uaamg_hierarchy_get_info(handle, ctypes.byref(info)))
        self._info = info
        self.singular = bool(info.singular)
        nl = info.n_levels - offset
        self.levels = [Level(self._native, offset + l) for l in range(nl)]
        n0 = self.levels[0].n
        nnz0 = max(self.levels[0].nnz, 1)
        self.grid_complexity = sum(l.n for l in self.levels) / n0
        self.operator_complexity = sum(l.nnz for l in self.levels) / nnz0
        self.setup_seconds = float(info.setup_seconds)
        self.coarsest_solver = CoarseSolver._of_hierarchy(self._native)

    def _level_view(self, l):
        return self._native.level_view(l)

    @property
    def n_levels(self):
        return len(self.levels)

    def matrix(self, level):
        return self.levels[level].matrix

    def sub(self, level):
        """View of the hierarchy starting at ``level``."""
        if level == 0:
            return self
        return Hierarchy(self._handle, self._offset + level, parent=self)

    def summary(self):
        rows = []
        for l, lev in enumerate(self.levels):
            row = {"level": l, "n": lev.n, "nnz": lev.nnz}
            agg = lev.aggregation
            if agg is not None:
                row["coarsening_ratio"] = agg.coarsening_ratio
            rows.append(row)
        return {"levels": rows, "grid_complexity": self.grid_complexity,
                "operator_complexity": self.operator_complexity, "singular": self.singular}

    def __repr__(self):
        return f"Hierarchy(levels={[l.n for l in self.levels]})"


def detect_singular(a):
    """A annihilates the constant vector (reference hierarchy.py:112-117)."""
    if a.nnz == 0:
        return True
    scale = np.max(np.abs(a.data))
    return np.max(np.abs(a.spmv(np.ones(a.n_rows)))) <= 1e-10 * scale


def _check_setup(rc, reshape_sweeps):
    if rc == _lib.UAAMG_EINVAL and reshape_sweeps > 0:
        from .reshaping import _raise_reshape_error
        _raise_reshape_error(_lib.last_error())
    _lib.check(rc)


def setup(a, config=AggregationConfig(), n0=100, max_levels=20, reshape_sweeps=0, singular=None,
          reshape_pair_cap=16):
    """Build the hierarchy on the GPU (reference hierarchy.py:120-153).

    ``a``: host SparseMatrix (uploaded by the library, the values
    overlapping the level-0 aggregation; a SparseMatrix whose cached device
    copy exists uses that) or DeviceCSR (used in place)."""
    if a.n_rows != a.n_cols:
        raise SetupError("matrix must be square")
    if reshape_sweeps > 0 and reshape_pair_cap > 16:
        raise NotImplementedError("reshape_pair_cap > 16: the device enumeration handles pairs of at most 16 vertices")
    P = _lib.SetupParams(size_cap=0 if config.size_cap is None else int(config.size_cap), seed=int(config.seed),
                         max_passes=int(config.max_passes), passes_per_level=int(config.passes_per_level),
                         n0=int(n0), max_levels=int(max_levels),
                         singular=-1 if singular is None else int(bool(singular)),
                         reshape_sweeps=int(reshape_sweeps), reshape_pair_cap=int(reshape_pair_cap), borrow=0)
    if not isinstance(a, DeviceCSR) and a._device is None:
        # the reference's host matrix, not yet on the device: the library
        # uploads it itself, the values overlapping the level-0 aggregation
        ip = np.ascontiguousarray(a.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(a.indices, dtype=np.int64)
        dv = np.ascontiguousarray(a.data, dtype=np.float64)
        h = ctypes.c_void_p()
        rc = _lib.load().uaamg_setup_host(a.n_rows, int(ix.shape[0]), ip.ctypes.data, ix.ctypes.data if ix.size else None,
                                          dv.ctypes.data if dv.size else None, ctypes.byref(P), ctypes.byref(h),
                                          stream())
        _check_setup(rc, reshape_sweeps)
        return Hierarchy(h)
    d = a if isinstance(a, DeviceCSR) else a.device()
    # level 0 aliases the caller's device arrays when the TMA tile kernel may
    # read them in place (int32/int32/float64, contiguous, 16-byte aligned,
    # 64 readable bytes past the end); otherwise the library copies them
    borrow = d.borrowable()
    if not borrow and (d.row_ptr.dtype != torch.int32 or d.col.dtype != torch.int32 or d.val.dtype != torch.float64
                       or d.row_ptr.device != cuda_device()):
        d = DeviceCSR.from_arrays(d.n_rows, d.row_ptr, d.col, d.val)
        borrow = True
    P.borrow = int(borrow)
    h = ctypes.c_void_p()
    rc = _lib.load().uaamg_setup(d.n_rows, d.nnz, ptr(d.row_ptr), ptr(d.col), ptr(d.val), ctypes.byref(P),
                                 ctypes.byref(h), stream())
    _check_setup(rc, reshape_sweeps)
    # level 0 aliases the device matrix (as the reference's Level 0 holds A)
    return Hierarchy(h, matrix_owner=d)
