"""Device-side plumbing: torch owns user-visible device memory and streams;
the CUDA work happens in libuaamg_b200.so.

``DeviceCSR`` is the device twin of :class:`~.sparse.SparseMatrix` (int32
row_ptr/col, fp64 val -- SURVEY.md section 8 layout).  Library-owned arrays
(the hierarchy) are exposed to torch zero-copy through
``__cuda_array_interface__`` views that keep their owner alive.
"""

import warnings

import numpy as np
import torch

from . import _lib

_TYPESTR = {np.dtype(np.int32): "<i4", np.dtype(np.float64): "<f8", np.dtype(np.uint8): "|u1",
            np.dtype(np.int64): "<i8"}
_TORCH = {np.dtype(np.int32): torch.int32, np.dtype(np.float64): torch.float64, np.dtype(np.uint8): torch.uint8,
          np.dtype(np.int64): torch.int64}
_NP = {v: k for k, v in _TORCH.items()}


def cuda_device():
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 UA-AMG path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    """Current torch CUDA stream handle (passed to every library call)."""
    return ctypes_stream(torch.cuda.current_stream())


def ctypes_stream(s):
    return s.cuda_stream


# host arrays at least this large go through the library's staged copies
STAGED_MIN_BYTES = 1 << 20


def _staged_ok(arr, dtype):
    dt = np.dtype(dtype)
    return (isinstance(arr, np.ndarray) and arr.flags.c_contiguous and arr.nbytes >= STAGED_MIN_BYTES
            and (arr.dtype == dt or (arr.dtype.kind == dt.kind == "i" and arr.itemsize == 8 and dt.itemsize == 4)))


def _staged_h2d(out, arr):
    _lib.check(_lib.load().uaamg_h2d(out.data_ptr(), arr.ctypes.data, int(arr.shape[0]), int(arr.itemsize),
                                     int(out.element_size()), stream()))
    return out


def to_device(a, dtype):
    """numpy / torch -> contiguous device tensor of ``dtype`` (numpy dtype).
    Large host arrays (e.g. the reference's int64 indices) are copied and
    narrowed through the library's pinned staging pipeline (uaamg_h2d)."""
    dt = _TORCH[np.dtype(dtype)]
    if isinstance(a, torch.Tensor):
        return a.to(device=cuda_device(), dtype=dt).contiguous()
    arr = np.asarray(a)
    if arr.ndim == 1 and _staged_ok(arr, dtype):
        return _staged_h2d(torch.empty(arr.shape[0], dtype=dt, device=cuda_device()), arr)
    arr = np.ascontiguousarray(arr, dtype=dtype)
    return _host_view(arr).to(device=cuda_device(), non_blocking=False)


# Bytes past the end of a level-0 array the TMA tile kernel may read: its
# bulk copies round every slice up to 16-byte granules
# (include/uaamg_b200.h, uaamg_setup_params.borrow).
TAIL_SLACK = 64


def device_empty(n, dtype):
    """Uninitialised device tensor of ``n`` elements with TAIL_SLACK readable
    bytes after the last one (a view of a slightly larger allocation)."""
    dt = _TORCH[np.dtype(dtype)]
    item = np.dtype(dtype).itemsize
    full = torch.empty(int(n) + -(-TAIL_SLACK // item), dtype=dt, device=cuda_device())
    return full[: int(n)]


def _host_view(arr):
    """torch view of a host array without copying it -- also of the
    reference's read-only SparseMatrix arrays (only read here)."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(arr)


def to_device_padded(a, dtype):
    """to_device into a device_empty buffer (borrowable by uaamg_setup)."""
    src = to_device(a, dtype) if isinstance(a, torch.Tensor) else None
    if src is not None and borrowable(src, dtype):
        return src
    if src is None:
        arr = np.asarray(a)
        if arr.ndim == 1 and _staged_ok(arr, dtype):
            return _staged_h2d(device_empty(arr.shape[0], dtype), arr)
        if arr.dtype != np.dtype(dtype) and arr.dtype.kind == np.dtype(dtype).kind and arr.flags.c_contiguous:
            # e.g. the reference's int64 indices -> int32: copy as is, narrow
            # on the device (cheaper than a host conversion pass)
            src = _host_view(arr).to(cuda_device())
        else:
            arr = np.ascontiguousarray(arr, dtype=dtype)
            out = device_empty(arr.shape[0], dtype)
            out.copy_(_host_view(arr))
            return out
    out = device_empty(src.shape[0], dtype)
    out.copy_(src)
    return out


def borrowable(t, dtype):
    """Can uaamg_setup alias ``t`` as a level-0 array: 1-D, contiguous, of
    ``dtype``, on the current device, 16-byte aligned (cp.async.bulk source
    alignment) and with TAIL_SLACK bytes of its storage after the end."""
    if not isinstance(t, torch.Tensor) or t.dtype != _TORCH[np.dtype(dtype)] or t.dim() != 1:
        return False
    if not t.is_cuda or t.device != cuda_device() or not t.is_contiguous():
        return False
    if t.data_ptr() % 16:
        return False
    end = (t.storage_offset() + t.numel()) * t.element_size()
    return t.untyped_storage().nbytes() - end >= TAIL_SLACK


def ptr(t):
    return None if t is None else t.data_ptr()


def to_host(t):
    """device tensor -> numpy (large contiguous tensors through uaamg_d2h)."""
    t = t.detach()
    if t.is_cuda and t.dtype in _NP and t.is_contiguous() and t.numel() * t.element_size() >= STAGED_MIN_BYTES:
        out = np.empty(t.shape, dtype=_NP[t.dtype])
        _lib.check(_lib.load().uaamg_d2h(out.ctypes.data, t.data_ptr(), int(t.numel() * t.element_size()),
                                         stream()))
        return out
    return t.cpu().numpy()


class _CudaView:
    """Minimal __cuda_array_interface__ exporter for library-owned memory."""

    def __init__(self, address, n, dtype, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": (int(n),), "typestr": _TYPESTR[np.dtype(dtype)], "data": (int(address or 0), False),
            "version": 2, "strides": None,
        }


def view(address, n, dtype, owner):
    """Zero-copy torch view of ``n`` elements at a library device address."""
    if n == 0 or not address:
        return torch.empty(0, dtype=_TORCH[np.dtype(dtype)], device=cuda_device())
    return torch.as_tensor(_CudaView(address, n, dtype, owner), device=cuda_device())


class _CsrOwner:
    """Keeps a library-owned CSR alive while torch views of it exist."""

    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            _lib.load().uaamg_csr_free(self.handle)
        except Exception:
            pass


class DeviceCSR:
    """Device CSR matrix: int32 row_ptr/col, float64 val (square)."""

    __slots__ = ("n_rows", "n_cols", "row_ptr", "col", "val", "lib_owned")

    def __init__(self, n_rows, n_cols, row_ptr, col, val, lib_owned=False):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_ptr, self.col, self.val = row_ptr, col, val
        self.lib_owned = lib_owned  # arrays are library buffers (tail slack guaranteed)

    def borrowable(self):
        """Level 0 of a hierarchy may alias these arrays (no copy)."""
        if self.lib_owned:
            ok = all(isinstance(t, torch.Tensor) and t.is_contiguous() and t.data_ptr() % 16 == 0
                     for t in (self.row_ptr, self.col, self.val))
            return ok and self.row_ptr.dtype == torch.int32 and self.col.dtype == torch.int32 \
                and self.val.dtype == torch.float64
        return borrowable(self.row_ptr, np.int32) and borrowable(self.col, np.int32) \
            and borrowable(self.val, np.float64)

    @classmethod
    def from_host(cls, a):
        if a.nnz >= 2 ** 31 or a.n_rows >= 2 ** 31:
            raise ValueError("matrix too large for int32 device indices")
        return cls(a.n_rows, a.n_cols, to_device_padded(a.indptr, np.int32), to_device_padded(a.indices, np.int32),
                   to_device_padded(a.data, np.float64))

    @classmethod
    def from_arrays(cls, n, row_ptr, col, val):
        return cls(n, n, to_device_padded(row_ptr, np.int32), to_device_padded(col, np.int32),
                   to_device_padded(val, np.float64))

    @classmethod
    def _from_lib(cls, handle):
        """Wrap a library-owned uaamg_csr (freed when the last view dies)."""
        import ctypes

        L = _lib.load()
        nr, nc, nnz = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        rp, ci, av = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        L.uaamg_csr_view(handle, ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(nnz), ctypes.byref(rp),
                         ctypes.byref(ci), ctypes.byref(av))
        owner = _CsrOwner(handle)
        return cls(nr.value, nc.value, view(rp.value, nr.value + 1, np.int32, owner),
                   view(ci.value, nnz.value, np.int32, owner), view(av.value, nnz.value, np.float64, owner),
                   lib_owned=True)

    @classmethod
    def from_coo(cls, n_rows, n_cols, rows, cols, vals):
        """Canonical CSR from triplets on the device: reference
        SparseMatrix.from_coo (sparse.py:56-74) -- stable (row, col) sort,
        duplicates summed like np.add.reduceat, exact zeros dropped."""
        import ctypes

        r = to_device(rows, np.int64)
        c = to_device(cols, np.int64)
        v = to_device(vals, np.float64)
        if not (r.shape == c.shape == v.shape) or r.dim() != 1:
            raise ValueError("rows, cols and vals must be 1-D of equal length")
        h = ctypes.c_void_p()
        rc = _lib.load().uaamg_from_coo(int(n_rows), int(n_cols), int(r.shape[0]), ptr(r), ptr(c), ptr(v),
                                        ctypes.byref(h), stream())
        if rc == _lib.UAAMG_EINVAL:
            from .sparse import SparseFormatError
            raise SparseFormatError(_lib.last_error())
        _lib.check(rc)
        return cls._from_lib(h)

    @property
    def nnz(self):
        return int(self.col.shape[0])

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    def to_host(self):
        from .sparse import SparseMatrix
        return SparseMatrix(self.n_rows, self.n_cols, to_host(self.row_ptr).astype(np.int64),
                            to_host(self.col).astype(np.int64), to_host(self.val), _validate=False)

    def spmv(self, x):
        """y = A x (bit-identical to the reference's sequential row sums)."""
        host = not isinstance(x, torch.Tensor)
        xd = to_device(x, np.float64)
        if xd.shape != (self.n_cols,):
            raise ValueError(f"spmv dimension mismatch: matrix {self.shape}, vector {tuple(xd.shape)}")
        y = torch.empty(self.n_rows, dtype=torch.float64, device=xd.device)
        _lib.check(_lib.load().uaamg_k_spmv(self.n_rows, ptr(self.row_ptr), ptr(self.col), ptr(self.val),
                                            ptr(xd), ptr(y), stream()))
        return to_host(y) if host else y

    def __repr__(self):
        return f"DeviceCSR(shape={self.shape}, nnz={self.nnz})"
