"""The reference kernel table, backed by the B200 kernels.

Same 16 names and numpy calling conventions as the reference backends
(/root/reference/pkg/src/uaamg/kernels/__init__.py:39-54; contracts in
kernels/numba_backend.py).  Each call uploads its arguments, runs the sm_100a
kernel through the C ABI (include/uaamg_b200.h, ``uaamg_k_*``) and downloads
the result -- this is the per-kernel drop-in surface and the subject of the
per-kernel parity tests; the setup/solve drivers keep everything on device.
Index outputs are int64 like the reference's; device arrays are int32.
"""

import numpy as np
import torch

from . import _lib
from .device import ptr, stream, to_device, to_host

NAME = "b200"


def set_num_threads(n):
    """No-op: results never depend on parallelism (reference numba_backend.py:21-22)."""
    return None


def _dev(a, dt):
    return to_device(a, dt)


def _f64(n):
    return torch.empty(max(int(n), 0), dtype=torch.float64, device="cuda")


def hash_u01(seed, pass_idx, idx):
    i = _dev(idx, np.int64)
    out = _f64(i.shape[0])
    _lib.check(_lib.load().uaamg_k_hash_u01(int(np.uint64(seed)), int(pass_idx), ptr(i), i.shape[0], ptr(out),
                                            stream()))
    return to_host(out)


def _csr(indptr, indices, data=None):
    ip = _dev(indptr, np.int32)
    ix = _dev(indices, np.int32)
    a = _dev(data, np.float64) if data is not None else None
    return ip.shape[0] - 1, ip, ix, a


def spmv(indptr, indices, data, x):
    n, ip, ix, a = _csr(indptr, indices, data)
    xd = _dev(x, np.float64)
    y = _f64(n)
    _lib.check(_lib.load().uaamg_k_spmv(n, ptr(ip), ptr(ix), ptr(a), ptr(xd), ptr(y), stream()))
    return to_host(y)


def diag_of(indptr, indices, data):
    n, ip, ix, a = _csr(indptr, indices, data)
    y = _f64(n)
    _lib.check(_lib.load().uaamg_k_diag_of(n, ptr(ip), ptr(ix), ptr(a), ptr(y), stream()))
    return to_host(y)


def l1_diag(indptr, indices, data):
    n, ip, ix, a = _csr(indptr, indices, data)
    y = _f64(n)
    _lib.check(_lib.load().uaamg_k_l1_diag(n, ptr(ip), ptr(ix), ptr(a), ptr(y), stream()))
    return to_host(y)


def degrees(indptr, indices):
    n, ip, ix, _ = _csr(indptr, indices)
    y = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().uaamg_k_degrees(n, ptr(ip), ptr(ix), ptr(y), stream()))
    return to_host(y).astype(np.int64)


def quasi_random_scores(indptr, indices, seed, pass_idx):
    n, ip, ix, _ = _csr(indptr, indices)
    y = _f64(n)
    _lib.check(_lib.load().uaamg_k_quasi_random_scores(n, ptr(ip), ptr(ix), int(np.uint64(seed)), int(pass_idx),
                                                       ptr(y), stream()))
    return to_host(y)


def squared_pattern(n, indptr, indices):
    n, ip, ix, _ = _csr(indptr, indices)
    optr = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    m = np.zeros(1, dtype=np.int64)
    L = _lib.load()
    # single call computes both (count + fill); sized by a first counting call
    _lib.check(L.uaamg_k_squared_pattern(n, ptr(ip), ptr(ix), ptr(optr), None, m.ctypes.data, stream()))
    oidx = torch.empty(max(int(m[0]), 1), dtype=torch.int32, device="cuda")
    _lib.check(L.uaamg_k_squared_pattern(n, ptr(ip), ptr(ix), ptr(optr), ptr(oidx), m.ctypes.data, stream()))
    return to_host(optr).astype(np.int64), to_host(oidx)[: int(m[0])].astype(np.int64)


def galerkin_coo(indptr, indices, data, v2a, n_coarse):
    n, ip, ix, a = _csr(indptr, indices, data)
    v = _dev(v2a, np.int32)
    nc = int(n_coarse)
    optr = torch.empty(nc + 1, dtype=torch.int32, device="cuda")
    m = np.zeros(1, dtype=np.int64)
    L = _lib.load()
    _lib.check(L.uaamg_k_galerkin(n, ptr(ip), ptr(ix), ptr(a), ptr(v), nc, ptr(optr), None, None, m.ctypes.data,
                                  stream()))
    mm = max(int(m[0]), 1)
    ocol = torch.empty(mm, dtype=torch.int32, device="cuda")
    oval = _f64(mm)
    _lib.check(L.uaamg_k_galerkin(n, ptr(ip), ptr(ix), ptr(a), ptr(v), nc, ptr(optr), ptr(ocol), ptr(oval),
                                  m.ctypes.data, stream()))
    k = int(m[0])
    return to_host(optr).astype(np.int64), to_host(ocol)[:k].astype(np.int64), to_host(oval)[:k]


def select_centers(a2ptr, a2idx, scores, processed):
    n, ip, ix, _ = _csr(a2ptr, a2idx)
    s = _dev(scores, np.float64)
    pr = _dev(np.asarray(processed, dtype=np.uint8), np.uint8)
    out = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.load().uaamg_k_select_centers(n, ptr(ip), ptr(ix), ptr(s), ptr(pr), ptr(out), stream()))
    return to_host(out).astype(bool)


def claim_owners(a2ptr, a2idx, scores, processed, is_center):
    n, ip, ix, _ = _csr(a2ptr, a2idx)
    s = _dev(scores, np.float64)
    pr = _dev(np.asarray(processed, dtype=np.uint8), np.uint8)
    ic = _dev(np.asarray(is_center, dtype=np.uint8), np.uint8)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().uaamg_k_claim_owners(n, ptr(ip), ptr(ix), ptr(s), ptr(pr), ptr(ic), ptr(out), stream()))
    return to_host(out).astype(np.int64)


def admit_members(indptr, indices, data, centers, bucket_ptr, bucket_js, cap, processed, vertex_to_agg, agg_base):
    """In place on ``processed`` and ``vertex_to_agg`` (reference numba_backend.py:223-273)."""
    n, ip, ix, a = _csr(indptr, indices, data)
    c = _dev(centers, np.int32)
    bp = _dev(bucket_ptr, np.int32)
    bj = _dev(bucket_js if len(bucket_js) else np.zeros(1, dtype=np.int64), np.int32)
    pr = _dev(np.asarray(processed, dtype=np.uint8), np.uint8)
    v = _dev(vertex_to_agg, np.int32)
    capv = int(cap)
    capv = capv if capv < 2 ** 62 else 0
    _lib.check(_lib.load().uaamg_k_admit_members(n, ptr(ip), ptr(ix), ptr(a), c.shape[0], ptr(c), ptr(bp), ptr(bj),
                                                 capv, ptr(pr), ptr(v), int(agg_base), stream()))
    processed[:] = to_host(pr).astype(processed.dtype)
    vertex_to_agg[:] = to_host(v)


def restrict(agg_ptr, agg_members, r):
    nc, ap, mem, _ = _csr(agg_ptr, agg_members)
    rd = _dev(r, np.float64)
    out = _f64(nc)
    _lib.check(_lib.load().uaamg_k_restrict(nc, ptr(ap), ptr(mem), ptr(rd), ptr(out), stream()))
    return to_host(out)


def prolongate_add(v2a, e_coarse, x):
    v = _dev(v2a, np.int32)
    e = _dev(e_coarse, np.float64)
    xd = _dev(x, np.float64)
    out = _f64(xd.shape[0])
    _lib.check(_lib.load().uaamg_k_prolongate_add(xd.shape[0], ptr(v), ptr(e), ptr(xd), ptr(out), stream()))
    return to_host(out)


def smooth_sweeps(indptr, indices, data, inv_m, x, b, sweeps):
    n, ip, ix, a = _csr(indptr, indices, data)
    im = _dev(inv_m, np.float64)
    xd = _dev(x, np.float64)
    bd = _dev(b, np.float64)
    out = _f64(n)
    _lib.check(_lib.load().uaamg_k_smooth_sweeps(n, ptr(ip), ptr(ix), ptr(a), ptr(im), ptr(xd), ptr(bd), int(sweeps),
                                                 ptr(out), stream()))
    return to_host(out)


# 2-hop variants (no A^2): the selection/claim the B200 setup path runs
def select_centers_2hop(indptr, indices, scores, processed):
    n, ip, ix, _ = _csr(indptr, indices)
    s = _dev(scores, np.float64)
    pr = _dev(np.asarray(processed, dtype=np.uint8), np.uint8)
    out = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.load().uaamg_k_select_centers_2hop(n, ptr(ip), ptr(ix), ptr(s), ptr(pr), ptr(out), stream()))
    return to_host(out).astype(bool)


def claim_owners_2hop(indptr, indices, scores, processed, is_center):
    n, ip, ix, _ = _csr(indptr, indices)
    s = _dev(scores, np.float64)
    pr = _dev(np.asarray(processed, dtype=np.uint8), np.uint8)
    ic = _dev(np.asarray(is_center, dtype=np.uint8), np.uint8)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().uaamg_k_claim_owners_2hop(n, ptr(ip), ptr(ix), ptr(s), ptr(pr), ptr(ic), ptr(out),
                                                     stream()))
    return to_host(out).astype(np.int64)
