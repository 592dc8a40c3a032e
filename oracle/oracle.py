"""ctypes front end of the CPU oracle (oracle/uaamg_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker and the CPU baseline.  The
product package (paper_1302_2547_b200) never imports this module; only
tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) do.

Arrays follow the reference SparseMatrix layout (int64 indptr/indices,
float64 data; /root/reference/pkg/src/uaamg/sparse.py:25-27).  Function names
follow the reference kernel table (pkg/src/uaamg/kernels/__init__.py:39-54)
and drivers (aggregation.py:172, hierarchy.py:120, solvers.py:190).
"""

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_vp = ctypes.c_void_p


class OracleError(RuntimeError):
    pass


def build():
    """Compile liboracle.so with the committed Makefile."""
    env = dict(os.environ)
    env.pop("CC", None)
    subprocess.run(["make", "-s", "-C", _HERE], check=True, env=env)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_setup.restype = _vp
        L.orc_setup.argtypes = [ctypes.c_int64, _vp, _vp, _vp, ctypes.c_uint64, ctypes.c_int64,
                                ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        L.orc_hier_free.argtypes = [_vp]
        L.orc_hier_nlevels.argtypes = [_vp]
        L.orc_hier_singular.argtypes = [_vp]
        L.orc_hier_level.argtypes = [_vp, ctypes.c_int] + [_vp] * 8
        L.orc_npcg_solve.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_double, _vp, ctypes.c_double, ctypes.c_int64,
                                     _vp, _vp, _vp, _vp, _vp]
        L.orc_aggregate.restype = ctypes.c_int64
        L.orc_aggregate.argtypes = [ctypes.c_int64, _vp, _vp, _vp, ctypes.c_uint64, ctypes.c_int64,
                                    ctypes.c_int64, _vp, _vp, _vp]
        L.orc_galerkin.restype = ctypes.c_int64
        L.orc_galerkin.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp, _vp, _vp]
        L.orc_squared_pattern.restype = ctypes.c_int64
        L.orc_squared_pattern.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp]
        L.orc_free.argtypes = [_vp]
        L.orc_hash_u01.argtypes = [ctypes.c_uint64, ctypes.c_int64, _vp, ctypes.c_int64, _vp]
        L.orc_scores.argtypes = [ctypes.c_int64, _vp, _vp, ctypes.c_uint64, ctypes.c_int64, _vp]
        for name in ("orc_spmv",):
            getattr(L, name).argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp, _vp]
        for name in ("orc_diag_of", "orc_l1_diag"):
            getattr(L, name).argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp]
        L.orc_degrees.argtypes = [ctypes.c_int64, _vp, _vp, _vp]
        L.orc_select_centers.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp, _vp]
        L.orc_claim_owners.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp, _vp, _vp]
        L.orc_admit_members.argtypes = [_vp, _vp, _vp, ctypes.c_int64, _vp, _vp, _vp, ctypes.c_int64,
                                        _vp, _vp, ctypes.c_int64]
        L.orc_restrict.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp]
        L.orc_prolongate_add.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp]
        L.orc_smooth_sweeps.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp]
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        L.orc_set_select_mode.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def set_num_threads(n):
    lib().orc_set_num_threads(int(n))


def set_select_mode(mode):
    """0: A^2 pattern unless it would exceed 2^29 entries (then two hops),
    1: always the A^2 pattern (the reference's formulation), 2: always two
    maximum hops over A (no A^2)."""
    lib().orc_set_select_mode(int(mode))


def get_num_threads():
    return int(lib().orc_get_num_threads())


def _p(arr):
    return arr.ctypes.data_as(_vp)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _err():
    return lib().orc_last_error().decode()


# --------------------------------------------------------------------------
# kernel table (K/numba_backend.py)
# --------------------------------------------------------------------------
def hash_u01(seed, pass_idx, idx):
    idx = _i64(idx)
    out = np.empty(idx.shape[0])
    lib().orc_hash_u01(int(seed), int(pass_idx), _p(idx), idx.shape[0], _p(out))
    return out


def spmv(indptr, indices, data, x):
    ip, ix, a, x = _i64(indptr), _i64(indices), _f64(data), _f64(x)
    y = np.empty(ip.shape[0] - 1)
    lib().orc_spmv(y.shape[0], _p(ip), _p(ix), _p(a), _p(x), _p(y))
    return y


def diag_of(indptr, indices, data):
    ip, ix, a = _i64(indptr), _i64(indices), _f64(data)
    y = np.empty(ip.shape[0] - 1)
    lib().orc_diag_of(y.shape[0], _p(ip), _p(ix), _p(a), _p(y))
    return y


def l1_diag(indptr, indices, data):
    ip, ix, a = _i64(indptr), _i64(indices), _f64(data)
    y = np.empty(ip.shape[0] - 1)
    lib().orc_l1_diag(y.shape[0], _p(ip), _p(ix), _p(a), _p(y))
    return y


def degrees(indptr, indices):
    ip, ix = _i64(indptr), _i64(indices)
    y = np.empty(ip.shape[0] - 1, dtype=np.int64)
    lib().orc_degrees(y.shape[0], _p(ip), _p(ix), _p(y))
    return y


def quasi_random_scores(indptr, indices, seed, pass_idx):
    ip, ix = _i64(indptr), _i64(indices)
    y = np.empty(ip.shape[0] - 1)
    lib().orc_scores(y.shape[0], _p(ip), _p(ix), int(seed), int(pass_idx), _p(y))
    return y


def squared_pattern(n, indptr, indices):
    ip, ix = _i64(indptr), _i64(indices)
    pp, px = ctypes.c_void_p(), ctypes.c_void_p()
    m = lib().orc_squared_pattern(int(n), _p(ip), _p(ix), ctypes.byref(pp), ctypes.byref(px))
    ptr = np.ctypeslib.as_array(ctypes.cast(pp, _i64p), shape=(int(n) + 1,)).copy()
    idx = np.ctypeslib.as_array(ctypes.cast(px, _i64p), shape=(max(m, 1),))[:m].copy()
    lib().orc_free(pp)
    lib().orc_free(px)
    return ptr, idx


def galerkin_coo(indptr, indices, data, v2a, n_coarse):
    ip, ix, a, v2a = _i64(indptr), _i64(indices), _f64(data), _i64(v2a)
    pp, px, pv = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    m = lib().orc_galerkin(ip.shape[0] - 1, _p(ip), _p(ix), _p(a), _p(v2a), int(n_coarse),
                           ctypes.byref(pp), ctypes.byref(px), ctypes.byref(pv))
    ptr = np.ctypeslib.as_array(ctypes.cast(pp, _i64p), shape=(int(n_coarse) + 1,)).copy()
    idx = np.ctypeslib.as_array(ctypes.cast(px, _i64p), shape=(max(m, 1),))[:m].copy()
    val = np.ctypeslib.as_array(ctypes.cast(pv, _f64p), shape=(max(m, 1),))[:m].copy()
    for q in (pp, px, pv):
        lib().orc_free(q)
    return ptr, idx, val


def select_centers(a2ptr, a2idx, scores, processed):
    p2, x2, s, pr = _i64(a2ptr), _i64(a2idx), _f64(scores), _u8(processed)
    out = np.empty(p2.shape[0] - 1, dtype=np.uint8)
    lib().orc_select_centers(out.shape[0], _p(p2), _p(x2), _p(s), _p(pr), _p(out))
    return out.astype(bool)


def claim_owners(a2ptr, a2idx, scores, processed, is_center):
    p2, x2, s, pr, ic = _i64(a2ptr), _i64(a2idx), _f64(scores), _u8(processed), _u8(is_center)
    out = np.empty(p2.shape[0] - 1, dtype=np.int64)
    lib().orc_claim_owners(out.shape[0], _p(p2), _p(x2), _p(s), _p(pr), _p(ic), _p(out))
    return out


def admit_members(indptr, indices, data, centers, bucket_ptr, bucket_js, cap, processed,
                  vertex_to_agg, agg_base):
    """In-place on processed (bool/uint8) and vertex_to_agg (int64), like the reference."""
    ip, ix, a = _i64(indptr), _i64(indices), _f64(data)
    c, bp, bj = _i64(centers), _i64(bucket_ptr), _i64(bucket_js)
    pr = np.ascontiguousarray(processed).view(np.uint8) if processed.dtype == bool else processed
    assert vertex_to_agg.dtype == np.int64 and vertex_to_agg.flags.c_contiguous
    lib().orc_admit_members(_p(ip), _p(ix), _p(a), c.shape[0], _p(c), _p(bp), _p(bj), int(cap),
                            _p(pr), _p(vertex_to_agg), int(agg_base))


def restrict(agg_ptr, agg_members, r):
    ap, m, r = _i64(agg_ptr), _i64(agg_members), _f64(r)
    out = np.empty(ap.shape[0] - 1)
    lib().orc_restrict(out.shape[0], _p(ap), _p(m), _p(r), _p(out))
    return out


def prolongate_add(v2a, e_coarse, x):
    v, e, x = _i64(v2a), _f64(e_coarse), _f64(x)
    out = np.empty(x.shape[0])
    lib().orc_prolongate_add(x.shape[0], _p(v), _p(e), _p(x), _p(out))
    return out


def smooth_sweeps(indptr, indices, data, inv_m, x, b, sweeps):
    ip, ix, a, im, b = _i64(indptr), _i64(indices), _f64(data), _f64(inv_m), _f64(b)
    cur = np.array(x, dtype=np.float64, copy=True)
    r = np.empty(cur.shape[0])
    lib().orc_smooth_sweeps(cur.shape[0], _p(ip), _p(ix), _p(a), _p(im), _p(cur), _p(b), int(sweeps), _p(r))
    return cur


# --------------------------------------------------------------------------
# drivers
# --------------------------------------------------------------------------
def aggregate(indptr, indices, data, seed=0, max_passes=20, size_cap=None, with_passes=False):
    """U/aggregation.py:172-203 -> (vertex_to_agg, coarse_vertex_of_agg[, pass_of_center])."""
    ip, ix, a = _i64(indptr), _i64(indices), _f64(data)
    n = ip.shape[0] - 1
    v2a = np.empty(n, dtype=np.int64)
    seeds = np.empty(max(n, 1), dtype=np.int64)
    passes = np.empty(max(n, 1), dtype=np.int64)
    nc = lib().orc_aggregate(n, _p(ip), _p(ix), _p(a), int(seed), int(max_passes),
                             -1 if size_cap is None else int(size_cap), _p(v2a), _p(seeds),
                             _p(passes) if with_passes else None)
    if nc < 0:
        raise OracleError(_err())
    if with_passes:
        return v2a, seeds[:nc].copy(), passes[:n].copy()
    return v2a, seeds[:nc].copy()


@dataclass
class OracleLevel:
    n: int
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray
    vertex_to_agg: np.ndarray | None
    coarse_vertex_of_agg: np.ndarray | None

    @property
    def nnz(self):
        return int(self.indices.shape[0])


class OracleHierarchy:
    """Owns an orc_hier*; levels are copied out to numpy on construction."""

    def __init__(self, handle, copy=True):
        self._h = handle
        L = lib()
        self.singular = bool(L.orc_hier_singular(handle))
        self.levels = []
        for l in range(L.orc_hier_nlevels(handle)):
            n, nnz, nc = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            ptrs = [ctypes.c_void_p() for _ in range(5)]
            L.orc_hier_level(handle, l, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(nc),
                             *[ctypes.byref(q) for q in ptrs])
            n, nnz, nc = n.value, nnz.value, nc.value

            def arr(q, m, t):
                if m == 0 or not q.value:
                    return np.zeros(0, dtype=np.int64 if t is _i64p else np.float64)
                v = np.ctypeslib.as_array(ctypes.cast(q, t), shape=(m,))
                return v.copy() if copy else v  # views live as long as the handle

            ip = arr(ptrs[0], n + 1, _i64p)
            ix = arr(ptrs[1], nnz, _i64p)
            a = arr(ptrs[2], nnz, _f64p)
            v2a = arr(ptrs[3], n, _i64p) if nc else None
            seeds = arr(ptrs[4], nc, _i64p) if nc else None
            self.levels.append(OracleLevel(n, ip, ix, a, v2a, seeds))

    @property
    def n_levels(self):
        return len(self.levels)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_hier_free(self._h)
            self._h = None


def setup(indptr, indices, data, seed=0, max_passes=20, size_cap=None, passes_per_level=1,
          n0=100, max_levels=20, singular=None, copy=True):
    """U/hierarchy.py:120-153 on host CSR arrays."""
    ip, ix, a = _i64(indptr), _i64(indices), _f64(data)
    h = lib().orc_setup(ip.shape[0] - 1, _p(ip), _p(ix), _p(a), int(seed), int(max_passes),
                        -1 if size_cap is None else int(size_cap), int(passes_per_level), int(n0),
                        int(max_levels), -1 if singular is None else int(bool(singular)))
    if not h:
        raise OracleError(_err())
    return OracleHierarchy(h, copy=copy)


@dataclass
class OracleReport:
    iterations: int
    residual_history: list
    converged: bool


def npcg_solve(h, b, tol=1e-6, max_iters=200, x0=None, kind="kcycle", inner_krylov_steps=2,
               pre_sweeps=1, post_sweeps=1, smoother="l1", omega=2.0 / 3.0):
    """U/solvers.py:190-255.  Raises OracleError on NumericalError/ValueError."""
    b = _f64(b)
    n = h.levels[0].n
    x = np.empty(n)
    hist = np.empty(int(max_iters) + 1)
    it = ctypes.c_int64()
    conv = ctypes.c_int()
    x0a = _f64(x0) if x0 is not None else None
    rc = lib().orc_npcg_solve(h._h, int(kind == "kcycle"), int(inner_krylov_steps), int(pre_sweeps),
                              int(post_sweeps), int(smoother == "l1"), float(omega), _p(b), float(tol),
                              int(max_iters), _p(x0a) if x0a is not None else None, _p(x), _p(hist),
                              ctypes.byref(it), ctypes.byref(conv))
    nh = it.value + 1
    rep = OracleReport(it.value, hist[:nh].tolist(), bool(conv.value))
    if rc != 0:
        err = OracleError(_err())
        err.report = rep
        raise err
    return x, rep
