"""ctypes binding of libuaamg_b200.so (the C ABI in include/uaamg_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no fallback: importing a compute entry point without the
library, or without a CUDA device, raises immediately.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libuaamg_b200.so")

UAAMG_OK = 0
UAAMG_EINVAL = -1
UAAMG_ECUDA = -2
UAAMG_ENUMERICAL = -3
UAAMG_ESETUP = -4
UAAMG_EAGG = -5
UAAMG_ENOMEM = -6
UAAMG_EUNSUPPORTED = -7

_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_d = ctypes.c_double


class SetupParams(ctypes.Structure):
    _fields_ = [("size_cap", _i64), ("seed", _u64), ("max_passes", _i), ("passes_per_level", _i),
                ("n0", _i), ("max_levels", _i), ("singular", _i), ("reshape_sweeps", _i),
                ("reshape_pair_cap", _i), ("borrow", _i)]


class HierarchyInfo(ctypes.Structure):
    _fields_ = [("n_levels", _i), ("singular", _i), ("grid_complexity", _d), ("operator_complexity", _d),
                ("setup_seconds", _d)]


class LevelView(ctypes.Structure):
    _fields_ = [("n", _i), ("nnz", _i64), ("row_ptr", _vp), ("col", _vp), ("val", _vp), ("n_coarse", _i),
                ("vertex_to_agg", _vp), ("coarse_vertex_of_agg", _vp), ("agg_ptr", _vp), ("members", _vp)]


class DHierInfo(ctypes.Structure):
    _fields_ = [("n_levels", _i), ("n_sharded", _i), ("singular", _i), ("grid_complexity", _d),
                ("operator_complexity", _d), ("setup_seconds", _d)]


class DLevelView(ctypes.Structure):
    _fields_ = [("n", _i), ("nnz", _i64), ("sharded", _i), ("row_begin", _i), ("row_end", _i), ("local_nnz", _i64),
                ("row_ptr", _vp), ("col", _vp), ("val", _vp), ("n_coarse", _i), ("vertex_to_agg", _vp),
                ("seeds", _vp), ("n_seeds", _i)]


class SolveParams(ctypes.Structure):
    _fields_ = [("kcycle", _i), ("inner_krylov_steps", _i), ("pre_sweeps", _i), ("post_sweeps", _i),
                ("smoother_l1", _i), ("omega", _d), ("tol", _d), ("max_iters", _i), ("use_graphs", _i),
                ("profile_level0", _i)]


class SolveResult(ctypes.Structure):
    _fields_ = [("iterations", _i), ("converged", _i), ("status", _i), ("solve_seconds", _d),
                ("l0_kernel_launches", _i64), ("l0_kernel_seconds", _d), ("l0_kernel_bytes", _d)]


_SIGS = {
    "uaamg_version": (_i, []),
    "uaamg_last_error": (ctypes.c_char_p, []),
    "uaamg_launch_count": (_u64, []),
    "uaamg_k_hash_u01": (_i, [_u64, _i64, _vp, _i64, _vp, _vp]),
    "uaamg_k_spmv": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_diag_of": (_i, [_i, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_l1_diag": (_i, [_i, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_degrees": (_i, [_i, _vp, _vp, _vp, _vp]),
    "uaamg_k_quasi_random_scores": (_i, [_i, _vp, _vp, _u64, _i64, _vp, _vp]),
    "uaamg_k_squared_pattern": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_select_centers": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_select_centers_2hop": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_claim_owners": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_claim_owners_2hop": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_admit_members": (_i, [_i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i64, _vp, _vp, _i, _vp]),
    "uaamg_k_galerkin": (_i, [_i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_restrict": (_i, [_i, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_prolongate_add": (_i, [_i, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_k_smooth_sweeps": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp]),
    "uaamg_aggregate": (_i, [_i, _vp, _vp, _vp, _u64, _i, _i64, _vp, _vp, _vp, _vp]),
    "uaamg_setup": (_i, [_i, _i64, _vp, _vp, _vp, ctypes.POINTER(SetupParams), ctypes.POINTER(_vp), _vp]),
    "uaamg_setup_host": (_i, [_i64, _i64, _vp, _vp, _vp, ctypes.POINTER(SetupParams), ctypes.POINTER(_vp), _vp]),
    "uaamg_hierarchy_free": (None, [_vp]),
    "uaamg_hierarchy_get_info": (_i, [_vp, ctypes.POINTER(HierarchyInfo)]),
    "uaamg_hierarchy_level": (_i, [_vp, _i, ctypes.POINTER(LevelView)]),
    "uaamg_coarse_factor": (_i, [_i, _i64, _vp, _vp, _vp, _i, _vp, ctypes.POINTER(_i), _vp]),
    "uaamg_hierarchy_coarse": (_i, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_i), ctypes.POINTER(_i)]),
    "uaamg_dense_apply": (_i, [_i, _vp, _vp, _i, _vp, _vp]),
    "uaamg_npcg_solve": (_i, [_vp, ctypes.POINTER(SolveParams), _vp, _vp, _vp, _vp, ctypes.POINTER(SolveResult),
                              _vp]),
    "uaamg_comm_create": (_i, [_i, _i, _i64, ctypes.POINTER(_vp)]),
    "uaamg_comm_handle": (_i, [_vp, _vp]),
    "uaamg_comm_connect": (_i, [_vp, _vp]),
    "uaamg_comm_barrier": (_i, [_vp]),
    "uaamg_comm_free": (None, [_vp]),
    "uaamg_dsetup": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(SetupParams), _i64, ctypes.POINTER(_vp),
                          _vp]),
    "uaamg_dhier_free": (None, [_vp]),
    "uaamg_dhier_get_info": (_i, [_vp, ctypes.POINTER(DHierInfo)]),
    "uaamg_dhier_level": (_i, [_vp, _i, _i, ctypes.POINTER(DLevelView)]),
    "uaamg_dsolve": (_i, [_vp, ctypes.POINTER(SolveParams), _vp, _vp, _vp, _vp, ctypes.POINTER(SolveResult), _vp]),
    "uaamg_partition_rows": (_i, [_i, _i, _vp]),
    "uaamg_h2d": (_i, [_vp, _vp, _i64, _i, _i, _vp]),
    "uaamg_reshape_sweep": (_i, [_i, _i64, _vp, _vp, _vp, _i, _vp, _vp, _i, _d, _i, _i, _vp, _vp]),
    "uaamg_d2h": (_i, [_vp, _vp, _i64, _vp]),
    "uaamg_coarse_bounds": (_i, [_vp, _i, _vp]),
    "uaamg_gen_grid3d": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_gen_grid3d_rows": (_i, [_i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_from_coo": (_i, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_assemble_laplacian": (_i, [_i, ctypes.c_int64, _vp, _vp, _vp, ctypes.c_int64, _vp, _vp, _vp, _vp]),
    "uaamg_csr_view": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "uaamg_csr_free": (None, [_vp]),
    "uaamg_solve_profile": (_i, [_vp, _vp, _vp, _vp]),
    "uaamg_tail_info": (_i, [_vp, _vp, _vp]),
    "uaamg_level_kernel": (_i, [_vp, _i, _vp]),
    "uaamg_cycle": (_i, [_vp, ctypes.POINTER(SolveParams), _i, _vp, _vp, _vp]),
    "uaamg_smooth": (_i, [_vp, ctypes.POINTER(SolveParams), _i, _vp, _vp, _i, _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load the shared library (raises OSError if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} not found: run __graft_entry__.build() (nvcc, sm_100a) first; "
                          "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error():
    return load().uaamg_last_error().decode(errors="replace")


def launch_count():
    return int(load().uaamg_launch_count())


def check(rc, what=""):
    """Map a UAAMG_E* code to the reference's exception types."""
    if rc == UAAMG_OK:
        return
    check_code(rc, last_error() or what)


def check_code(rc, msg):
    """check() with the error message already read."""
    if rc == UAAMG_OK:
        return
    if rc == UAAMG_EINVAL:
        raise ValueError(msg)
    if rc == UAAMG_ENUMERICAL:
        from .solvers import NumericalError
        raise NumericalError(msg)
    if rc == UAAMG_ESETUP:
        from .hierarchy import SetupError
        raise SetupError(msg)
    if rc == UAAMG_EAGG:
        from .aggregation import AggregationError
        raise AggregationError(msg)
    if rc == UAAMG_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"uaamg CUDA error: {msg}")
