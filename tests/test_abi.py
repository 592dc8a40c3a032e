"""The C-ABI library loads and exports every symbol include/uaamg_b200.h
declares (no compute calls: this runs without a GPU)."""

import ctypes
import os
import re

from paper_1302_2547_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "uaamg_b200.h")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(uaamg_\w+)\s*\(", txt)))


def test_header_declares_entry_points():
    names = declared()
    assert "uaamg_setup" in names and "uaamg_npcg_solve" in names and "uaamg_k_spmv" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(L, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    assert sorted(_lib.EXPORTED) == declared()


def test_version_and_error_string():
    L = _lib.load()
    assert L.uaamg_version() == 1
    assert isinstance(_lib.last_error(), str)


def test_setup_host_validates_before_touching_the_device():
    """uaamg_setup_host (the reference's int64 host layout) rejects malformed
    row pointers and sizes with UAAMG_EINVAL before any CUDA call, so this
    runs without a GPU."""
    import numpy as np
    L = _lib.load()
    P = _lib.SetupParams(size_cap=0, seed=0, max_passes=20, passes_per_level=1, n0=100, max_levels=20, singular=-1,
                         reshape_sweeps=0, reshape_pair_cap=16, borrow=0)
    h = ctypes.c_void_p()
    ix = np.array([0, 1, 0, 1], dtype=np.int64)
    av = np.array([2.0, -1.0, -1.0, 2.0])
    for ip, n, nnz in ((np.array([1, 2, 4], dtype=np.int64), 2, 4),    # indptr[0] != 0
                       (np.array([0, 2, 3], dtype=np.int64), 2, 4),    # indptr[n] != nnz
                       (np.array([0], dtype=np.int64), 0, 0)):        # empty
        rc = L.uaamg_setup_host(n, nnz, ip.ctypes.data, ix.ctypes.data, av.ctypes.data, ctypes.byref(P),
                                ctypes.byref(h), None)
        assert rc == _lib.UAAMG_EINVAL, rc
        assert _lib.last_error()
