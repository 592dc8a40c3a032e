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
