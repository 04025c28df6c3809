"""The C-ABI library loads and exports every symbol include/pmfem.h declares (no GPU needed)."""
import ctypes
import os
import re

from paper_2409_13958_b200 import LIB_PATH, library_symbols

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "pmfem.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pmfem_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(LIB_PATH)
    names = declared_symbols()
    assert "pmfem_setup" in names and "pmfem_heff" in names and len(names) >= 13
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_symbols():
    assert all(library_symbols().values())


def test_error_path_no_gpu():
    # invalid arguments are reported with a status and a message, never an exception/abort
    import numpy as np
    from paper_2409_13958_b200 import Context, PmfemError
    xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    tets = np.array([[0, 1, 2, 3]])
    try:
        Context(xyz, tets, (1, 0, 0), (0, 0, 0), (8, 8, 8), device=-1)
    except PmfemError as e:
        assert e.status == 1 and "period" in str(e)
    else:
        raise AssertionError("expected PMFEM_E_INVALID_ARG")
    try:
        Context(xyz, np.array([[0, 1, 2, 7]]), (1, 0, 0), (1.0, 0, 0), (8, 8, 8), device=-1)
    except PmfemError as e:
        assert e.status == 2
    else:
        raise AssertionError("expected PMFEM_E_MESH")
