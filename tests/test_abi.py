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


def _tiny_periodic():
    from synth import make_config
    cfg = make_config("C1", coarsen=5)
    return cfg


def test_lattice_vectors_must_be_diagonal():
    # pmfem_periodicity.lattice holds 3x3 lattice vectors (rows); P:36 uses L_x x, L_y y, L_z z
    from paper_2409_13958_b200 import Context, PmfemError
    cfg = _tiny_periodic()
    m = cfg["mesh"]
    L = cfg["lattice"][0]
    lat = [[L, 0, 0], [0, L, 0], [0, 0, L]]
    ctx = Context(m.xyz, m.tets, cfg["periodic"], lat, (8, 8, 8), rer_scale=1.0, device=-1)
    assert ctx.n_parents > 0
    ctx.close()
    lat[0][1] = 0.1 * L
    try:
        Context(m.xyz, m.tets, cfg["periodic"], lat, (8, 8, 8), rer_scale=1.0, device=-1)
    except PmfemError as e:
        assert e.status == 1 and "diagonal" in str(e)
    else:
        raise AssertionError("expected PMFEM_E_INVALID_ARG for a sheared lattice")


def test_pgf_target_and_achieved_error():
    # build_pgf honours target_rel_err: the measured truncation error is reported, and a target
    # below fp64 resolution fails with PMFEM_E_PGF_NOT_CONVERGED
    from paper_2409_13958_b200 import Context, PmfemError
    cfg = _tiny_periodic()
    m = cfg["mesh"]
    ctx = Context(m.xyz, m.tets, cfg["periodic"], cfg["lattice"], (8, 8, 8), rer_scale=1.0, device=-1)
    ctx.build_pgf(1e-6)
    a6 = ctx.query()["pgf_achieved_rel_err"]
    assert 0 < a6 <= 1e-6
    ctx.build_pgf(1e-12)
    a12 = ctx.query()["pgf_achieved_rel_err"]
    assert a12 <= 1e-12
    try:
        ctx.build_pgf(1e-22)
    except PmfemError as e:
        assert e.status == 7 and "above target" in str(e)
    else:
        raise AssertionError("expected PMFEM_E_PGF_NOT_CONVERGED")
    ctx.close()
