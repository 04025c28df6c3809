"""GPU-built setup artifacts. C_box (cbox_gpu.cu, device contexts) vs the host-built one
(setup_aim.cpp, host-only contexts) -- itself pinned to the oracle by test_setup_parity.py.
Same near set (exact), values equal to fp32 storage rounding."""
import numpy as np
import pytest

from helpers import SMALL, lib_context

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt", ["u4", "seg", "c4x", "b4", "w4"])
@pytest.mark.parametrize("key", sorted(SMALL))
def test_device_cbox_matches_host(key, fmt, monkeypatch):
    """Both packed C_box formats (C4x chunks, B4 aligned blocks) decode to the host matrix."""
    monkeypatch.setenv("PMFEM_CBOX_FORMAT", fmt)
    dev = lib_context(key, device=0)
    assert dev.export("cbox_device_format")[0] == {"c4x": 0, "b4": 1, "seg": 2, "u4": 3, "w4": 5}[fmt]
    host = lib_context(key, device=-1)
    n = host.n_parents
    perm = dev.export("perm")                     # internal -> user parent id
    rp = dev.export("cbox_device_rowptr")
    col = dev.export("cbox_device_col")
    val = dev.export("cbox_device_val").astype(np.float64)
    D = np.zeros((n, n))
    for i in range(n):
        for e in range(rp[i], rp[i + 1]):
            if val[e] != 0.0:                           # skip padding / empty block slots
                D[perm[i], perm[col[e]]] += val[e]
    hrp = host.export("cbox_rowptr")
    hcol = host.export("cbox_col")
    hval = host.export("cbox_val")
    Hm = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(hrp))
    np.add.at(Hm, (rows, hcol), hval)
    assert np.array_equal(D != 0, Hm != 0)
    assert np.abs(D - Hm).max() <= 1e-6 * np.abs(Hm).max()
    assert dev.query()["nnz_cbox"] == hcol.size


@pytest.mark.parametrize("key", sorted(SMALL))
def test_device_z0_matches_host(key):
    """Z0 element integrals on the GPU (z0_gpu.cu) vs the host (same cone quadrature, fp64)."""
    dev = lib_context(key, device=0)
    host = lib_context(key, device=-1)
    for name in ("z0_rowptr", "z0_col"):
        assert np.array_equal(dev.export(name), host.export(name))
    a, b = dev.export("z0_val"), host.export("z0_val")
    assert np.abs(a - b).max() <= 1e-11 * np.abs(b).max()
    a, b = dev.export("rowsumZ"), host.export("rowsumZ")
    assert np.abs(a - b).max() <= 1e-11 * np.abs(host.export("z0_val")).max()


@pytest.mark.parametrize("key,k0", [("C1r0", (3.0e5, -1.0e5, 2.0e5)), ("C3p1", (1.0e5, 0, 0)),
                                    ("C2p2", (-2.0e5, 1.5e5, 0)), ("R1p2", (0, 0, 4.0e5))])
def test_device_bloch_kernel_matches_host(key, k0):
    """NEXT-4: the Bloch-phase kernel tabulated on the GPU (k_pgf_table_bloch, fp64) equals the
    host table, itself pinned to the oracle (tests/test_oracle_bloch.py)."""
    dev = lib_context(key, device=0)
    host = lib_context(key, device=-1)
    Kd, Gd = dev.build_pgf_bloch(k0)
    Kh, Gh = host.build_pgf_bloch(k0)
    assert np.abs(Kd - Kh).max() <= 1e-12 * np.abs(Kh).max()
    assert np.abs(Gd - Gh).max() <= 1e-12 * np.abs(Gh).max()
