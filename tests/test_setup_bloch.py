"""Host-logic parity of the NEXT-4 Bloch operators (no GPU): the library's fp64 setup_bloch_ops
(host-only context, pmfem_build_bloch + pmfem_export) vs the oracle (oracle/bloch_heff.py,
pinned in test_oracle_bloch_heff.py).  Bars as test_setup_parity: 1e-12 for the closed-form
assembly and the precorrection, 3e-8 of max |Z0| for the two independent quadratures, 1e-10
for the kernel half spectra (fp64 Ewald tables of two implementations)."""
import numpy as np
import pytest

from helpers import lib_context, bloch_oracle, bloch_k0, dense_c

KEYS = ["C1r1", "C2p2", "R1p2"]


@pytest.fixture(scope="module", params=KEYS)
def pair(request):
    key = request.param
    ctx = lib_context(key, device=-1)
    ctx.build_bloch(bloch_k0(key))
    return key, bloch_oracle(key), ctx


def test_bloch_local_operators(pair):
    key, bm, ctx = pair
    n = bm.n_parents
    R = dense_c(ctx, "bloch_r1", 7, n)
    o = bm.ops
    refs = [-o["S"].toarray() / o["Vt"][:, None]] + [o[k].toarray() for k in ("Dx", "Dy", "Dz", "Gx", "Gy", "Gz")]
    for x, ref in enumerate(refs):
        assert np.abs(R[:, :, x] - ref).max() <= 1e-12 * np.abs(ref).max(), x
    # the phases matter: some entry is genuinely complex
    assert np.abs(R[:, :, 1].imag).max() > 1e-3 * np.abs(R[:, :, 1]).max()


def test_bloch_z0(pair):
    key, bm, ctx = pair
    Z = dense_c(ctx, "bloch_z0", 3, bm.n_parents)
    for x, nm in enumerate(("Zx", "Zy", "Zz")):
        ref = bm.z0[nm].toarray()
        assert np.abs(Z[:, :, x] - ref).max() <= 3e-8 * np.abs(ref).max()


def test_bloch_modulation_and_cbox(pair):
    key, bm, ctx = pair
    md = ctx.export("bloch_mod")
    assert np.abs(md[0::2] + 1j * md[1::2] - bm.mod).max() <= 1e-12
    C = dense_c(ctx, "bloch_cbox", 1, bm.n_parents)[:, :, 0]
    ref = bm.C.toarray()
    assert np.abs(C - ref).max() <= 1e-12 * np.abs(ref).max()


def test_bloch_half_spectra(pair):
    key, bm, ctx = pair
    P = bm.grid.fft
    tot = float(np.prod(P))
    H0 = P[0] // 2 + 1
    # oracle: FFT of Re G~ (real) and of Im G~ (imaginary), [x][y][z] -> [z][y][x], x < H0
    fa = (np.fft.fftn(bm.K.real) / tot).transpose(2, 1, 0)[:, :, :H0]
    fb = (np.fft.fftn(bm.K.imag) / tot).transpose(2, 1, 0)[:, :, :H0]
    assert np.abs(fa.imag).max() <= 1e-12 * np.abs(fa).max()      # even kernel part
    assert np.abs(fb.real).max() <= 1e-12 * np.abs(fb).max()      # odd kernel part
    ga = ctx.export("bloch_fa").reshape(fa.shape)
    gb = ctx.export("bloch_fb").reshape(fb.shape)
    assert np.abs(ga - fa.real).max() <= 1e-10 * np.abs(fa).max()
    assert np.abs(gb - fb.imag).max() <= 1e-10 * np.abs(fb).max()
