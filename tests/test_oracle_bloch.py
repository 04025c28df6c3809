"""Oracle pins: the Bloch-phase periodic Green's function (NEXT-4; Eq. 2 with k0 != 0).

* Bloch shift G(r + L_a e_a; k0) = exp(-j k0_a L_a) G(r; k0) on every periodic axis;
* independence of the Ewald splitting parameter;
* the 1D zone-boundary closed form (k0 = pi/L): sum_n (-1)^n / |x - nL| = [beta(x/L) - beta(1 - x/L)] / L;
* k0 -> 0: G(r; k0) minus its G = 0 reciprocal term tends to the static kernel (oracle/pgf.py)
  minus the static normalisation's zero-mode term, in 1D, 2D and 3D."""
import math

import numpy as np
import pytest

from oracle import bloch as B
from oracle import pgf as P

CASES = [((1, 0, 0), (1.0, 0, 0), (0.9, 0, 0)), ((0, 0, 1), (0, 0, 1.3), (0, 0, -1.7)),
         ((1, 1, 0), (1.0, 1.2, 0), (0.8, -1.1, 0)), ((1, 1, 1), (1.0, 1.1, 0.9), (0.7, 1.3, -0.4))]


@pytest.mark.parametrize("per,lat,k0", CASES)
def test_bloch_shift(per, lat, k0):
    s = B.BlochSpec(per, lat, k0)
    r = np.random.default_rng(2).uniform(-0.6, 0.6, (6, 3))
    g = B.bloch_pgf(r, s)
    for a in range(3):
        if not per[a]:
            continue
        sh = np.zeros(3)
        sh[a] = lat[a]
        for n in (1, -2):
            gs = B.bloch_pgf(r + n * sh, s)
            assert np.allclose(gs, np.exp(-1j * k0[a] * n * lat[a]) * g, rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("per,lat,k0", CASES)
def test_bloch_alpha_independence(per, lat, k0):
    r = np.random.default_rng(4).uniform(-0.7, 0.7, (5, 3))
    a = B.bloch_pgf(r, B.BlochSpec(per, lat, k0, alpha=math.sqrt(math.pi)))
    b = B.bloch_pgf(r, B.BlochSpec(per, lat, k0, alpha=2 * math.sqrt(math.pi)))
    assert np.allclose(a, b, rtol=1e-11, atol=1e-11)
    sa = B.bloch_pgf(None, B.BlochSpec(per, lat, k0, alpha=math.sqrt(math.pi)), self_term=True)
    sb = B.bloch_pgf(None, B.BlochSpec(per, lat, k0, alpha=2 * math.sqrt(math.pi)), self_term=True)
    assert np.allclose(sa, sb, rtol=1e-11, atol=1e-11)


def test_bloch_1d_zone_boundary_closed_form():
    L = 1.0
    s = B.BlochSpec((1, 0, 0), (L, 0, 0), (math.pi / L, 0, 0))
    for x in (0.2, 0.5, 0.85):
        g = B.bloch_pgf(np.array([[x, 0.0, 0.0]]), s)[0]
        ref = (B.beta_dirichlet(x / L) - B.beta_dirichlet(1 - x / L)) / L
        assert g.real == pytest.approx(ref, rel=1e-11) and abs(g.imag) < 1e-11


@pytest.mark.parametrize("per,lat", [((1, 0, 0), (1.0, 0, 0)), ((1, 1, 0), (1.0, 1.0, 0)),
                                     ((1, 1, 1), (1.0, 1.0, 1.0))])
def test_bloch_static_limit(per, lat):
    r = np.random.default_rng(6).uniform(-0.4, 0.4, (5, 3))
    st = P.PgfSpec(per, lat)
    g0 = P.pgf(r, st) - B.static_zero_mode(r, B.BlochSpec(per, lat, (1, 1, 1)))
    for eps in (1e-4, 1e-5):
        k0 = tuple(eps * 2 * math.pi * v for v in (1.0, 0.6, 0.3))
        s = B.BlochSpec(per, lat, k0, alpha=st.alpha)
        g = B.bloch_pgf(r, s) - B.zero_mode(r, s)
        assert np.allclose(g, g0, rtol=0, atol=50 * eps)


# ---- library Bloch kernel (host-only contexts) vs this oracle
def _lib_vs_oracle(key, k0):
    from helpers import config, lib_context
    from oracle import aim
    cfg, spec = config(key)
    ctx = lib_context(key, device=-1)
    K, G = ctx.build_pgf_bloch(k0)
    om_grid = aim.Grid(spec["grid"], cfg["periodic"],
                       tuple(float(cfg["lattice"][a]) if cfg["periodic"][a] else 0.0 for a in range(3)),
                       ctx.export("xw").reshape(-1, 3))
    P = om_grid.fft
    axes = []
    for a in range(3):
        j = np.arange(P[a])
        axes.append((j if cfg["periodic"][a] else np.where(j < om_grid.n[a], j, j - P[a])) * om_grid.delta[a])
    D = np.stack(np.meshgrid(*axes, indexing="ij"), -1).reshape(-1, 3)
    s = B.BlochSpec(cfg["periodic"], cfg["lattice"], k0)
    ref = np.zeros(D.shape[0], complex)
    nz = np.any(D != 0, axis=1)
    kr = D @ np.array(k0, dtype=float)
    ref[nz] = np.exp(1j * kr[nz]) * B.bloch_pgf(D[nz], s)
    ref[~nz] = B.bloch_pgf(None, s, self_term=True)[0]
    for a in range(3):                       # K6: the unused index N on padded axes is 0
        if not cfg["periodic"][a]:
            sl = [slice(None)] * 3
            sl[a] = om_grid.n[a]
            r3 = ref.reshape(tuple(P))
            r3[tuple(sl)] = 0
    ref = ref.reshape(tuple(P))
    Kl = np.transpose(K, (2, 1, 0))          # library [P2][P1][P0] -> [x][y][z]
    assert np.abs(Kl - ref).max() <= 1e-11 * np.abs(ref).max()
    Gl = np.transpose(G, (2, 1, 0))
    Gref = np.fft.fftn(ref) / ref.size
    assert np.abs(Gl - Gref).max() <= 1e-11 * np.abs(Gref).max()


@pytest.mark.parametrize("key,k0", [("C1r0", (3.0e5, -1.0e5, 2.0e5)), ("C3p1", (1.0e5, 0, 0)),
                                    ("C2p2", (-2.0e5, 1.5e5, 0)), ("R1p2", (0, 0, 4.0e5))])
def test_library_bloch_kernel(key, k0):
    _lib_vs_oracle(key, k0)
