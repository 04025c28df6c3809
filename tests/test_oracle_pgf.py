"""Oracle pins: periodic Green's functions (Eq. 2).

Closed forms (not the Ewald formula retyped): the simple-cubic and NaCl Madelung
constants, 4 zeta(1/2) beta(1/2) for the square lattice, the digamma on-axis form and
Schlomilch K0 series of the 1D sum, renormalised / spherical-order direct sums.
"""
import math

import numpy as np
import pytest
from scipy import special

from oracle import pgf as P

# Dirichlet beta(1/2) and zeta(1/2) (closed-form constants, independent of Ewald)
ZETA_HALF = -1.4603545088095868
BETA_HALF = 0.6676914571896091


def test_3d_simple_cubic_self():
    # regularised self value of the tinfoil SC lattice sum: -2.8372974795 / L
    for L in (1.0, 3e-5):
        s = P.PgfSpec((1, 1, 1), (L, L, L))
        assert P.pgf_self(s) * L == pytest.approx(-2.8372974794806, rel=1e-12)


def test_3d_nacl_madelung():
    # NaCl: cell L = 2 with +-1 charges on the 8 sites of a unit-spaced cubic sublattice;
    # potential at a + site (excluding itself) = -1.747564594633 (Madelung constant)
    s = P.PgfSpec((1, 1, 1), (2.0, 2.0, 2.0))
    sites = np.array([[i, j, k] for i in (0, 1) for j in (0, 1) for k in (0, 1)], float)
    q = np.array([(-1) ** int(a.sum()) for a in sites])
    pot = P.pgf_self(s) * q[0] + sum(q[i] * P.pgf(sites[i][None] - sites[0][None], s)[0] for i in range(1, 8))
    assert pot == pytest.approx(-1.747564594633, rel=1e-11)


def test_2d_square_self():
    # 2D square lattice: G2_reg(0) = 4 zeta(1/2) beta(1/2) / L
    s = P.PgfSpec((1, 1, 0), (1.0, 1.0, 0))
    assert P.pgf_self(s) == pytest.approx(4 * ZETA_HALF * BETA_HALF, rel=1e-11)


def test_2d_far_field_normalisation():
    # DESIGN R3: G2 + 2 pi |z| / A -> 0 exponentially as |z| -> inf
    s = P.PgfSpec((1, 1, 0), (1.0, 1.0, 0))
    r = np.array([[0.3, 0.1, z] for z in (2.0, 3.0, 5.0, -5.0)])
    v = P.pgf(r, s) + 2 * np.pi * np.abs(r[:, 2])
    assert abs(v[0]) < 1e-5 and abs(v[1]) < 1e-7 and abs(v[2]) < 1e-12 and abs(v[3]) < 1e-12


def test_1d_closed_forms():
    s = P.PgfSpec((1, 0, 0), (1.0, 0, 0))
    assert abs(P.pgf_self(s)) < 1e-13                  # renormalisation R3: G1_reg(0) = 0
    for x in (0.25, 0.5, 0.8):
        digamma = (-2 * P.EULER_GAMMA - special.digamma(x) - special.digamma(1 - x))
        assert P.pgf(np.array([[x, 0, 0]]), s)[0] == pytest.approx(digamma, rel=1e-12)
    assert P.pgf(np.array([[0.5, 0, 0]]), s)[0] == pytest.approx(4 * math.log(2), rel=1e-12)
    for (x, rho) in ((0.3, 0.2), (0.1, 0.7), (0.5, 1.5)):
        k0 = P.schlomilch_1d(x, rho, 1.0)
        assert P.pgf(np.array([[x, rho * 0.6, rho * 0.8]]), s)[0] == pytest.approx(k0, rel=1e-11)
    # renormalised direct sum (slowly convergent; truncation error ~rho^2 / n^2)
    d = P.direct_sum_1d(np.array([[0.5, 0.3, 0.0]]), 1.0, 200000)[0]
    assert P.pgf(np.array([[0.5, 0.3, 0.0]]), s)[0] == pytest.approx(d, rel=1e-9)
    # non-unit period and another periodic axis (the rod of P:277 is periodic along z)
    s2 = P.PgfSpec((0, 0, 1), (0, 0, 2.0))
    assert P.pgf(np.array([[0.0, 0.0, 0.5]]), s2)[0] == pytest.approx(
        (-2 * P.EULER_GAMMA - special.digamma(0.25) - special.digamma(0.75)) / 2.0, rel=1e-12)


def test_3d_spherical_order_direct_sum():
    # spherical-order direct pair sum = G3(r1) - G3(r2) - (2 pi/3V)(|r1|^2 - |r2|^2) (tinfoil vs
    # vacuum boundary); fixes the sign/normalisation of the 3D sum
    s = P.PgfSpec((1, 1, 1), (1.0, 1.0, 1.0))
    r1 = np.array([0.1, 0.2, 0.3]); r2 = np.array([-0.2, 0.05, 0.15])
    d = P.direct_sum_3d_spherical_pair(r1, r2, 1.0, 14)
    g = P.pgf(r1[None], s)[0] - P.pgf(r2[None], s)[0] - (2 * np.pi / 3) * (r1 @ r1 - r2 @ r2)
    assert d == pytest.approx(g, abs=2e-4)           # truncation of the radius-14 sum


@pytest.mark.parametrize("per", [(1, 1, 1), (1, 1, 0), (1, 0, 0), (0, 1, 1)])
def test_alpha_independence_periodicity_parity(per):
    lat = tuple(1.3 if per[a] else 0.0 for a in range(3))
    lat = tuple(v * (1 + 0.2 * a) for a, v in enumerate(lat))
    s1 = P.PgfSpec(per, lat)
    s2 = P.PgfSpec(per, lat, alpha=2.0 * s1.alpha)
    rng = np.random.default_rng(0)
    r = rng.uniform(-0.6, 0.6, size=(20, 3))
    g1 = P.pgf(r, s1)
    assert np.allclose(P.pgf(r, s2), g1, rtol=1e-12, atol=1e-12)
    assert np.allclose(P.pgf(-r, s1), g1, rtol=1e-12, atol=1e-12)
    for a in range(3):
        if per[a]:
            sh = np.zeros(3); sh[a] = lat[a]
            assert np.allclose(P.pgf(r + sh, s1), g1, rtol=1e-12, atol=1e-12)
    assert P.pgf_self(s2) == pytest.approx(P.pgf_self(s1), rel=1e-12, abs=1e-12)


def test_self_limit():
    # G_reg(0) = lim_{r->0} G(r) - 1/r
    for per in [(1, 1, 1), (1, 1, 0), (1, 0, 0)]:
        s = P.PgfSpec(per, (1.0, 1.0, 1.0))
        eps = 1e-4
        r = np.array([[eps, 0.0, 0.0]])
        assert P.pgf(r, s)[0] - 1 / eps == pytest.approx(P.pgf_self(s), abs=1e-6)


def test_structure_factor_potential_matches_pairwise():
    s = P.PgfSpec((1, 1, 1), (1.0, 1.1, 0.9))
    rng = np.random.default_rng(2)
    t = rng.random((6, 3)); src = rng.random((9, 3)); src[4] = t[1]
    q = rng.normal(size=9)
    a = P.pgf_potential(t, src, q, s)
    b = np.array([sum(q[k] * P.pgf((t[n] - src[k])[None], s)[0] for k in range(9)
                      if np.any(t[n] != src[k])) for n in range(6)])
    assert np.allclose(a, b, rtol=1e-12, atol=1e-12)
