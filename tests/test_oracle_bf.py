"""Oracle pins: the C brute-force pair sums (oracle/bf.c, O12) used by the AIM-vs-brute-force
checks.  Pinned (a) against closed forms directly -- the simple-cubic and NaCl Madelung
constants, the square-lattice 4 zeta(1/2) beta(1/2), the 1D digamma on-axis form and the
Schlomilch K0 series -- and (b) against the NumPy oracle
(oracle/pgf.py, itself pinned in test_oracle_pgf.py) on random points and random charge sets,
including the 3D structure-factor reordering of the reciprocal sum."""
import math

import numpy as np
import pytest
from scipy import special

from oracle import bf, pgf as P

ZETA_HALF = -1.4603545088095868
BETA_HALF = 0.6676914571896091


def test_bf_closed_forms():
    L = 1.0
    s3 = P.PgfSpec((1, 1, 1), (L, L, L))
    assert bf.pgf_self(s3) == pytest.approx(-2.8372974794806, rel=1e-12)
    s2 = P.PgfSpec((1, 1, 0), (L, L, 0))
    assert bf.pgf_self(s2) == pytest.approx(4 * ZETA_HALF * BETA_HALF, rel=1e-11)
    s1 = P.PgfSpec((1, 0, 0), (L, 0, 0))
    assert abs(bf.pgf_self(s1)) < 1e-13
    x = np.array([0.25, 0.5, 0.8])
    dig = -2 * P.EULER_GAMMA - special.digamma(x) - special.digamma(1 - x)
    assert np.allclose(bf.pgf(np.stack([x, 0 * x, 0 * x], 1), s1), dig, rtol=1e-12)
    for (xx, rho) in ((0.3, 0.2), (0.1, 0.7)):
        v = bf.pgf(np.array([[xx, rho * 0.6, rho * 0.8]]), s1)[0]
        assert v == pytest.approx(P.schlomilch_1d(xx, rho, 1.0), rel=1e-11)


def test_bf_nacl_potential():
    # NaCl through the pair sum: potential at a + site of the 8-site cell (L = 2) = Madelung
    s = P.PgfSpec((1, 1, 1), (2.0, 2.0, 2.0))
    sites = np.array([[i, j, k] for i in (0, 1) for j in (0, 1) for k in (0, 1)], float)
    q = np.array([(-1.0) ** int(a.sum()) for a in sites])
    u = bf.potential(sites[:1], sites, q, s)[0] + bf.pgf_self(s) * q[0]
    assert u == pytest.approx(-1.747564594633, rel=1e-11)


@pytest.mark.parametrize("per,lat", [((1, 0, 0), (1.0, 0, 0)), ((0, 1, 0), (0, 0.7, 0)), ((0, 0, 1), (0, 0, 1.3)),
                                     ((1, 1, 0), (1.0, 1.3, 0)), ((1, 0, 1), (0.8, 0, 1.1)),
                                     ((1, 1, 1), (1.0, 1.2, 0.9))])
def test_bf_matches_numpy_oracle(per, lat):
    s = P.PgfSpec(per, lat)
    rng = np.random.default_rng(3)
    r = rng.uniform(-1.5, 1.5, (100, 3))
    assert np.allclose(bf.pgf(r, s), P.pgf(r, s), rtol=1e-12, atol=1e-12)
    assert bf.pgf_self(s) == pytest.approx(P.pgf_self(s), rel=1e-12, abs=1e-13)
    src = rng.uniform(0, 1, (150, 3))
    q = rng.normal(size=150)
    tgt = np.concatenate([src[:20], rng.uniform(0, 1, (5, 3))])     # with and without t == s
    u1 = P.pgf_potential(tgt, src, q, s)
    u2 = bf.potential(tgt, src, q, s)
    assert np.max(np.abs(u1 - u2)) <= 1e-12 * np.max(np.abs(u1))


def test_bf_alpha_independence():
    # the Ewald splitting parameter must not change the sum (exponential convergence)
    r = np.random.default_rng(5).uniform(-1, 1, (30, 3))
    for per, lat in (((1, 0, 0), (1.0, 0, 0)), ((1, 1, 0), (1.0, 1.0, 0)), ((1, 1, 1), (1.0, 1.0, 1.0))):
        a = bf.pgf(r, P.PgfSpec(per, lat, alpha=math.sqrt(math.pi)))
        b = bf.pgf(r, P.PgfSpec(per, lat, alpha=2 * math.sqrt(math.pi)))
        assert np.allclose(a, b, rtol=1e-11, atol=1e-11)
