"""Oracle pins: BAIM grid, stencils, FFT convolution, precorrection (K4-K9)."""
import itertools

import numpy as np
import pytest

from oracle import aim
from oracle.pgf import PgfSpec, pgf, pgf_self


def _grid(n, periodic, lattice, xyz):
    return aim.Grid(n, periodic, lattice, xyz)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_lagrange_moments(p):
    rng = np.random.default_rng(p)
    t = rng.uniform(5, 6, 50)
    s = (np.floor(t) - (p - 1) // 2) if p % 2 else (np.floor(t + 0.5) - p // 2)
    w = aim.lagrange_weights(t, s, p)
    nodes = s[:, None] + np.arange(p + 1)[None, :]
    for e in range(p + 1):                       # moments reproduced to order p (AIM)
        assert np.allclose(np.sum(w * nodes ** e, axis=1), t ** e, rtol=1e-12)
    # node on a grid point -> delta
    wi = aim.lagrange_weights(np.array([7.0]), np.array([7.0 - (p - 1) // 2 if p % 2 else 7.0 - p // 2]), p)
    assert np.sum(wi == 1.0) == 1 and np.sum(wi == 0.0) == p


def test_periodic_wrap_example():
    # S:265 [DERIVED]: node at x = L - Delta/2 on a periodic axis wraps to index 0 with weight 1/2
    L, N = 1.0, 8
    xyz = np.array([[L - L / N / 2, 0.25, 0.5]])
    g = _grid((N, N, N), (1, 1, 1), (L, L, L), xyz)
    S, W = aim.stencils(g, xyz, 1)
    P = aim.projection_matrix(g, S, W).toarray()[:, 0].reshape(N, N, N)
    assert P[N - 1].sum() == pytest.approx(0.5) and P[0].sum() == pytest.approx(0.5)


def test_grid_rules():
    xyz = np.array([[0.0, 0.0, 0.1], [0.5, 0.3, 1.1]])
    g = _grid((16, 4, 17), (1, 0, 0), (1.0, 0, 0), xyz)
    assert g.delta[0] == 1 / 16                    # periodic: L / N
    assert g.delta[2] == pytest.approx(1 / 16)     # non-periodic: D / (N-1)  (Eq. grid)
    assert g.origin[2] == 0.1
    assert list(g.fft) == [16, 8, 34]              # K6


def _direct_conv(grid, K, Q):
    n = grid.n
    U = np.zeros(tuple(n))
    for i in itertools.product(*[range(v) for v in n]):
        acc = 0.0
        for j in itertools.product(*[range(v) for v in n]):
            idx = []
            for a in range(3):
                d = i[a] - j[a]
                idx.append(d % n[a] if grid.periodic[a] else d % (2 * n[a]))
            acc += K[tuple(idx)] * Q[j]
        U[i] = acc
    return U


def test_fft_convolution_vs_direct_sum():
    # O(G^2) direct circular (periodic axes) / linear (non-periodic axes) sum
    rng = np.random.default_rng(0)
    xyz = np.array([[0, 0, 0], [1.0, 1.0, 1.0]])
    g = _grid((5, 4, 3), (1, 0, 1), (1.0, 0, 0.7), xyz)
    spec = PgfSpec((1, 0, 1), (1.0, 0, 0.7))
    K = aim.kernel_table(g, spec)
    Gh = aim.kernel_spectrum(K)
    assert np.allclose(np.imag(np.fft.fftn(K)), 0, atol=1e-12 * np.abs(K).max())   # K even -> real
    Q = rng.normal(size=(5, 4, 3)); Q -= Q.mean()   # sum Q = 0 (G_hat[0] := 0 is then exact)
    U = aim.convolve(g, Gh, Q)
    assert np.allclose(U, _direct_conv(g, K, Q), rtol=1e-12, atol=1e-12 * np.abs(U).max())
    # delta response: Q = d_a - d_b gives K(. - a) - K(. - b)
    Q2 = np.zeros((5, 4, 3)); Q2[1, 2, 0] = 1; Q2[3, 0, 2] = -1
    assert np.allclose(aim.convolve(g, Gh, Q2), _direct_conv(g, K, Q2), atol=1e-12)


def test_kernel_table_samples():
    xyz = np.array([[0, 0, 0], [1.0, 1.0, 1.0]])
    g = _grid((4, 4, 4), (1, 1, 0), (1.0, 1.0, 0), xyz)
    spec = PgfSpec((1, 1, 0), (1.0, 1.0, 0))
    K = aim.kernel_table(g, spec)
    assert K[0, 0, 0] == pytest.approx(pgf_self(spec))
    assert K[1, 3, 6] == pytest.approx(pgf(np.array([[0.25, 0.75, -2 / 3]]), spec)[0])
    assert np.all(K[:, :, 4] == 0)                 # j = N on the padded axis


def _pair_setup(xyz, n=(16, 16, 16), s=2.0, p=1, L=1.0):
    g = _grid(n, (1, 1, 1), (L, L, L), xyz)
    spec = PgfSpec((1, 1, 1), (L, L, L))
    S, W = aim.stencils(g, xyz, p)
    C = aim.precorrection(g, xyz, (L, L, L), S, W, s, p)
    P = aim.projection_matrix(g, S, W)
    Gh = aim.kernel_spectrum(aim.kernel_table(g, spec))
    return g, spec, S, W, C, P, Gh


def test_precorrection_pair_exact_and_symmetric():
    # grid-mediated + C_box for a pair inside r_ER reproduces G_p(r_n - r_k) (the near part is
    # replaced by the direct G0); C_box is symmetric; boundary image pair present
    xyz = np.array([[0.51, 0.49, 0.52], [0.57, 0.45, 0.55], [0.995, 0.3, 0.3], [0.01, 0.31, 0.29],
                    [0.2, 0.8, 0.1]])
    g, spec, S, W, C, P, Gh = _pair_setup(xyz)
    Cd = C.toarray()
    assert np.allclose(Cd, Cd.T, rtol=1e-12, atol=1e-12 * np.abs(Cd).max())
    assert Cd[2, 3] != 0.0                         # pair across the periodic face
    assert Cd[4, 0] == 0.0 and Cd[4, 1] == 0.0     # far pairs: no entry
    for (n, k) in ((0, 1), (2, 3)):
        q = np.zeros(5); q[k] = 1.0; q[4] = -1.0    # neutral; node 4 is far from n
        Q = (P @ q).reshape(16, 16, 16)
        u = P.T @ aim.convolve(g, Gh, Q).ravel() + C @ q
        ref = pgf((xyz[n] - xyz[k])[None], spec)[0] - pgf((xyz[n] - xyz[4])[None], spec)[0]
        assert u[n] == pytest.approx(ref, rel=1e-3)


def test_rer_validity():
    xyz = np.array([[0.1, 0.1, 0.1]])
    g = _grid((8, 8, 8), (1, 1, 1), (1.0, 1.0, 1.0), xyz)
    with pytest.raises(ValueError):
        aim.check_rer(g, (1.0, 1.0, 1.0), 3.0, 1)   # s + p + 1 = 5 >= N/2 = 4
    g2 = _grid((8, 8, 32), (1, 1, 1), (1.0, 1.0, 1.0), xyz)
    with pytest.raises(ValueError):
        aim.check_rer(g2, (1.0, 1.0, 1.0), 2.0, 1)  # r_ER = 2 max(Delta) spans 16 z-planes
