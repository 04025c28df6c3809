"""Oracle pins for the LLG integrator (NEXT-2): macrospin closed form,
precession without damping conserves m.H, RK4 4th-order convergence."""
import numpy as np
import pytest

from oracle import llg


def _run(m0, dt, nsteps, alpha, H0):
    m = m0.copy()
    zero = lambda x: np.zeros_like(x)   # noqa: E731
    for _ in range(nsteps):
        m = llg.rk4_step(zero, m, dt, alpha, (0, 0, H0))
    return m


def test_macrospin_closed_form():
    H0, alpha = 1000.0, 0.1
    period = 2 * np.pi * (1 + alpha ** 2) / (llg.GAMMA * H0)
    theta0, phi0 = 1.0, 0.3
    m0 = llg.macrospin(theta0, phi0, 0.0, H0, alpha)[None, :]
    n = 2000
    dt = 10 * period / n
    m = _run(m0, dt, n, alpha, H0)
    ref = llg.macrospin(theta0, phi0, 10 * period, H0, alpha)
    assert np.abs(m[0] - ref).max() < 1e-6


def test_undamped_precession_conserves_energy():
    H0 = 500.0
    m0 = np.array([[np.sin(0.7), 0.0, np.cos(0.7)]])
    m = _run(m0, 1e-13, 500, 0.0, H0)
    assert m[0, 2] == pytest.approx(np.cos(0.7), abs=1e-10)
    assert np.linalg.norm(m[0]) == pytest.approx(1.0, abs=1e-14)


def test_rk4_fourth_order():
    H0, alpha = 800.0, 0.2
    period = 2 * np.pi * (1 + alpha ** 2) / (llg.GAMMA * H0)
    m0 = llg.macrospin(1.2, 0.0, 0.0, H0, alpha)[None, :]
    T = 2 * period
    ref = llg.macrospin(1.2, 0.0, T, H0, alpha)
    errs = [np.abs(_run(m0, T / n, n, alpha, H0)[0] - ref).max() for n in (50, 100)]
    assert np.log2(errs[0] / errs[1]) > 3.7


# ---- NEXT-2: anisotropy field and the AM2 predictor-corrector
def test_anisotropy_field_is_energy_gradient():
    # H_an = -(1/Ms) dw/dm, checked by central differences of the energy density (any m, not unit)
    rng = np.random.default_rng(3)
    m = rng.normal(size=(5, 3))
    Ms, K = 800.0, 5e5
    for kind, axis in ((1, (0.3, -0.2, 0.9)), (2, (0, 0, 1))):
        H = llg.anisotropy_field(m, kind, K, Ms, axis)
        g = np.zeros_like(m)
        for c in range(3):
            e = np.zeros(3)
            e[c] = 1e-6
            g[:, c] = (llg.anisotropy_energy(m + e, kind, K, axis) - llg.anisotropy_energy(m - e, kind, K, axis)) / 2e-6
        assert np.allclose(H, -g / Ms, rtol=1e-7, atol=1e-6)


def test_uniaxial_macrospin_precession():
    # alpha = 0, uniaxial axis z: H_an = H_K m_z z (H_K = 2K/Ms), m precesses about z at the
    # constant rate gamma H_K cos(theta0) (closed form)
    Ms, K = 800.0, 4e5
    HK = 2 * K / Ms
    th0 = 0.5
    m0 = np.array([[np.sin(th0), 0.0, np.cos(th0)]])
    w = llg.GAMMA * HK * np.cos(th0)
    T = 2 * np.pi / w
    n = 1000
    m = m0.copy()
    zero = lambda x: np.zeros_like(x)   # noqa: E731
    for _ in range(n):
        m = llg.rk4_step(zero, m, T / n, 0.0, anis=(1, K, Ms, (0, 0, 1)))
    assert np.abs(m[0] - m0[0]).max() < 1e-8           # one full period
    m = m0.copy()
    for _ in range(n // 4):
        m = llg.rk4_step(zero, m, T / n, 0.0, anis=(1, K, Ms, (0, 0, 1)))
    ref = np.array([np.sin(th0) * np.cos(np.pi / 2), np.sin(th0) * np.sin(np.pi / 2), np.cos(th0)])
    assert np.abs(m[0] - ref).max() < 1e-8             # quarter period (sense of -m x H)


def test_cubic_anisotropy_conserves_energy_undamped():
    Ms, K = 800.0, -3e5
    m = np.array([[0.3, 0.5, 0.8]])
    m = m / np.linalg.norm(m)
    e0 = llg.anisotropy_energy(m, 2, K)[0]
    zero = lambda x: np.zeros_like(x)   # noqa: E731
    for _ in range(400):
        m = llg.rk4_step(zero, m, 2e-13, 0.0, anis=(2, K, Ms, (0, 0, 1)))
    assert llg.anisotropy_energy(m, 2, K)[0] == pytest.approx(e0, rel=1e-9)


def test_am2_second_order_and_adaptive():
    H0, alpha = 800.0, 0.1
    period = 2 * np.pi * (1 + alpha ** 2) / (llg.GAMMA * H0)
    m0 = llg.macrospin(1.0, 0.0, 0.0, H0, alpha)[None, :]
    T = period
    ref = llg.macrospin(1.0, 0.0, T, H0, alpha)
    zero = lambda x: np.zeros_like(x)   # noqa: E731
    errs = []
    for n in (200, 400):
        m, acc, rej = llg.am2_integrate(zero, m0, T, T / n, np.inf, alpha, (0, 0, H0), dt_max=T / n)
        assert acc == n and rej == 0
        errs.append(np.abs(m[0] - ref).max())
    assert 1.8 < np.log2(errs[0] / errs[1]) < 2.3      # second order
    m, acc, rej = llg.am2_integrate(zero, m0, T, T / 1000, 1e-7, alpha, (0, 0, H0))
    assert np.abs(m[0] - ref).max() < 1e-4 and acc > 10


def test_kalinikos_limits():
    # closed-form limits of Eq. sw_disp: k -> 0 along M (theta = 0) with H0 gives the
    # in-plane Kittel film mode sqrt(H0 (H0 + 4 pi Ms)) gamma; theta = 90 deg, no exchange, gives the
    # Damon-Eshbach small-kd limit; the paper's P = kd/2 is the exact P to first order in kd
    Ms, A, H0 = 637.0, 1.4e-6, 300.0
    w = llg.kalinikos_omega(1e-3, 1e-6, 0.0, Ms, A, H0=H0)
    assert w == pytest.approx(llg.GAMMA * np.sqrt(H0 * (H0 + 4 * np.pi * Ms)), rel=1e-6)
    k, d = 1e3, 1e-6            # kd = 1e-3
    wM, wH = llg.GAMMA * 4 * np.pi * Ms, llg.GAMMA * H0
    de = np.sqrt(wH * (wH + wM) + wM ** 2 * (k * d / 2) * (1 - k * d / 2))
    assert llg.kalinikos_omega(k, d, np.pi / 2, Ms, 0.0, H0=H0) == pytest.approx(de, rel=1e-3)
    for kd in (0.01, 0.1):
        a = llg.kalinikos_omega(kd / 1e-6, 1e-6, 0.7, Ms, A, exact_P=True)
        b = llg.kalinikos_omega(kd / 1e-6, 1e-6, 0.7, Ms, A, exact_P=False)
        assert abs(a / b - 1) < kd / 4           # P = kd/2 - (kd)^2/6 + ...: O(kd) in omega
