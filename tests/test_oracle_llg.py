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
