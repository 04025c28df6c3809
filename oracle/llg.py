"""Oracle LLG time integration (NEXT-2 of SURVEY.md 8(f)).  TEST INFRASTRUCTURE ONLY.

P:67-71 / P:101-105 (Eq. llg, discrete form; reading R18: the bare M in "M x M_n x H" is M_n):
    dM_n/dt = -gamma/(1+alpha^2) [ M_n x H_eff,n + (alpha/Ms) M_n x (M_n x H_eff,n) ]
i.e. for the unit vector m = M/Ms:
    dm/dt = -gamma/(1+alpha^2) [ m x H + alpha m x (m x H) ]
H_eff = H_ms + H_ex + H_ap (uniform applied field, anisotropy is not modelled here).
Integrator: classical RK4 with |m| = 1 renormalisation after every step (SURVEY.md CS5,
config C5: "1000 RK steps").
"""
import numpy as np

GAMMA = 1.7595e7        # gyromagnetic ratio, rad / (s Oe)


def llg_rhs(m, H, alpha, gamma=GAMMA):
    """dm/dt of the Landau-Lifshitz-Gilbert equation (Eq. llg)."""
    mxh = np.cross(m, H)
    return -gamma / (1.0 + alpha * alpha) * (mxh + alpha * np.cross(m, mxh))


def rk4_step(heff, m, dt, alpha, H_ap=(0.0, 0.0, 0.0), gamma=GAMMA):
    """One classical RK4 step of the LLG equation followed by renormalisation.
    heff: callable m -> H_eff [N,3] (Oe), without the applied field."""
    Hap = np.asarray(H_ap, dtype=np.float64)[None, :]
    f = lambda x: llg_rhs(x, heff(x) + Hap, alpha, gamma)   # noqa: E731
    k1 = f(m)
    k2 = f(m + 0.5 * dt * k1)
    k3 = f(m + 0.5 * dt * k2)
    k4 = f(m + dt * k3)
    mn = m + dt / 6.0 * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    return mn / np.linalg.norm(mn, axis=1, keepdims=True)


def macrospin(theta0, phi0, t, H0, alpha, gamma=GAMMA):
    """Closed form for a macrospin in a static field H0 along +z (pins rk4_step):
    tan(theta/2) = tan(theta0/2) exp(-alpha gamma H0 t / (1 + alpha^2)),
    phi = phi0 + gamma H0 t / (1 + alpha^2)   (precession sense of -m x H)."""
    g = gamma * H0 / (1.0 + alpha * alpha)
    theta = 2.0 * np.arctan(np.tan(theta0 / 2.0) * np.exp(-alpha * g * t))
    phi = phi0 + g * t
    return np.stack([np.sin(theta) * np.cos(phi), np.sin(theta) * np.sin(phi), np.cos(theta)], axis=-1)
