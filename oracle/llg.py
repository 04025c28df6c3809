"""Oracle LLG time integration (NEXT-2 of SURVEY.md 8(f)).  TEST INFRASTRUCTURE ONLY.

P:67-71 / P:101-105 (Eq. llg, discrete form; reading R18: the bare M in "M x M_n x H" is M_n):
    dM_n/dt = -gamma/(1+alpha^2) [ M_n x H_eff,n + (alpha/Ms) M_n x (M_n x H_eff,n) ]
i.e. for the unit vector m = M/Ms:
    dm/dt = -gamma/(1+alpha^2) [ m x H + alpha m x (m x H) ]
H_eff = H_ms + H_ex + H_an + H_ap (uniform applied field, uniaxial / cubic anisotropy).
Integrators: classical RK4 with |m| = 1 renormalisation after every step (SURVEY.md CS5,
config C5: "1000 RK steps"), and the paper's adaptive second-order Adams predictor-corrector
(AB2 predictor, AM2 corrector, Milne error estimate).
"""
import numpy as np

GAMMA = 1.7595e7        # gyromagnetic ratio, rad / (s Oe)


def llg_rhs(m, H, alpha, gamma=GAMMA):
    """dm/dt of the Landau-Lifshitz-Gilbert equation (Eq. llg)."""
    mxh = np.cross(m, H)
    return -gamma / (1.0 + alpha * alpha) * (mxh + alpha * np.cross(m, mxh))


def rk4_step(heff, m, dt, alpha, H_ap=(0.0, 0.0, 0.0), gamma=GAMMA, anis=None):
    """One classical RK4 step of the LLG equation followed by renormalisation.
    heff: callable m -> H_eff [N,3] (Oe), without the applied and anisotropy fields;
    anis = (kind, K, Ms, axis) or None."""
    Hap = np.asarray(H_ap, dtype=np.float64)[None, :]

    def f(x):
        H = heff(x) + Hap
        if anis is not None:
            H = H + anisotropy_field(x, *anis)
        return llg_rhs(x, H, alpha, gamma)
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


# ---------------------------------------------------------------- anisotropy (NEXT-2)
def anisotropy_field(m, kind, K, Ms, axis=(0.0, 0.0, 1.0)):
    """H_an (P:73 Eq. heff; local, "straightforward"), Oe, from the energy densities
    uniaxial  w = -K (m.u)^2            -> H = (2K/Ms) (m.u) u
    cubic     w = K (mx^2 my^2 + my^2 mz^2 + mz^2 mx^2)   (axes x, y, z)
              -> H = -(2K/Ms) (mx (my^2 + mz^2), my (mz^2 + mx^2), mz (mx^2 + my^2)),
    H = -(1/Ms) dw/dm.  kind 0: none."""
    m = np.asarray(m, dtype=np.float64)
    if kind == 0:
        return np.zeros_like(m)
    if kind == 1:
        u = np.asarray(axis, dtype=np.float64)
        u = u / np.linalg.norm(u)
        return (2.0 * K / Ms) * (m @ u)[:, None] * u[None, :]
    if kind == 2:
        mx, my, mz = m[:, 0], m[:, 1], m[:, 2]
        return -(2.0 * K / Ms) * np.stack([mx * (my ** 2 + mz ** 2), my * (mz ** 2 + mx ** 2),
                                          mz * (mx ** 2 + my ** 2)], axis=1)
    raise ValueError(kind)


def anisotropy_energy(m, kind, K, axis=(0.0, 0.0, 1.0)):
    """Energy density per node (erg/cm^3) of anisotropy_field's two forms."""
    if kind == 1:
        u = np.asarray(axis, dtype=np.float64)
        u = u / np.linalg.norm(u)
        return -K * (m @ u) ** 2
    mx, my, mz = m[:, 0], m[:, 1], m[:, 2]
    return K * (mx ** 2 * my ** 2 + my ** 2 * mz ** 2 + mz ** 2 * mx ** 2)


# ---------------------------------------------------------------- AM2 predictor-corrector (NEXT-2)
def am2_step(f, m, fn, fprev, dt, r):
    """One PECE step of the second-order Adams pair ("predictor-corrector schemes based on
    explicit second order Adams-Moulton (midpoint) approach"):
      P:  m_p = m_n + dt [(1 + r/2) f_n - (r/2) f_{n-1}]    (variable-step AB2, r = dt / dt_prev;
                                                             forward Euler when f_{n-1} is None)
      E:  f_p = f(m_p)
      C:  m_c = m_n + (dt/2) (f_n + f_p)                     (AM2 = trapezoidal rule)
      m_{n+1} = m_c / |m_c|;  E: f_{n+1} = f(m_{n+1}) (by the caller)
    Local error estimate (Milne's device for the AB2/AM2 pair, error constants 5/12 and -1/12):
      err = max_n |m_c - m_p| / 6."""
    if fprev is None:
        mp = m + dt * fn
    else:
        mp = m + dt * ((1.0 + 0.5 * r) * fn - 0.5 * r * fprev)
    fp = f(mp)
    mc = m + 0.5 * dt * (fn + fp)
    err = float(np.max(np.linalg.norm(mc - mp, axis=1))) / 6.0
    return mc / np.linalg.norm(mc, axis=1, keepdims=True), err


def am2_integrate(heff, m, t_end, dt0, tol, alpha, H_ap=(0.0, 0.0, 0.0), gamma=GAMMA, anis=None,
                  dt_max=None):
    """Adaptive AM2 integration to t_end.  A step is accepted when err <= tol; the next step is
    dt * min(2, max(0.2, 0.9 (tol/err)^(1/3))) (third-order local error of the corrector), a
    rejected step retries with the shrunk dt.  anis = (kind, K, Ms, axis) or None.
    Returns (m, accepted steps, rejected steps)."""
    Hap = np.asarray(H_ap, dtype=np.float64)[None, :]

    def f(x):
        H = heff(x) + Hap
        if anis is not None:
            H = H + anisotropy_field(x, *anis)
        return llg_rhs(x, H, alpha, gamma)

    t, dt, dt_prev = 0.0, dt0, None
    fn, fprev = f(m), None
    acc = rej = 0
    while t < t_end * (1 - 1e-12):
        dt = min(dt, t_end - t)
        if dt_max is not None:
            dt = min(dt, dt_max)
        r = dt / dt_prev if dt_prev else 0.0
        mn, err = am2_step(f, m, fn, fprev, dt, r)
        fac = 2.0 if err == 0 else min(2.0, max(0.2, 0.9 * (tol / err) ** (1.0 / 3.0)))
        if err <= tol:
            t += dt
            m, fprev, fn, dt_prev = mn, fn, f(mn), dt
            acc += 1
        else:
            rej += 1
        dt *= fac
    return m, acc, rej


def kalinikos_omega(k, d, theta, Ms, Aex, gamma=GAMMA, H0=0.0, exact_P=True):
    """Lowest (uniform-thickness) spin-wave mode of a film of thickness d in the dipole-exchange
    theory of Kalinikos and Slavin, the paper's Eq. sw_disp (written there for H0 = 0
    with the small-kd form P = kd/2):
        omega^2 = (w_H + w_M l^2 k^2) (w_H + w_M l^2 k^2 + w_M F),
        F = 1 - P cos^2(theta) + w_M P (1 - P) sin^2(theta) / (w_H + w_M l^2 k^2),
        P = 1 - (1 - exp(-k d)) / (k d),   w_M = gamma 4 pi Ms,  w_H = gamma H0,
    l^2 = gamma_ex = Aex / (2 pi Ms^2) (CGS), theta = angle between k and M.  Returns rad/s."""
    wM = gamma * 4 * np.pi * Ms
    wH = gamma * H0
    l2 = Aex / (2 * np.pi * Ms ** 2)
    P = 1.0 - (1.0 - np.exp(-k * d)) / (k * d) if exact_P else 0.5 * k * d
    a = wH + wM * l2 * k * k
    F = 1.0 - P * np.cos(theta) ** 2 + wM * P * (1.0 - P) * np.sin(theta) ** 2 / a
    return np.sqrt(a * (a + wM * F))
