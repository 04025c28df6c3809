"""Oracle Bloch-phase periodic Green's function (NEXT-4 of SURVEY.md 8(f)).  TEST INFRASTRUCTURE ONLY.

P:183-185 (Eq. 2): G_p(r) = sum_i exp(-j k0 . R_i) G_0(r - R_i), R_i the lattice vectors of the
periodic axes, G_0 = 1/|r| -- the static kernel of pgf.py is k0 = 0 (reading R4).  For
k0 off the reciprocal lattice every sum converges absolutely after the Ewald split and needs no
renormalisation.  Poisson summation of the smooth part (F = Fourier transform of erf(a r)/r)
gives, with q_G = G + k0 over the reciprocal lattice vectors G of the periodic axes:

  real (all dims): sum_i exp(-j k0.R_i) erfc(a |r - R_i|) / |r - R_i|
  3D: (4 pi / V) sum_G exp(-|q|^2 / 4a^2) / |q|^2 exp(-j q.r)
  2D: (1 / A) sum_G exp(-j q.rho) (pi/|q|) [e^{|q| z} erfc(|q|/2a + a z) + e^{-|q| z} erfc(|q|/2a - a z)]
  1D: (1 / L) sum_m exp(-j q_m x) I(q_m^2 / 4a^2, rho^2 q_m^2 / 4),  I(a, b) = int_a^inf e^{-u - b/u} du/u

(the static formulas of pgf.py with cos(k.r) -> exp(-j q.r) and the G = 0 term kept).  The
regularised self value is lim_{r->0} [G(r) - 1/r] (the i = 0 real term -> -2a/sqrt(pi)).
Pins (tests/test_oracle_bloch.py): the Bloch shift G(r + L_a e_a) = exp(-j k0_a L_a) G(r); alpha
independence; the 1D zone-boundary closed form (k0 = pi/L: sum_n (-1)^n / |x - nL| = [beta(x/L) -
beta(1 - x/L)] / L with beta(y) = (psi((y+1)/2) - psi(y/2)) / 2); and k0 -> 0: G minus its G = 0
term tends to the static kernel minus the static zero-mode term.
"""
import itertools
import math

import numpy as np
from scipy import special

from .pgf import PgfSpec, _ein, incomplete_bessel, EULER_GAMMA


class BlochSpec(PgfSpec):
    """PgfSpec plus the Bloch wave vector k0 (components along the periodic axes, rad/cm)."""

    def __init__(self, periodic, lattice, k0, alpha=None, tol=1e-15):
        super().__init__(periodic, lattice, alpha, tol)
        if self.dim == 0:
            raise ValueError("a Bloch phase needs a periodic axis")
        self.k0 = np.array([float(k0[a]) for a in self.axes])
        # reciprocal sums are centred on -k0 (q = G + k0 within the static cutoff + one shell)
        self.m_recip = [m + 1 + int(math.ceil(abs(k) * L / (2 * np.pi))) for m, k, L in
                        zip(self.m_recip, self.k0, self.L)]


def _split(r, spec):
    """components along the periodic axes (NOT wrapped: the phase depends on the image) and the
    free components"""
    rp = r[:, spec.axes]
    rf = r[:, spec.free] if spec.free else np.zeros((r.shape[0], 0))
    return rp, rf


def _real(rp, rf, spec, exclude_origin):
    a = spec.alpha
    out = np.zeros(rp.shape[0], complex)
    rf2 = np.sum(rf * rf, axis=1) if rf.shape[1] else np.zeros(rp.shape[0])
    # image range around each point: rp is not wrapped, so shift the window by round(rp / L)
    c = np.round(rp / spec.L[None, :]).astype(np.int64)
    ranges = [range(-n - 1, n + 2) for n in spec.n_real]
    for dn in itertools.product(*ranges):
        n = c + np.array(dn)[None, :]                      # image index per point
        R = n * spec.L[None, :]
        d2 = np.sum((rp - R) ** 2, axis=1) + rf2
        ph = np.exp(-1j * (n * spec.L[None, :]) @ spec.k0)
        with np.errstate(divide="ignore", invalid="ignore"):
            d = np.sqrt(d2)
            t = special.erfc(a * d) / d
        mask = d > 0
        if exclude_origin:
            mask &= np.any(n != 0, axis=1)
        out += np.where(mask, ph * np.where(d > 0, t, 0.0), 0.0)
    return out


def bloch_pgf(r, spec, self_term=False):
    """G(r; k0) for points r [P,3] (r not a lattice point unless self_term: then the regularised
    self value at r = 0)."""
    r = np.atleast_2d(np.asarray(r, dtype=np.float64))
    if self_term:
        r = np.zeros((1, 3))
    a = spec.alpha
    rp, rf = _split(r, spec)
    out = _real(rp, rf, spec, exclude_origin=self_term)
    if self_term:
        out += -2.0 * a / math.sqrt(math.pi)
    ms = [np.arange(-m, m + 1) for m in spec.m_recip]
    if spec.dim == 3:
        V = float(np.prod(spec.L))
        for g in itertools.product(*ms):
            q = 2 * np.pi * np.array(g) / spec.L + spec.k0
            q2 = float(q @ q)
            if q2 == 0.0:
                continue
            out += (4 * np.pi / V) * math.exp(-q2 / (4 * a * a)) / q2 * np.exp(-1j * (rp @ q))
    elif spec.dim == 2:
        A = float(np.prod(spec.L))
        z = rf[:, 0]
        for g in itertools.product(*ms):
            q = 2 * np.pi * np.array(g) / spec.L + spec.k0
            qn = float(np.linalg.norm(q))
            if qn == 0.0:
                continue
            br = np.zeros_like(z)
            for sgn in (1.0, -1.0):
                w = qn / (2 * a) + sgn * a * z
                pos = w >= 0
                t = np.empty_like(z)
                t[pos] = special.erfcx(w[pos]) * np.exp(-qn * qn / (4 * a * a) - a * a * z[pos] ** 2)
                t[~pos] = np.exp(sgn * qn * z[~pos]) * special.erfc(w[~pos])
                br += t
            out += (1.0 / A) * (np.pi / qn) * br * np.exp(-1j * (rp @ q))
    else:
        L = float(spec.L[0])
        rho2 = np.sum(rf * rf, axis=1)
        for m in ms[0]:
            q = 2 * np.pi * m / L + spec.k0[0]
            if q == 0.0:
                continue
            out += (1.0 / L) * np.exp(-1j * q * rp[:, 0]) * incomplete_bessel(q * q / (4 * a * a), rho2 * q * q / 4.0)
    return out


def zero_mode(r, spec):
    """The G = 0 term of the reciprocal sum (it carries the k0 -> 0 divergence)."""
    r = np.atleast_2d(np.asarray(r, dtype=np.float64))
    a = spec.alpha
    rp, rf = _split(r, spec)
    q = spec.k0
    qn = float(np.linalg.norm(q))
    ph = np.exp(-1j * (rp @ q))
    if spec.dim == 3:
        return (4 * np.pi / float(np.prod(spec.L))) * math.exp(-qn * qn / (4 * a * a)) / (qn * qn) * ph
    if spec.dim == 2:
        z = rf[:, 0]
        br = (np.exp(qn * z) * special.erfc(qn / (2 * a) + a * z) +
              np.exp(-qn * z) * special.erfc(qn / (2 * a) - a * z))
        return (1.0 / float(np.prod(spec.L))) * (np.pi / qn) * br * ph
    rho2 = np.sum(rf * rf, axis=1)
    return (1.0 / float(spec.L[0])) * ph * incomplete_bessel(qn * qn / (4 * a * a), rho2 * qn * qn / 4.0)


def static_zero_mode(r, spec):
    """The term the static kernel (pgf.py, normalisation R3) puts in place of the G = 0 term."""
    r = np.atleast_2d(np.asarray(r, dtype=np.float64))
    a = spec.alpha
    rp, rf = _split(r, spec)
    if spec.dim == 3:
        return np.full(r.shape[0], -math.pi / (a * a * float(np.prod(spec.L))))
    if spec.dim == 2:
        z = rf[:, 0]
        return -(2 * np.pi / float(np.prod(spec.L))) * (z * special.erf(a * z) + np.exp(-a * a * z * z) / (a * math.sqrt(math.pi)))
    rho2 = np.sum(rf * rf, axis=1)
    L = float(spec.L[0])
    return -(1.0 / L) * (_ein(a * a * rho2) - 2.0 * math.log(2 * a * L) + EULER_GAMMA)


def beta_dirichlet(y):
    """beta(y) = sum_{k>=0} (-1)^k / (y + k) = (psi((y+1)/2) - psi(y/2)) / 2."""
    return 0.5 * (special.digamma((y + 1) / 2.0) - special.digamma(y / 2.0))
