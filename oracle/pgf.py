"""Oracle periodic Green's functions (Eq. 2 with k0 = 0).  TEST INFRASTRUCTURE ONLY.

G_p(r) = sum over lattice images of G_0(r - R), G_0 = 1/|r|.  The static sums
diverge (1D/2D) or converge conditionally (3D); the normalisation is DESIGN.md R3:
  3D  zero cell mean ("tinfoil", k = 0 term dropped)
  2D  G + 2*pi*|z|/A -> 0 as |z| -> inf
  1D  renormalised sum_n [1/|r - nL x| - (1 - delta_n0)/|nL|]   (so G1_reg(0) = 0)
The "exponentially rapidly convergent sums" of P:20/P:188/P:214 are Ewald sums
(SURVEY.md App. B).  Direct (slowly convergent) sums are provided as independent
pins: ``direct_sum_1d``, ``direct_sum_3d_spherical``.

All functions are vectorised over points r [P,3] (cm); lattice periods in cm.
"""
import itertools
import math
import numpy as np
from scipy import special

EULER_GAMMA = 0.57721566490153286061


class PgfSpec:
    """Periodic axes + periods.  ``axes`` lists the periodic axes (len 1, 2 or 3; 0 = the
    non-periodic free-space kernel of NEXT-3)."""

    def __init__(self, periodic, lattice, alpha=None, tol=1e-15):
        self.axes = [a for a in range(3) if periodic[a]]
        self.free = [a for a in range(3) if not periodic[a]]
        self.dim = len(self.axes)
        if self.dim == 0:
            # non-periodic mode: the free-space kernel G0 = 1/|r|,
            # no images, regularised self value 0
            self.L = np.zeros(0)
            self.alpha = None
            self.n_real, self.m_recip = [], []
            return
        self.L = np.array([float(lattice[a]) for a in self.axes])
        self.alpha = alpha if alpha is not None else math.sqrt(math.pi) / self.L.min()
        # cutoffs: erfc(x) < tol for x > xr; exp(-k^2/4a^2) < tol for k > kr
        xr = 6.2
        self.n_real = [int(math.ceil(xr / (self.alpha * Li) + 1.0)) for Li in self.L]
        kmax = 2.0 * self.alpha * math.sqrt(-math.log(tol)) * 1.1
        self.m_recip = [int(math.ceil(kmax * Li / (2 * math.pi))) + 1 for Li in self.L]


def _wrap_half(x, L):
    """x mod L into [-L/2, L/2)."""
    return x - L * np.floor(x / L + 0.5)


def _real_space(rp, rf, spec, exclude_origin):
    """sum_n erfc(a|r+R_n|)/|r+R_n|; rp periodic comps [P,d], rf free comps [P,3-d]."""
    a = spec.alpha
    out = np.zeros(rp.shape[0])
    rf2 = np.sum(rf * rf, axis=1) if rf.shape[1] else np.zeros(rp.shape[0])
    ranges = [range(-n, n + 1) for n in spec.n_real]
    rc = 6.2 / a
    for n in itertools.product(*ranges):
        # rp is wrapped into [-L/2, L/2): |rp + nL| >= sum_a max(0, |n_a| - 1/2)^2 L_a^2
        lb = sum(max(0.0, abs(n[i]) - 0.5) ** 2 * spec.L[i] ** 2 for i in range(len(n)))
        if lb > rc * rc:
            continue
        R = np.array(n, dtype=np.float64) * spec.L
        d2 = np.sum((rp + R) ** 2, axis=1) + rf2
        if exclude_origin and not any(n):
            continue
        d = np.sqrt(d2)
        with np.errstate(divide='ignore', invalid='ignore'):
            t = special.erfc(a * d) / d
        out += np.where(d > 0, t, 0.0)
    return out


def _ein(x):
    """Ein(x) = sum_{k>=1} (-1)^{k+1} x^k / (k k!) = E1(x) + ln x + gamma (entire)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    small = x < 1.0
    xs = x[small]
    term = np.ones_like(xs)
    acc = np.zeros_like(xs)
    for k in range(1, 40):
        term = term * xs / k
        acc += ((-1) ** (k + 1)) * term / k
    out[small] = acc
    xl = x[~small]
    out[~small] = special.exp1(xl) + np.log(xl) + EULER_GAMMA
    return out


_GL_S, _GL_W = np.polynomial.legendre.leggauss(64)


def incomplete_bessel(a, b):
    """I(a, b) = int_a^inf exp(-u - b/u) du/u, a > 0, b >= 0 (vectorised over b).
    Substitution u = a e^s; Gauss-Legendre on s in [0, S] with a e^S = 60."""
    b = np.asarray(b, dtype=np.float64)
    S = max(math.log(60.0 / a), 0.5)
    s = 0.5 * S * (_GL_S + 1.0)
    w = 0.5 * S * _GL_W
    ue = a * np.exp(s)                       # [Q]
    f = np.exp(-ue[None, :] - b[:, None] / ue[None, :])
    return f @ w


def pgf(r, spec):
    """G_p(r) for r [P,3] not on a lattice point (Ewald)."""
    r = np.atleast_2d(np.asarray(r, dtype=np.float64))
    return _pgf(r, spec, self_term=False)


def pgf_self(spec):
    """G_p^reg(0) = lim_{r->0} [G_p(r) - 1/r]   (reading R7/R13)."""
    return float(_pgf(np.zeros((1, 3)), spec, self_term=True)[0])


def _pgf(r, spec, self_term):
    if spec.dim == 0:
        # free space: G0(r) = 1/|r|; lim_{r->0} [G0(r) - 1/r] = 0
        return np.zeros(r.shape[0]) if self_term else 1.0 / np.linalg.norm(r, axis=1)
    a = spec.alpha
    rp = np.stack([_wrap_half(r[:, ax], spec.L[i]) for i, ax in enumerate(spec.axes)], axis=1)
    rf = r[:, spec.free] if spec.free else np.zeros((r.shape[0], 0))
    out = _real_space(rp, rf, spec, exclude_origin=self_term)
    if self_term:
        out += -2.0 * a / math.sqrt(math.pi)
    if spec.dim == 3:
        V = float(np.prod(spec.L))
        ms = [np.arange(-m, m + 1) for m in spec.m_recip]
        # separable phases: e^{i k.r} = prod_axis e^{i k_a r_a}
        Ex = np.exp(1j * 2 * np.pi * np.outer(rp[:, 0], ms[0]) / spec.L[0])
        Ey = np.exp(1j * 2 * np.pi * np.outer(rp[:, 1], ms[1]) / spec.L[1])
        Ez = np.exp(1j * 2 * np.pi * np.outer(rp[:, 2], ms[2]) / spec.L[2])
        KX, KY, KZ = np.meshgrid(2 * np.pi * ms[0] / spec.L[0], 2 * np.pi * ms[1] / spec.L[1],
                                 2 * np.pi * ms[2] / spec.L[2], indexing="ij")
        k2 = KX ** 2 + KY ** 2 + KZ ** 2
        with np.errstate(divide='ignore', invalid='ignore'):
            coef = np.where(k2 > 0, np.exp(-k2 / (4 * a * a)) / k2, 0.0) * (4 * np.pi / V)
        t = np.einsum('pa,abc->pbc', Ex, coef)
        t = np.einsum('pb,pbc->pc', Ey, t)
        out += np.real(np.einsum('pc,pc->p', Ez, t))
        out += -np.pi / (a * a * V)
    elif spec.dim == 2:
        A = float(np.prod(spec.L))
        z = rf[:, 0]
        m0 = np.arange(-spec.m_recip[0], spec.m_recip[0] + 1)
        m1 = np.arange(-spec.m_recip[1], spec.m_recip[1] + 1)
        acc = np.zeros(r.shape[0])
        for i in m0:
            for j in m1:
                if i == 0 and j == 0:
                    continue
                kx = 2 * np.pi * i / spec.L[0]
                ky = 2 * np.pi * j / spec.L[1]
                k = math.hypot(kx, ky)
                br = _bracket_2d(k, z, a)
                acc += np.cos(kx * rp[:, 0] + ky * rp[:, 1]) / k * br
        out += (np.pi / A) * acc
        out += -(2 * np.pi / A) * (z * special.erf(a * z) + np.exp(-a * a * z * z) / (a * math.sqrt(math.pi)))
    else:
        L = float(spec.L[0])
        rho2 = np.sum(rf * rf, axis=1)
        x = rp[:, 0]
        acc = np.zeros(r.shape[0])
        for m in range(1, spec.m_recip[0] + 1):
            km = 2 * np.pi * m / L
            am = km * km / (4 * a * a)
            acc += np.cos(km * x) * incomplete_bessel(am, rho2 * km * km / 4.0)
        out += (2.0 / L) * acc
        out += -(1.0 / L) * (_ein(a * a * rho2) - 2.0 * math.log(2 * a * L) + EULER_GAMMA)
    return out


def _bracket_2d(k, z, a):
    """e^{kz} erfc(k/2a + a z) + e^{-kz} erfc(k/2a - a z), overflow-safe via erfcx."""
    out = np.zeros_like(z)
    for sgn in (1.0, -1.0):
        w = k / (2 * a) + sgn * a * z
        pos = w >= 0
        t = np.empty_like(z)
        t[pos] = special.erfcx(w[pos]) * np.exp(-k * k / (4 * a * a) - a * a * z[pos] ** 2)
        t[~pos] = np.exp(sgn * k * z[~pos]) * special.erfc(w[~pos])
        out += t
    return out


# ---------------------------------------------------------------- direct-sum pins

def direct_sum_1d(r, L, n_terms):
    """Renormalised direct sum (DESIGN R3): sum_{|n|<=n_terms} 1/|r - nL x| - (1-d_n0)/|nL|.
    Periodic along x.  Truncation error ~ O(rho^2 / (n_terms^2 L^3))."""
    r = np.atleast_2d(r)
    out = np.zeros(r.shape[0])
    n = np.arange(1, n_terms + 1, dtype=np.float64)
    for i in range(r.shape[0]):
        x, y, z = r[i]
        rho2 = y * y + z * z
        s = 1.0 / math.sqrt(x * x + rho2)
        s += np.sum(1.0 / np.sqrt((x - n * L) ** 2 + rho2) + 1.0 / np.sqrt((x + n * L) ** 2 + rho2)
                    - 2.0 / (n * L))
        out[i] = s
    return out


def schlomilch_1d(x, rho, L, n_terms=60):
    """Off-axis 1D PGF as a K0 series (pins Ewald 1D): -(2/L)[ln(rho/2L) + gamma]
    + (4/L) sum_{m>=1} K0(2 pi m rho / L) cos(2 pi m x / L)."""
    m = np.arange(1, n_terms + 1)
    s = np.sum(special.k0(2 * np.pi * m * rho / L) * np.cos(2 * np.pi * m * x / L))
    return -(2.0 / L) * (math.log(rho / (2 * L)) + EULER_GAMMA) + (4.0 / L) * s


def digamma_on_axis_1d(x, L):
    """On-axis 1D PGF closed form (-2 gamma - psi(x/L) - psi(1 - x/L)) / L, 0 < x < L."""
    return (-2 * EULER_GAMMA - special.digamma(x / L) - special.digamma(1 - x / L)) / L


def direct_sum_3d_spherical_pair(r1, r2, L, radius):
    """sum over images |n| <= radius (spherical order) of 1/|r1+nL| - 1/|r2+nL| (cubic cell).
    Under spherical summation order this equals G3(r1)-G3(r2) - (2 pi/3V)(|r1|^2-|r2|^2)
    for the tinfoil G3 (DESIGN R3): the pin that fixes the 3D normalisation."""
    R = int(math.ceil(radius))
    rng = np.arange(-R, R + 1)
    N = np.stack(np.meshgrid(rng, rng, rng, indexing="ij"), axis=-1).reshape(-1, 3).astype(np.float64)
    N = N[np.sum(N * N, axis=1) <= radius * radius]
    d1 = np.linalg.norm(r1[None, :] + N * L, axis=1)
    d2 = np.linalg.norm(r2[None, :] + N * L, axis=1)
    return float(np.sum(1.0 / d1 - 1.0 / d2))


def pgf_potential(targets, sources, q, spec, chunk=512):
    """sum_k q_k G_p(t_n - s_k) over all pairs with t_n != s_k (O12 building block).
    3D: real-space part pairwise + reciprocal part by structure factors
    S(k) = sum_k q_k exp(-i k.s_k) (the same Ewald sum, reordered); 1D/2D: pairwise."""
    targets = np.atleast_2d(targets); sources = np.atleast_2d(sources)
    nt = targets.shape[0]
    out = np.zeros(nt)
    if spec.dim != 3:
        for s0 in range(0, nt, chunk):
            t = targets[s0:s0 + chunk]
            d = (t[:, None, :] - sources[None, :, :]).reshape(-1, 3)
            nz = np.any(d != 0.0, axis=1)
            g = np.zeros(d.shape[0])
            g[nz] = pgf(d[nz], spec)
            out[s0:s0 + chunk] = g.reshape(t.shape[0], -1) @ q
        return out
    a = spec.alpha
    V = float(np.prod(spec.L))
    for s0 in range(0, nt, chunk):
        t = targets[s0:s0 + chunk]
        d = (t[:, None, :] - sources[None, :, :]).reshape(-1, 3)
        nz = np.any(d != 0.0, axis=1)
        rp = np.stack([_wrap_half(d[:, i], spec.L[i]) for i in range(3)], axis=1)
        g = np.zeros(d.shape[0])
        g[nz] = _real_space(rp[nz], np.zeros((int(nz.sum()), 0)), spec, exclude_origin=False)
        out[s0:s0 + chunk] = g.reshape(t.shape[0], -1) @ q
    ms = [np.arange(-m, m + 1) for m in spec.m_recip]
    KX, KY, KZ = np.meshgrid(*[2 * np.pi * ms[i] / spec.L[i] for i in range(3)], indexing="ij")
    k = np.stack([KX.ravel(), KY.ravel(), KZ.ravel()], axis=1)
    k2 = np.sum(k * k, axis=1)
    keep = k2 > 0
    k = k[keep]; k2 = k2[keep]
    coef = (4 * np.pi / V) * np.exp(-k2 / (4 * a * a)) / k2
    Sk = np.exp(-1j * (sources @ k.T)).T @ q                 # [K]
    # the pair sum excludes t_n == s_k; those pairs have zero displacement: remove their
    # reciprocal and constant contributions (they belong to the self term)
    for s0 in range(0, nt, chunk):
        t = targets[s0:s0 + chunk]
        out[s0:s0 + chunk] += np.real(np.exp(1j * (t @ k.T)) @ (coef * Sk))
    out += -np.pi / (a * a * V) * np.sum(q)
    same = np.all(targets[:, None, :] == sources[None, :, :], axis=2)
    if same.any():
        out -= (same.astype(np.float64) @ q) * (np.sum(coef) - np.pi / (a * a * V))
    return out
