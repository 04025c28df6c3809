"""Oracle BAIM / AIM: O8-O11 and E2-E5 of SURVEY.md 8(c).  TEST INFRASTRUCTURE ONLY.

BAIM steps: (1) project nodal charges onto a Cartesian grid, (2) convolve
with the PGF by FFT, (3) interpolate back, (4) precorrect near interactions.  Periodic
modifications: step 2 uses G_p with no padding on periodic axes (P:214,
P:340); step 4 subtracts / adds back G_0 only, over near periodic images (P:216-231,
Eq. new_er).  The conventions contract K4-K9 fixes every discrete choice.
"""
import itertools
import numpy as np
import scipy.fft as sfft
import scipy.sparse as sp
from scipy.spatial import cKDTree

from .pgf import PgfSpec, pgf, pgf_self


class Grid:
    """K4 / Eq. grid (reading R6): periodic axis x_i = i*Delta, Delta = L/N;
    non-periodic axis x_i = x_min + i*Delta, Delta = (x_max - x_min)/(N - 1)."""

    def __init__(self, n, periodic, lattice, xyz_wrapped):
        self.n = np.array(n, dtype=np.int64)
        self.periodic = tuple(int(p) for p in periodic)
        self.origin = np.zeros(3)
        self.delta = np.zeros(3)
        for a in range(3):
            if self.periodic[a]:
                self.delta[a] = lattice[a] / n[a]
            else:
                lo, hi = xyz_wrapped[:, a].min(), xyz_wrapped[:, a].max()
                self.origin[a] = lo
                self.delta[a] = (hi - lo) / (n[a] - 1)
        # K6: FFT lengths
        self.fft = np.array([n[a] if self.periodic[a] else 2 * n[a] for a in range(3)], dtype=np.int64)


def lagrange_weights(t, s, p):
    """Lagrange basis on the integer nodes s..s+p evaluated at t (AIM moment matching,
    reading R7): w_j = prod_{i != j} (t - (s+i)) / (j - i)."""
    t = np.asarray(t, dtype=np.float64)
    w = np.ones(t.shape + (p + 1,))
    for j in range(p + 1):
        for i in range(p + 1):
            if i != j:
                w[..., j] *= (t - (s + i)) / (j - i)
    return w


def stencils(grid, xyz_wrapped, p):
    """K5: per node and axis the unwrapped start index s and the p+1 weights.
    p odd: s = floor(t) - (p-1)/2; p even: s = floor(t + 1/2) - p/2; non-periodic axes
    clamp s to [0, N-1-p]."""
    n = xyz_wrapped.shape[0]
    S = np.zeros((n, 3), dtype=np.int64)
    W = np.zeros((n, 3, p + 1))
    for a in range(3):
        t = (xyz_wrapped[:, a] - grid.origin[a]) / grid.delta[a]
        if p % 2 == 1:
            s = np.floor(t).astype(np.int64) - (p - 1) // 2
        else:
            s = np.floor(t + 0.5).astype(np.int64) - p // 2
        if not grid.periodic[a]:
            s = np.clip(s, 0, grid.n[a] - 1 - p)
        S[:, a] = s
        W[:, a, :] = lagrange_weights(t, s, p)
    return S, W


def projection_matrix(grid, S, W):
    """P as a sparse [G, N'] matrix (G = prod n, C order [x][y][z]); periodic indices
    wrap mod N.  Interpolation is P^T (reading R7)."""
    n_nodes, _, p1 = W.shape
    rows, cols, vals = [], [], []
    for off in itertools.product(range(p1), repeat=3):
        idx = [S[:, a] + off[a] for a in range(3)]
        for a in range(3):
            if grid.periodic[a]:
                idx[a] = np.mod(idx[a], grid.n[a])
        lin = (idx[0] * grid.n[1] + idx[1]) * grid.n[2] + idx[2]
        w = W[:, 0, off[0]] * W[:, 1, off[1]] * W[:, 2, off[2]]
        rows.append(lin); cols.append(np.arange(n_nodes)); vals.append(w)
    G = int(np.prod(grid.n))
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(G, n_nodes)).tocsr()


def kernel_table(grid, spec):
    """O10 / K6-K7: K on the padded grid.  Index j on a periodic axis -> j*Delta;
    non-periodic: j < N -> j*Delta, j > N -> (j - 2N)*Delta, j = N -> value 0 (never used
    by the linear convolution).  K(0) = G_p^reg(0)."""
    axes = []
    for a in range(3):
        P = grid.fft[a]
        j = np.arange(P)
        if grid.periodic[a]:
            d = j * grid.delta[a]
        else:
            d = np.where(j < grid.n[a], j, j - P) * grid.delta[a]
        axes.append(d)
    D = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 3)
    K = np.zeros(D.shape[0])
    nz = np.any(D != 0.0, axis=1)
    K[nz] = pgf(D[nz], spec)
    K[~nz] = pgf_self(spec)
    K = K.reshape(tuple(grid.fft))
    for a in range(3):
        if not grid.periodic[a]:
            sl = [slice(None)] * 3
            sl[a] = grid.n[a]
            K[tuple(sl)] = 0.0
    return K


def kernel_spectrum(K):
    """G_hat = real(FFT(K)), G_hat[0,0,0] := 0 (K7: exact, since sum Q = sum q = 0)."""
    Gh = np.real(np.fft.fftn(K))
    Gh[0, 0, 0] = 0.0
    return Gh


# threads of the grid FFTs (scipy.fft workers; the CPU baseline times 1 and all cores)
FFT_WORKERS = 1


def convolve(grid, Ghat, Q):
    """E3: U = real(IFFT(G_hat * FFT(Q_pad))) restricted to the unpadded grid."""
    Qp = np.zeros(tuple(grid.fft))
    Qp[:grid.n[0], :grid.n[1], :grid.n[2]] = Q
    U = np.real(sfft.ifftn(Ghat * sfft.fftn(Qp, workers=FFT_WORKERS), workers=FFT_WORKERS))
    return U[:grid.n[0], :grid.n[1], :grid.n[2]]


def g0_star(d):
    """G0*(d) = 1/|d| for d != 0, 0 at d = 0 (K9)."""
    r = np.linalg.norm(d, axis=-1)
    with np.errstate(divide='ignore'):
        return np.where(r > 0, 1.0 / np.where(r > 0, r, 1.0), 0.0)


def r_er(grid, s):
    """r_ER = s * max(Delta_x, Delta_y, Delta_z), the same on every axis (P:220:
    "|r_ER| = max(Delta_x, Delta_y, Delta_z)"; the cube region of P:225; reading R8)."""
    return s * float(np.max(grid.delta))


def check_rer(grid, lattice, s, p):
    """K8 validity on periodic axes: r_ER < L/2 and r_ER/Delta + p + 1 < N/2 (no near pair's
    stencils reach the next periodic image of the singularity)."""
    r = r_er(grid, s)
    for a in range(3):
        if grid.periodic[a]:
            if not (r < lattice[a] / 2 and r / grid.delta[a] + p + 1 < grid.n[a] / 2):
                raise ValueError("r_ER too large on periodic axis %d" % a)


def near_pairs(grid, xyz_w, lattice, s, rows=None):
    """K8: all (n, k, img) with |x_n - x_k - img*L| <= r_ER on every axis (closed),
    img in {-1,0,1} on periodic axes (Eq. new_er; readings R8, R9).
    With `rows`, only observers n in rows."""
    rER = np.full(3, r_er(grid, s))
    y = xyz_w / rER[None, :]
    tree = cKDTree(y)
    out_n, out_k, out_img = [], [], []
    obs = np.arange(xyz_w.shape[0]) if rows is None else np.asarray(rows)
    rng = [(-1, 0, 1) if grid.periodic[a] else (0,) for a in range(3)]
    for img in itertools.product(*rng):
        sh = np.array(img, dtype=np.float64) * np.array([lattice[a] if grid.periodic[a] else 0.0
                                                         for a in range(3)])
        # |x_n - (x_k + sh)| <= rER  <=>  query points x_n - sh against tree of x_k
        hits = tree.query_ball_point((xyz_w[obs] - sh[None, :]) / rER[None, :], r=1.0, p=np.inf)
        for nidx, ks in zip(obs, hits):
            for k in ks:
                d = xyz_w[nidx] - xyz_w[k] - sh
                if np.all(np.abs(d) <= rER):       # closed interval in unscaled fp64
                    out_n.append(nidx); out_k.append(k); out_img.append(img)
    return np.array(out_n, dtype=np.int64), np.array(out_k, dtype=np.int64), np.array(out_img, dtype=np.int64).reshape(-1, 3)


def precorrection(grid, xyz_w, lattice, S, W, s, p, rows=None):
    """O11 / K9: C_box[n,k] = G0*(d) - sum_{a in st(n)} sum_{b in st(k)} w_na w_kb
    G0*((a - b - img*N) o Delta), d = x_n - x_k - img*L (subtract the grid's
    G_0 contribution and add it back directly).  With `rows`, only those rows."""
    check_rer(grid, lattice, s, p)
    nn, kk, img = near_pairs(grid, xyz_w, lattice, s, rows)
    Lv = np.array([lattice[a] if grid.periodic[a] else 0.0 for a in range(3)])
    d = xyz_w[nn] - xyz_w[kk] - img * Lv[None, :]
    val = g0_star(d)
    p1 = p + 1
    for oa in itertools.product(range(p1), repeat=3):
        wa = W[nn, 0, oa[0]] * W[nn, 1, oa[1]] * W[nn, 2, oa[2]]
        for ob in itertools.product(range(p1), repeat=3):
            wb = W[kk, 0, ob[0]] * W[kk, 1, ob[1]] * W[kk, 2, ob[2]]
            idx = (S[nn] + np.array(oa)) - (S[kk] + np.array(ob)) - img * grid.n[None, :]
            val = val - wa * wb * g0_star(idx * grid.delta[None, :])
    n = xyz_w.shape[0]
    return sp.coo_matrix((val, (nn, kk)), shape=(n, n)).tocsr()
