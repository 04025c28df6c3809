"""Oracle Bloch-periodic H_eff (NEXT-4 of SURVEY.md 8(f): complex fields).  TEST INFRASTRUCTURE ONLY.

P:183-185 (Eq. 2): G_p(r) = sum_i exp(-j k0 . R_i) G_0(r - R_i).  It is the unit-cell kernel of
a charge density that is Bloch-periodic with the same phase, rho(r + R) = exp(-j k0 . R) rho(r)
(sum the free-space potential over the cells), so the field path of the static method carries
over to complex magnetisation amplitudes m(r + R) = exp(-j k0 . R) m(r) (reading R27):

* local operators (assembled over all tets and folded to the parents as in
  fem.py): a tet entry between copies a (row) and b (column) of parents n, m with lattice shifts
  s_a, s_b picks up exp(j k0 . L (s_a - s_b)) -- the column value is m(r_m + s_b L) =
  exp(-j k0 . s_b L) m_m and the row equation at the copy r_n + s_a L is exp(-j k0 . s_a L)
  times the equation at r_n.  Shift-free entries are the static ones.
* Z0: element image (t, s) seen from r_n: vertex v carries
  exp(-j k0 . L (shift_v + s)); the point-charge term of near source (p, ell) carries
  exp(-j k0 . L ell).
* AIM on modulated charges: with G~(r) = exp(j k0 . r) G_p(r) (L-periodic),
  u_n = sum_m G_p(r_n - r_m) q_m = exp(-j k0 . r_n) sum_m G~(x_n - x_m) q~_m,
  q~_m = exp(j k0 . r_m) q_m, r the unwrapped and x the wrapped parent coordinates -- the
  static AIM with the kernel G~ (a complex spectrum, no zero-mode removal: k0 is off the
  reciprocal lattice) and the precorrection of near image (n, k, img), d = x_n - x_k - img L,
  C~ = exp(j k0 . d) G0*(d) - sum w w exp(j k0 . d_g) G0*(d_g).
* brute force: u_n = sum_{k != n} G_p(r_n - r_k) q_k + G_p^reg(0) q_n + (Z0 m)_n.

Pins (tests/test_oracle_bloch_heff.py): at k0 = 2 pi j / (M L) a Bloch mode of the unit cell
IS a field of the M-cell supercell, so the Bloch brute force equals the static brute force
(oracle.heff, pinned separately) on the supercell mesh with the phased m, node by node; AIM vs
brute force <= 1e-3 and falling with the near zone; k0 -> reciprocal lattice vector is excluded.
"""
import numpy as np
import scipy.fft as sfft
import scipy.sparse as sp

from . import mesh as omesh
from . import fem, aim, z0 as oz0
from .bloch import BlochSpec, bloch_pgf


def _phase(k0, shifts, L):
    """exp(j k0 . (shifts * L)) for integer shifts [.., 3]."""
    return np.exp(1j * (np.asarray(shifts, float) * L[None, :]) @ k0)


def assemble_bloch(pm, Ms_tet, Aex_tet, k0):
    """fem.assemble with the Bloch phases of the folding (module docstring).  Returns Vt and the
    complex S, Dx..Dz, Gx..Gz (same conventions as fem.assemble)."""
    grads, vol = fem.element_gradients(pm.xyz, pm.tets)
    T = pm.tets.shape[0]
    Np = pm.n_parents
    Ms_tet = np.broadcast_to(np.asarray(Ms_tet, dtype=np.float64), (T,))
    Aex_tet = np.broadcast_to(np.asarray(Aex_tet, dtype=np.float64), (T,))
    pid = pm.pid[pm.tets]
    sh = pm.shift[pm.tets]                          # [T,4,3]
    Vt = np.zeros(Np)
    np.add.at(Vt, pid.ravel(), np.repeat(vol / 4.0, 4))
    rows, cols, s_val = [], [], []
    d_val = [[], [], []]
    g_val = [[], [], []]
    coef = 2.0 * Aex_tet / Ms_tet
    for a in range(4):
        for b in range(4):
            ph = _phase(k0, sh[:, a] - sh[:, b], pm.L)
            rows.append(pid[:, a]); cols.append(pid[:, b])
            s_val.append(ph * coef * vol * np.einsum('ij,ij->i', grads[:, a], grads[:, b]))
            for x in range(3):
                d_val[x].append(ph * Ms_tet * vol / 4.0 * grads[:, a, x])
                g_val[x].append(ph * vol / 4.0 * grads[:, b, x])
    rows = np.concatenate(rows); cols = np.concatenate(cols)

    def mk(v):
        return sp.coo_matrix((np.concatenate(v), (rows, cols)), shape=(Np, Np)).tocsr()

    Ginv = sp.diags(1.0 / Vt)
    return dict(Vt=Vt, S=mk(s_val), Dx=mk(d_val[0]), Dy=mk(d_val[1]), Dz=mk(d_val[2]),
                Gx=(Ginv @ mk(g_val[0])).tocsr(), Gy=(Ginv @ mk(g_val[1])).tocsr(),
                Gz=(Ginv @ mk(g_val[2])).tocsr(), grads=grads, vol=vol)


def assemble_z0_bloch(pm, ops, Ms_tet, k0, z0_ring=1, nquad=20):
    """z0.assemble_z0 with the Bloch phases (module docstring); ops = assemble_bloch's."""
    items, near = oz0.near_structure(pm, z0_ring)
    Np = pm.n_parents
    T = pm.tets.shape[0]
    Ms_tet = np.broadcast_to(np.asarray(Ms_tet, dtype=np.float64), (T,))
    n_it = np.array([it[0] for it in items], dtype=np.int64)
    t_it = np.array([it[1] for it in items], dtype=np.int64)
    s_it = np.array([it[2] for it in items], dtype=np.int64).reshape(-1, 3)
    va = np.array([it[3] for it in items], dtype=np.int64)
    mask = np.array([it[4] for it in items], dtype=bool).reshape(-1, 4)
    P = pm.xyz[pm.tets[t_it]] + (s_it * pm.L[None, :])[:, None, :]
    o = pm.xyz[pm.parent[n_it]]
    A, Bm = oz0.tet_moments(P, o, va, nquad)
    grads = ops["grads"][t_it]
    rows, cols, vals = [], [], [[], [], []]
    for k in range(4):
        sel = mask[:, k]
        for m in range(4):
            vm = pm.tets[t_it[sel], m]
            ph = _phase(k0, -(pm.shift[vm] + s_it[sel]), pm.L)
            w = Ms_tet[t_it[sel], None] * (Bm[sel, k, m, :] + grads[sel, k, :] * A[sel, m, None])
            rows.append(n_it[sel]); cols.append(pm.pid[vm])
            for x in range(3):
                vals[x].append(ph * w[:, x])
    D = [ops["Dx"].tocsr(), ops["Dy"].tocsr(), ops["Dz"].tocsr()]
    xyz_p = pm.xyz[pm.parent]
    for (n, p, ell) in near:
        d = xyz_p[n] - xyz_p[p] - np.array(ell) * pm.L
        r = np.linalg.norm(d)
        if r == 0.0:
            continue
        g = np.exp(-1j * float((np.array(ell) * pm.L) @ k0)) / r
        for x in range(3):
            lo, hi = D[x].indptr[p], D[x].indptr[p + 1]
            cc = D[x].indices[lo:hi]
            for y in range(3):
                vals[y].append(-g * D[x].data[lo:hi] if y == x else np.zeros(hi - lo, complex))
            rows.append(np.full(cc.size, n)); cols.append(cc)
    rows = np.concatenate(rows); cols = np.concatenate(cols)
    Z = [sp.coo_matrix((np.concatenate(vals[x]), (rows, cols)), shape=(Np, Np)).tocsr() for x in range(3)]
    return dict(Zx=Z[0], Zy=Z[1], Zz=Z[2])


def kernel_table_bloch(grid, spec):
    """aim.kernel_table for G~(d) = exp(j k0 . d) G_p(d; k0) (complex); G~(0) = G_p^reg(0; k0)."""
    axes = []
    for a in range(3):
        P = grid.fft[a]
        j = np.arange(P)
        axes.append(j * grid.delta[a] if grid.periodic[a] else np.where(j < grid.n[a], j, j - P) * grid.delta[a])
    D = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 3)
    k3 = np.zeros(3)
    k3[spec.axes] = spec.k0
    K = np.zeros(D.shape[0], complex)
    nz = np.any(D != 0.0, axis=1)
    K[nz] = np.exp(1j * (D[nz] @ k3)) * bloch_pgf(D[nz], spec)
    K[~nz] = bloch_pgf(None, spec, self_term=True)[0]
    K = K.reshape(tuple(grid.fft))
    for a in range(3):
        if not grid.periodic[a]:
            sl = [slice(None)] * 3
            sl[a] = grid.n[a]
            K[tuple(sl)] = 0.0
    return K


def precorrection_bloch(grid, xyz_w, lattice, S, W, s, p, k3):
    """aim.precorrection with the modulation exp(j k0 . d) on every G0* term."""
    aim.check_rer(grid, lattice, s, p)
    nn, kk, img = aim.near_pairs(grid, xyz_w, lattice, s)
    Lv = np.array([lattice[a] if grid.periodic[a] else 0.0 for a in range(3)])
    d = xyz_w[nn] - xyz_w[kk] - img * Lv[None, :]
    val = np.exp(1j * (d @ k3)) * aim.g0_star(d)
    p1 = p + 1
    for oa in np.ndindex(p1, p1, p1):
        wa = W[nn, 0, oa[0]] * W[nn, 1, oa[1]] * W[nn, 2, oa[2]]
        for ob in np.ndindex(p1, p1, p1):
            wb = W[kk, 0, ob[0]] * W[kk, 1, ob[1]] * W[kk, 2, ob[2]]
            dg = ((S[nn] + np.array(oa)) - (S[kk] + np.array(ob)) - img * grid.n[None, :]) * grid.delta[None, :]
            val = val - wa * wb * np.exp(1j * (dg @ k3)) * aim.g0_star(dg)
    n = xyz_w.shape[0]
    return sp.coo_matrix((val, (nn, kk)), shape=(n, n)).tocsr()


class BlochModel:
    """The Bloch H_eff of complex amplitudes m [N',3] (module docstring).  k0 (3-vector, rad/cm,
    user frame) must have a non-zero component on some periodic axis; components on free axes
    are ignored (no phase there)."""

    def __init__(self, xyz, tets, periodic, lattice, grid_n, k0, Ms=637.0, Aex=1.4e-6, order=1,
                 rer_scale=2.0, z0_ring=1, match_tol=0.0, nquad=20, build_aim=True):
        self.pm = omesh.PeriodicMesh(xyz, tets, periodic, lattice, match_tol)
        T = self.pm.tets.shape[0]
        self.Ms_tet = np.full(T, float(Ms)) if np.isscalar(Ms) else np.asarray(Ms, float)
        self.Aex_tet = np.full(T, float(Aex)) if np.isscalar(Aex) else np.asarray(Aex, float)
        self.periodic = self.pm.periodic
        self.lattice = tuple(float(lattice[a]) if periodic[a] else 0.0 for a in range(3))
        self.k3 = np.array([float(k0[a]) if periodic[a] else 0.0 for a in range(3)])
        self.spec = BlochSpec(self.periodic, self.lattice, self.k3)
        self.ops = assemble_bloch(self.pm, self.Ms_tet, self.Aex_tet, self.k3)
        self.z0 = assemble_z0_bloch(self.pm, self.ops, self.Ms_tet, self.k3, z0_ring, nquad)
        self.r = self.pm.xyz[self.pm.parent]             # unwrapped parent coordinates
        self.xw = self.pm.wrapped_parent_xyz()
        self.mod = np.exp(1j * (self.r @ self.k3))       # exp(j k0 . r_n)
        if build_aim:
            self.grid = aim.Grid(grid_n, self.periodic, self.lattice, self.xw)
            self.S, self.W = aim.stencils(self.grid, self.xw, order)
            self.P = aim.projection_matrix(self.grid, self.S, self.W)
            self.K = kernel_table_bloch(self.grid, self.spec)
            self.Ghat = sfft.fftn(self.K)                # complex, every frequency kept
            self.C = precorrection_bloch(self.grid, self.xw, self.lattice, self.S, self.W, rer_scale, order,
                                         self.k3)

    @property
    def n_parents(self):
        return self.pm.n_parents

    def charges(self, m):
        o = self.ops
        return o["Dx"] @ m[:, 0] + o["Dy"] @ m[:, 1] + o["Dz"] @ m[:, 2]

    def u_loc(self, m):
        z = self.z0
        return z["Zx"] @ m[:, 0] + z["Zy"] @ m[:, 1] + z["Zz"] @ m[:, 2]

    def exchange(self, m):
        return -(self.ops["S"] @ m) / self.ops["Vt"][:, None]

    def potential_aim(self, m):
        q = self.charges(m)
        qt = self.mod * q
        Qp = np.zeros(tuple(self.grid.fft), complex)
        n = self.grid.n
        Qp[:n[0], :n[1], :n[2]] = (self.P @ qt).reshape(tuple(n))
        U = sfft.ifftn(self.Ghat * sfft.fftn(Qp))[:n[0], :n[1], :n[2]]
        ut = self.P.T @ U.ravel() + self.C @ qt
        return np.conj(self.mod) * ut + self.u_loc(m)

    def potential_bf(self, m, chunk=64):
        q = self.charges(m)
        u = np.zeros(self.n_parents, complex)
        N = self.n_parents
        for s in range(0, N, chunk):
            rows = np.arange(s, min(N, s + chunk))
            d = (self.r[rows, None, :] - self.r[None, :, :]).reshape(-1, 3)
            off = (rows[:, None] != np.arange(N)[None, :]).ravel()
            g = np.zeros(d.shape[0], complex)
            g[off] = bloch_pgf(d[off], self.spec)
            u[rows] = g.reshape(rows.size, N) @ q
        u += bloch_pgf(None, self.spec, self_term=True)[0] * q
        return u + self.u_loc(m)

    def gradient(self, u):
        o = self.ops
        return -np.stack([o["Gx"] @ u, o["Gy"] @ u, o["Gz"] @ u], axis=1)

    def demag(self, m, method="aim"):
        return self.gradient(self.potential_aim(m) if method == "aim" else self.potential_bf(m))

    def heff(self, m, method="aim"):
        return self.demag(m, method) + self.exchange(m)
