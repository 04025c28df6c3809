"""Oracle H_eff pipeline (E1-E7 of SURVEY.md 8(c)) and O(N'^2) brute force (O12).
TEST INFRASTRUCTURE ONLY.

AIM:   u = P^T F^-1( G_hat . F P q ) + C_box q + Z0 m,   H_ms = -G u
BF:    u_n = sum_{k != n} G_p(r_n - r_k) q_k + G_p^reg(0) q_n + (Z0 m)_n  (reading R13)
H_eff = H_ms + H_ex  (anisotropy / applied fields are NEXT-2)
"""
import numpy as np

from . import mesh as omesh
from . import fem, aim, z0 as oz0
from .pgf import PgfSpec, pgf, pgf_self, pgf_potential


class OracleModel:
    def __init__(self, xyz, tets, periodic, lattice, grid_n, Ms=637.0, Aex=1.4e-6,
                 order=1, rer_scale=2.0, z0_ring=1, match_tol=0.0, nquad=20, build_aim=True, rows=None):
        """rows: if given, Z0 and C_box are built only for these parent rows (sampled
        full-size checks: u is then valid on `rows` only)."""
        self.pm = omesh.PeriodicMesh(xyz, tets, periodic, lattice, match_tol)
        T = self.pm.tets.shape[0]
        self.Ms_tet = np.full(T, float(Ms)) if np.isscalar(Ms) else np.asarray(Ms, float)
        self.Aex_tet = np.full(T, float(Aex)) if np.isscalar(Aex) else np.asarray(Aex, float)
        self.ops = fem.assemble(self.pm, self.Ms_tet, self.Aex_tet)
        self.rows = rows
        # rows = [] defers Z0 to the caller (sampled full-size checks pick their rows later)
        self.z0 = oz0.assemble_z0(self.pm, self.ops, self.Ms_tet, z0_ring, nquad, rows) \
            if rows is None or len(rows) else None
        self.xw = self.pm.wrapped_parent_xyz()
        self.periodic = self.pm.periodic
        self.lattice = tuple(float(lattice[a]) if periodic[a] else 0.0 for a in range(3))
        self.spec = PgfSpec(self.periodic, self.lattice)
        self.order = order
        self.rer_scale = rer_scale
        if build_aim:
            self.grid = aim.Grid(grid_n, self.periodic, self.lattice, self.xw)
            self.S, self.W = aim.stencils(self.grid, self.xw, order)
            self.P = aim.projection_matrix(self.grid, self.S, self.W)
            self.K = aim.kernel_table(self.grid, self.spec)
            self.Ghat = aim.kernel_spectrum(self.K)
            self.C = aim.precorrection(self.grid, self.xw, self.lattice, self.S, self.W, rer_scale, order,
                                       rows)

    @property
    def n_parents(self):
        return self.pm.n_parents

    # ---------------------------------------------------------------- E1
    def charges(self, m):
        return fem.charges(self.ops, m)

    def u_loc(self, m):
        return self.z0["Zx"] @ m[:, 0] + self.z0["Zy"] @ m[:, 1] + self.z0["Zz"] @ m[:, 2]

    def exchange(self, m):
        return fem.exchange_field(self.ops, m)

    # ---------------------------------------------------------------- E2-E5
    def potential_aim(self, m, parts=False):
        q = self.charges(m)
        Q = (self.P @ q).reshape(tuple(self.grid.n))
        U = aim.convolve(self.grid, self.Ghat, Q)
        ut = self.P.T @ U.ravel()
        uc = self.C @ q
        ul = self.u_loc(m)
        u = ut + uc + ul
        if parts:
            return dict(q=q, Q=Q, U=U, u_grid=ut, u_corr=uc, u_loc=ul, u=u)
        return u

    def potential_bf(self, m, chunk=256):
        """O12: u_n = sum_{k != n} G_p(r_n - r_k) q_k + G_p^reg(0) q_n + (Z0 m)_n.
        Periodic kernels use the C pair sums of oracle/bf.c (pinned to oracle.pgf to 1e-13 in
        tests/test_oracle_bf.py); free space the NumPy sum."""
        q = self.charges(m)
        if self.spec.dim > 0:
            from . import bf
            u = bf.potential(self.xw, self.xw, q, self.spec)
        else:
            u = pgf_potential(self.xw, self.xw, q, self.spec, chunk)
        u += pgf_self(self.spec) * q
        return u + self.u_loc(m)

    # ---------------------------------------------------------------- E6-E7
    def demag(self, m, method="aim"):
        u = self.potential_aim(m) if method == "aim" else self.potential_bf(m)
        return fem.gradient_field(self.ops, u)

    def heff(self, m, method="aim"):
        return self.demag(m, method) + self.exchange(m)
