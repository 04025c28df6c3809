"""Oracle pins: exact near-field integrals Z0.

Pins: (1) the volume form of the node-k potential equals the surface form
sum_{F ∋ k} (n_F . M) int_F G0 phi_k dS for uniform M (divergence theorem), with the surface
integrals done by an independent 2D quadrature here; (2) sum over all elements of the
volume form of an isolated uniformly magnetised box equals the closed-form potential of
its two charged faces (rectangle potential formula); (3) uniform m in a filled periodic
cell gives Z0 m = 0; (4) quadrature-order convergence.
"""
import itertools

import numpy as np
import pytest

from oracle import z0 as Z, mesh as om, fem
from oracle.heff import OracleModel
from synth import kuhn_voxel_mesh, make_config


def _tri_integral_phi_over_r(V, o, k_local, n=40):
    """int_F phi_k(y)/|o - y| dA on triangle V[3], 2D collapse at the vertex nearest o."""
    d = np.linalg.norm(V - o, axis=1)
    a = int(np.argmin(d))
    order = [a] + [i for i in range(3) if i != a]
    W = V[order]
    x, w = np.polynomial.legendre.leggauss(n)
    x = 0.5 * (x + 1); w = 0.5 * w
    U, Vv = np.meshgrid(x, x, indexing="ij")
    U = U.ravel(); Vv = Vv.ravel(); ww = np.outer(w, w).ravel()
    lam = np.stack([1 - U, U * (1 - Vv), U * Vv], 1)          # barycentrics of W
    y = lam @ W
    area2 = np.linalg.norm(np.cross(W[1] - W[0], W[2] - W[0]))
    jac = area2 * U
    phi = lam[:, order.index(k_local)]
    return np.sum(ww * jac * phi / np.linalg.norm(o - y, axis=1))


@pytest.mark.parametrize("observer", ["vertex", "near", "far"])
def test_volume_form_equals_surface_form(observer):
    rng = np.random.default_rng(4)
    P = np.array([[0, 0, 0], [1, 0.1, 0], [0.2, 1, 0.1], [0.1, 0.2, 0.9]]) + rng.uniform(-0.05, 0.05, (4, 3))
    if observer == "vertex":
        o, va = P[2].copy(), 2
    elif observer == "near":
        o, va = P[0] - np.array([0.3, 0.4, 0.35]), -1
    else:
        o, va = np.array([2.0, 1.5, -1.0]), -1
    A, B = Z.tet_moments(P[None], o[None], np.array([va]))
    grads, vol = fem.element_gradients(P, np.array([[0, 1, 2, 3]]))
    M = np.array([0.3, -0.5, 0.8])
    faces = [(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)]
    cen = P.mean(axis=0)
    for k in range(4):
        vol_form = (B[0, k].sum(axis=0) + grads[0, k] * A[0].sum()) @ M
        surf = 0.0
        for f in faces:
            if k not in f:
                continue
            V = P[list(f)]
            nrm = np.cross(V[1] - V[0], V[2] - V[0]); nrm /= np.linalg.norm(nrm)
            if nrm @ (V[0] - cen) < 0:
                nrm = -nrm
            surf += (nrm @ M) * _tri_integral_phi_over_r(V, o, list(f).index(k))
        assert vol_form == pytest.approx(surf, rel=1e-9, abs=1e-12)


def _rect_potential(o, zf, a, b):
    """int_{a0}^{a1} int_{b0}^{b1} dx dy / sqrt((x-ox)^2 + (y-oy)^2 + (zf-oz)^2), closed form
    F = X ln(Y+R) + Y ln(X+R) - Z atan(XY/(ZR)) over the four corners."""
    Zd = zf - o[2]
    tot = 0.0
    for (i, sa) in ((1, 1), (0, -1)):
        for (j, sb) in ((1, 1), (0, -1)):
            X = a[i] - o[0]; Y = b[j] - o[1]
            R = np.sqrt(X * X + Y * Y + Zd * Zd)
            F = X * np.log(Y + R) + Y * np.log(X + R) - Zd * np.arctan(X * Y / (Zd * R))
            tot += sa * sb * F
    return tot


def test_box_potential_closed_form():
    # uniform M_z in an isolated box: sum over all elements of int grad'G0 . M dV equals
    # M_z [I(top face) - I(bottom face)] (surface charges +-M_z)
    m = kuhn_voxel_mesh(np.ones((3, 3, 2), bool), 1.0, jitter=0.15, seed=9)
    xyz, tets = m.xyz, m.tets
    lo, hi = xyz.min(axis=0), xyz.max(axis=0)
    interior = np.nonzero(np.all((xyz > lo + 1e-9) & (xyz < hi - 1e-9), axis=1))[0]
    for obs in interior[:2]:
        o = xyz[obs]
        va = np.array([list(t).index(obs) if obs in t else -1 for t in tets])
        A, B = Z.tet_moments(xyz[tets], np.tile(o, (len(tets), 1)), va)
        u = B.sum(axis=(0, 1, 2))[2]          # sum_k sum_m B_km . z_hat
        ref = _rect_potential(o, hi[2], (lo[0], hi[0]), (lo[1], hi[1])) - \
            _rect_potential(o, lo[2], (lo[0], hi[0]), (lo[1], hi[1]))
        assert u == pytest.approx(ref, rel=1e-9)


def test_uniform_m_filled_cell_zero():
    c = make_config("C1", coarsen=2)
    mo = OracleModel(c["mesh"].xyz, c["mesh"].tets, c["periodic"], c["lattice"], (8, 8, 8),
                     z0_ring=1, build_aim=False)
    m = np.tile([0.6, 0.0, 0.8], (mo.n_parents, 1))
    # scale: the row sums of |Z| (the size of the terms that cancel)
    scale = (abs(mo.z0["Zx"]) + abs(mo.z0["Zz"])).sum(axis=1).max()
    assert np.abs(mo.u_loc(m)).max() < 1e-8 * scale      # regular-element quadrature ~1e-9


def test_quadrature_convergence():
    rng = np.random.default_rng(1)
    P = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]) + rng.uniform(-0.1, 0.1, (4, 3))
    for va in range(4):
        a1, b1 = Z.moments_vertex(P[None], np.array([va]), n=20)
        a2, b2 = Z.moments_vertex(P[None], np.array([va]), n=40)
        assert np.abs(a1 - a2).max() < 1e-11 * np.abs(a2).max()
        assert np.abs(b1 - b2).max() < 1e-11 * np.abs(b2).max()
    o = P[0] + np.array([-0.4, -0.3, -0.2])
    a1, b1 = Z.moments_regular(P[None], o[None], n=8, level=1)
    a2, b2 = Z.moments_regular(P[None], o[None], n=12, level=2)
    assert np.abs(a1 - a2).max() < 1e-8 * np.abs(a2).max()
    assert np.abs(b1 - b2).max() < 1e-8 * np.abs(b2).max()
