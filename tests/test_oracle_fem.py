"""Oracle pins: element operators and LCA folding."""
import numpy as np
import pytest

from oracle import mesh as om, fem
from synth import kuhn_voxel_mesh, make_config

UNIT_TET = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)


def _pm(mask, h, periodic, lattice, jitter=0.15, seed=3, wrap=None):
    wrap = wrap or tuple(bool(p) for p in periodic)
    m = kuhn_voxel_mesh(mask, h, wrap=wrap, jitter=jitter, seed=seed)
    return m, om.PeriodicMesh(m.xyz, m.tets, periodic, lattice)


def test_unit_tet_gradients_and_stiffness():
    # S:128 [DERIVED]: unit tet, int grad(phi_1).grad(phi_1) dV = 1/2
    g, v = fem.element_gradients(UNIT_TET, np.array([[0, 1, 2, 3]]))
    assert v[0] == pytest.approx(1 / 6)
    assert np.allclose(g[0], [[-1, -1, -1], [1, 0, 0], [0, 1, 0], [0, 0, 1]], atol=1e-15)
    pm = om.PeriodicMesh(UNIT_TET, np.array([[0, 1, 2, 3]]), (0, 0, 0), (0, 0, 0))
    ops = fem.assemble(pm, 1.0, 0.5)        # 2A/Ms = 1
    assert ops["S"][0, 0] == pytest.approx(0.5)
    assert ops["S"][1, 1] == pytest.approx(1 / 6)
    assert ops["Vt"].sum() == pytest.approx(1 / 6)


@pytest.mark.parametrize("periodic", [(1, 0, 0), (1, 1, 0), (1, 1, 1)])
def test_stiffness_symmetric_zero_rowsum(periodic):
    n = 4
    L = (n * 1.0,) * 3
    _, pm = _pm(np.ones((n, n, n), bool), 1.0, periodic, L)
    ops = fem.assemble(pm, 1.0, 0.5)
    S = ops["S"].toarray()
    assert np.allclose(S, S.T, atol=1e-13)            # S:152 folded symmetry
    assert np.abs(S.sum(axis=1)).max() < 1e-13 * np.abs(S).max()   # S:149 zero row sum
    # uniform m -> H_ex = 0
    H = fem.exchange_field(ops, np.tile([0.3, 0.4, 0.5], (pm.n_parents, 1)))
    assert np.abs(H).max() < 1e-12


def test_fold_equivalence_unrolled_bar():
    # S:150 / acceptance 5: operators on a 1D T-PBC bar of n cells equal (entrywise) the
    # operators of the explicitly unrolled 2-period bar, restricted to one period and folded.
    n, ny, h = 4, 2, 1.0
    m1 = kuhn_voxel_mesh(np.ones((n, ny, ny), bool), h, wrap=(True, False, False), jitter=0.15, seed=5)
    m2 = kuhn_voxel_mesh(np.ones((2 * n, ny, ny), bool), h, wrap=(True, False, False), jitter=0.15, seed=5)
    # m2's jitter table has period 2n; re-jitter it with the period-n table of m1 so that the
    # geometry is the exact 2-period unrolling of m1
    idx1 = m1.meta["lattice_index"]; idx2 = m2.meta["lattice_index"]
    base1 = {tuple(i): m1.xyz[k] - i * h for k, i in enumerate(idx1)}
    xyz2 = np.array([i * h + base1[(i[0] % n if i[0] < 2 * n else n, i[1], i[2])]
                     if i[0] % n or i[0] == 0 else i * h + base1[(0 if i[0] < 2 * n else n, i[1], i[2])]
                     for i in idx2])
    pm1 = om.PeriodicMesh(m1.xyz, m1.tets, (1, 0, 0), (n * h, 0, 0))
    pm2 = om.PeriodicMesh(xyz2, m2.tets, (1, 0, 0), (2 * n * h, 0, 0))
    ops1 = fem.assemble(pm1, 1.0, 0.5)
    ops2 = fem.assemble(pm2, 1.0, 0.5)
    # map parents of pm2 to parents of pm1 via coordinates mod L
    key1 = {tuple(np.round(np.mod(pm1.xyz[p], [n * h, 1e9, 1e9]), 9)): i for i, p in enumerate(pm1.parent)}
    map21 = np.array([key1[tuple(np.round(np.mod(pm2.xyz[p], [n * h, 1e9, 1e9]), 9))] for p in pm2.parent])
    for name in ("S", "Dx", "Gy"):
        A2 = ops2[name].toarray()
        fold = np.zeros((pm2.n_parents, pm1.n_parents))
        for j in range(pm2.n_parents):
            fold[:, map21[j]] += A2[:, j]
        A1 = ops1[name].toarray()
        for i in range(pm2.n_parents):
            assert np.allclose(fold[i], A1[map21[i]], rtol=0, atol=1e-12 * np.abs(A1).max())


def test_exchange_sinusoid_second_order():
    # S:127 / acceptance 4: m_z = cos(2 pi x / L) on a 1D T-PBC bar ->
    # H_ex,z = -(2A/Ms) (2 pi / L)^2 m_z with 2nd-order convergence
    L = 1.0
    errs = []
    for n in (8, 16, 32):
        h = L / n
        _, pm = _pm(np.ones((n, 1, 1), bool), h, (1, 0, 0), (L, 0, 0), jitter=0.0)
        ops = fem.assemble(pm, 2.0, 1.0)            # 2A/Ms = 1
        x = pm.xyz[pm.parent, 0]
        k = 2 * np.pi / L
        m = np.stack([0 * x, np.sin(k * x), np.cos(k * x)], 1)
        H = fem.exchange_field(ops, m)
        errs.append(np.abs(H[:, 2] + k * k * m[:, 2]).max() / (k * k))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(rates > 1.9), (errs, rates)


def test_charge_neutrality_and_dipole():
    # sum_n q_n = 0 for any M; dipole identity sum_n q_n r_n = int M dV (isolated body)
    _, pm = _pm(np.ones((3, 3, 2), bool), 1.0, (0, 0, 0), (0, 0, 0))
    ops = fem.assemble(pm, 2.5, 1.0)
    m = np.random.default_rng(1).normal(size=(pm.n_parents, 3))
    q = fem.charges(ops, m)
    assert abs(q.sum()) < 1e-13 * np.abs(q).max()
    # int M_h dV = sum_T V_T/4 sum_{m in T} Ms m_m
    Mint = 2.5 * np.einsum('t,tmx->x', pm.vol / 4, m[pm.pid[pm.tets]])
    assert np.allclose(q @ pm.xyz[pm.parent], Mint, rtol=1e-12, atol=1e-14)
    # S:136 uniform M_z on an isolated box: sum q z = M_z V
    mz = np.tile([0, 0, 1.0], (pm.n_parents, 1))
    assert q.sum() == pytest.approx(0, abs=1e-12)
    qz = fem.charges(ops, mz)
    assert qz @ pm.xyz[pm.parent, 2] == pytest.approx(2.5 * pm.vol.sum(), rel=1e-12)


def test_charge_zero_in_filled_periodic_cell():
    # uniform M filling a fully periodic 3D T-PBC cell -> q = 0
    c = make_config("C1", coarsen=2)
    pm = om.PeriodicMesh(c["mesh"].xyz, c["mesh"].tets, c["periodic"], c["lattice"])
    ops = fem.assemble(pm, 637.0, 1.4e-6)
    q = fem.charges(ops, np.tile([0.6, 0.0, 0.8], (pm.n_parents, 1)))
    scale = 637.0 * pm.vol.mean() ** (2 / 3)
    assert np.abs(q).max() < 1e-12 * scale


def test_gradient_linear_reproduction():
    # u = const -> 0; u = a.r -> grad = a exactly (non-periodic mesh)
    _, pm = _pm(np.ones((3, 2, 2), bool), 1.0, (0, 0, 0), (0, 0, 0))
    ops = fem.assemble(pm, 1.0, 1.0)
    x = pm.xyz[pm.parent]
    assert np.abs(fem.gradient_field(ops, np.ones(pm.n_parents))).max() < 1e-13
    a = np.array([0.3, -1.2, 2.0])
    H = fem.gradient_field(ops, x @ a)
    assert np.allclose(H, -a[None, :], atol=1e-12)
