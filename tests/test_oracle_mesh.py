"""Oracle pins: mesh, T-PBC pairs, LCA, fold."""
import numpy as np
import pytest

from oracle import mesh as om
from synth import kuhn_voxel_mesh, make_config

UNIT_TET = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)


def test_unit_tet_volume_and_orientation():
    # S:42-43 [TRIVIAL]: unit tetrahedron volume 1/6, negative orientation fixed
    t = np.array([[0, 1, 2, 3]])
    assert om.signed_volumes(UNIT_TET, t)[0] == pytest.approx(1 / 6, abs=1e-15)
    tn = np.array([[0, 2, 1, 3]])
    assert om.signed_volumes(UNIT_TET, tn)[0] == pytest.approx(-1 / 6, abs=1e-15)
    fixed = om.orient(UNIT_TET, tn)
    assert om.signed_volumes(UNIT_TET, fixed)[0] == pytest.approx(1 / 6, abs=1e-15)


def test_cube_six_tets_volume():
    # S:44 [DERIVED]: 2x2x2-node unit cube split into 6 tets -> N=8, total volume 1
    m = kuhn_voxel_mesh(np.ones((1, 1, 1), bool), 1.0)
    assert m.n_nodes == 8 and m.n_tets == 6
    assert om.signed_volumes(m.xyz, m.tets).sum() == pytest.approx(1.0, abs=1e-14)


def test_degenerate_rejected():
    xyz = np.concatenate([UNIT_TET, [[0.5, 0.5, 0.0]]])
    with pytest.raises(om.MeshError):
        om.orient(xyz, np.array([[0, 1, 2, 3], [0, 1, 2, 4]]))


def test_1d_pair():
    # S:51 [TRIVIAL]: L_x = 1, nodes at x=0 and x=1 -> one pair, N' = N - 1
    m = kuhn_voxel_mesh(np.ones((1, 1, 1), bool), 1.0)
    pm = om.PeriodicMesh(m.xyz, m.tets, (1, 0, 0), (1.0, 0, 0))
    assert pm.n_parents == 4
    # every x=1 node is the child of the x=0 node with the same (y,z)
    for i in range(8):
        p = pm.lca[i]
        assert np.allclose(m.xyz[i, 1:], m.xyz[p, 1:]) and m.xyz[p, 0] == 0.0


def test_corner_lca_seven_children():
    # P:96 "a corner point of a cubic unit cell with 3D PBC can have up to 7 children"
    m = kuhn_voxel_mesh(np.ones((1, 1, 1), bool), 1.0)
    pm = om.PeriodicMesh(m.xyz, m.tets, (1, 1, 1), (1.0, 1.0, 1.0))
    assert pm.n_parents == 1
    assert np.all(pm.lca == 0)
    assert len(pm.children_of()[0]) == 8          # the LCA + 7 children


def test_chain_merge():
    # P:96 "(i,j) and (j,k) ... are merged to (i,j) and (i,k)": nodes at x=0,1,2 with L=1
    m = kuhn_voxel_mesh(np.ones((2, 1, 1), bool), 1.0)
    pm = om.PeriodicMesh(m.xyz, m.tets, (1, 0, 0), (1.0, 0, 0))
    x = m.xyz[:, 0]
    for i in np.nonzero(x == 2.0)[0]:
        k = pm.lca[i]
        assert x[k] == 0.0 and np.allclose(m.xyz[k, 1:], m.xyz[i, 1:])
    assert pm.n_parents == 4                       # 12 nodes, chains of 3 copies
    # idempotence
    assert np.all(pm.lca[pm.lca] == pm.lca)


def test_ambiguous_pair_rejected():
    xyz = np.array([[0, 0, 0], [1, 0, 0], [1, 1e-12, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], float)
    tets = np.array([[0, 1, 3, 4], [1, 5, 3, 4]])
    with pytest.raises(om.MeshError):
        om.detect_pbc(xyz, tets, (1, 0, 0), (1.0, 0, 0), match_tol=1e-9)


def test_fold_examples():
    # S:69 [TRIVIAL]: x = 2.5, L = 2, r0 = 1 -> 0.5 (delta = -1)
    out, d = om.fold_manhattan(np.array([[2.5, 0, 0]]), (1, 0, 0), (2.0, 0, 0), r0=np.array([1.0, 0, 0]))
    assert out[0, 0] == 0.5 and d[0, 0] == -1
    # parallelogram with L_x = 2, D_x = 3 folds to D_x <= 2
    y = np.linspace(0, 1, 11)
    pts = np.concatenate([np.stack([s * 2.0 + y, y, 0 * y], 1) for s in np.linspace(0, 1, 11)])
    assert np.ptp(pts[:, 0]) == pytest.approx(3.0)
    out, d = om.fold_manhattan(pts, (1, 0, 0), (2.0, 0, 0))
    assert np.ptp(out[:, 0]) <= 2.0 + 1e-12
    # round trip (S:66 says bit-exact; x + dL - dL is exact only up to one rounding of
    # x + dL, so the pin is 1 ulp of the period)
    back = out - d * np.array([2.0, 0, 0])
    assert np.max(np.abs(back - pts)) <= 2.0 * np.finfo(float).eps * 2
    # non-protruding identity
    pts2 = np.array([[0.2, 0, 0], [0.9, 0, 0]])
    out2, d2 = om.fold_manhattan(pts2, (1, 0, 0), (2.0, 0, 0))
    assert np.all(d2 == 0)


def test_classification():
    c1 = make_config("C1", coarsen=5)
    pm = om.PeriodicMesh(c1["mesh"].xyz, c1["mesh"].tets, c1["periodic"], c1["lattice"])
    assert pm.classify() == (True, False)           # T-NP (P:340 cube)
    c4 = make_config("C4", coarsen=40)
    pm4 = om.PeriodicMesh(c4["mesh"].xyz, c4["mesh"].tets, c4["periodic"], c4["lattice"])
    assert pm4.classify() == (False, True)          # NT-P: corner sphere meshed whole


def test_wrap_rule():
    c1 = make_config("C1", coarsen=5)
    pm = om.PeriodicMesh(c1["mesh"].xyz, c1["mesh"].tets, c1["periodic"], c1["lattice"])
    w = pm.wrapped_parent_xyz()
    L = c1["lattice"][0]
    assert np.all(w >= 0) and np.all(w < L)
