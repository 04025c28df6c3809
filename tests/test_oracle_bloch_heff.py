"""Oracle pins of the Bloch field path (NEXT-4, oracle/bloch_heff.py; reading R27).

1. Supercell identity (exact).  For k0 = 2 pi j / (M L) along a periodic axis, a Bloch mode of
   the unit cell, m(r + R) = exp(-j k0.R) m(r), IS an ordinary field of the M-cell supercell
   (period M L; the supercell's own Bloch phase is exp(-j k0 M L) = 1), and the static kernel of
   the supercell summed against it reproduces G_p(r; k0) (Eq. 2: the phases of the
   cells c = 0..M-1 combine the M L-periodic sums into the L-periodic Bloch sum; the static
   zero mode drops out because sum_c exp(-j k0 c L) = 0).  So the Bloch brute force on the unit
   cell equals the static brute force (oracle.heff, pinned in test_oracle_bf.py /
   test_oracle_pgf.py / test_oracle_fem.py / test_oracle_z0.py) on the supercell mesh with the
   phased m, node by node -- which fixes every phase of the folded operators, of Z0 and of the
   Bloch kernel (a sign error in any of them fails: with k0 -> -k0 the demag differs by 12 %).
   M = 3 gives genuinely complex phases; the cases span 1D (x and z), 2D and 3D lattices.
2. AIM vs brute force (the approximation level): <= 1e-3 at p = 2, s = 4 on a
   tiny strip, and the error falls as the precorrected zone grows.
"""
import functools

import numpy as np
import pytest
from scipy.spatial import cKDTree

from oracle.bloch_heff import BlochModel
from oracle.heff import OracleModel
from synth import make_config


def supercell(xyz, tets, axis, L, M):
    """M translated copies of the mesh along `axis`, coincident nodes merged.  Returns the
    supercell nodes, tets and for each supercell node the index of one original copy
    (copy c of unit node u has index c * N + u)."""
    N = xyz.shape[0]
    X = np.concatenate([xyz + np.eye(3)[axis] * (c * L) for c in range(M)])
    T = np.concatenate([tets + c * N for c in range(M)])
    h = np.min(np.linalg.norm(xyz[tets[:, 1]] - xyz[tets[:, 0]], axis=1))
    par = np.arange(X.shape[0])
    for i, j in sorted(cKDTree(X).query_pairs(1e-6 * h)):
        a, b = min(par[i], par[j]), max(par[i], par[j])
        par[par == b] = a
    keep = np.unique(par)
    new = np.full(X.shape[0], -1)
    new[keep] = np.arange(keep.size)
    return X[keep], new[par][T], keep


def _m(n, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))


@pytest.mark.parametrize("name,coarsen,M,axis", [("C5", 40, 3, 0), ("C2", 20, 3, 0), ("R1", 4, 2, 2),
                                                 ("C1", 3.4, 3, 1)])
def test_supercell_identity(name, coarsen, M, axis):
    cfg = make_config(name, coarsen=coarsen)
    mesh = cfg["mesh"]
    L = cfg["lattice"][axis]
    k3 = np.zeros(3)
    k3[axis] = 2 * np.pi / (M * L)
    bm = BlochModel(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], k3, Ms=cfg["Ms"],
                    Aex=cfg["Aex"], nquad=8, build_aim=False)
    m = _m(bm.n_parents, 1)
    Hb = bm.demag(m, "bf")
    Hx = bm.exchange(m)
    Xs, Ts, orig = supercell(mesh.xyz, mesh.tets, axis, L, M)
    lat = list(cfg["lattice"])
    lat[axis] = M * L
    om = OracleModel(Xs, Ts, cfg["periodic"], lat, cfg["grid"], Ms=cfg["Ms"], Aex=cfg["Aex"], nquad=8,
                     build_aim=False)
    assert om.n_parents == M * bm.n_parents
    N = mesh.xyz.shape[0]
    u = orig[om.pm.parent] % N                      # unit node of each supercell parent
    pu = bm.pm.pid[u]
    R = Xs[om.pm.parent] - bm.r[pu]                 # lattice vector to the unit-cell parent
    ph = np.exp(-1j * (R @ k3))
    msc = ph[:, None] * m[pu]
    Hs = om.demag(msc.real, "bf") + 1j * om.demag(msc.imag, "bf")
    Hxs = om.exchange(msc.real) + 1j * om.exchange(msc.imag)
    for got, ref in ((Hs, ph[:, None] * Hb[pu]), (Hxs, ph[:, None] * Hx[pu])):
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@functools.lru_cache(maxsize=None)
def _model(name, coarsen, p, s):
    cfg = make_config(name, coarsen=coarsen)
    mesh = cfg["mesh"]
    ax = [a for a in range(3) if cfg["periodic"][a]]
    k3 = np.zeros(3)
    for i, a in enumerate(ax):
        k3[a] = 2 * np.pi / cfg["lattice"][a] * (0.3, 0.15, 0.1)[i]
    bm = BlochModel(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], k3, Ms=cfg["Ms"],
                    Aex=cfg["Aex"], nquad=8, order=p, rer_scale=s, z0_ring=0)
    # a random field and a smooth Bloch mode (uniform m_x plus a transverse wave at k0)
    w = np.exp(-1j * (bm.r @ k3))
    smooth = np.stack([np.full(bm.n_parents, 0.9), 0.4 * w, 0.4j * w], 1)
    return bm, {"random": _m(bm.n_parents, 3), "smooth": smooth}


def _err(name, coarsen, p, s):
    bm, fields = _model(name, coarsen, p, s)
    out = {}
    for nm, f in fields.items():
        Ha, Hb = bm.demag(f, "aim"), bm.demag(f, "bf")
        out[nm] = float(np.linalg.norm(Ha - Hb) / np.linalg.norm(Hb))
    return out


def test_bloch_aim_matches_bruteforce_1e3():
    e = _err("C5", 40, 2, 4.0)
    print(e)
    assert max(e.values()) <= 1e-3


@pytest.mark.parametrize("name,coarsen", [("C2", 20), ("C5", 40)])
def test_bloch_aim_error_controllable(name, coarsen):
    e2 = _err(name, coarsen, 1, 2.0)
    e3 = _err(name, coarsen, 1, 3.0)
    print(name, e2, e3)
    for nm in e2:
        assert e3[nm] < e2[nm]
    assert max(e3.values()) < 3e-2
