"""Oracle end-to-end closed forms (BASELINE.json north_star; SURVEY.md 8(c) "End-to-end physics").

  filled 3D-periodic cell, uniform m      -> H_ms = 0                  (no charges)
  2D-periodic film, uniform in-plane m   -> H_ms = 0  (N_xx = N_yy = 0)
  2D-periodic film, out-of-plane m       -> volume-averaged N_zz = 1
  1D-periodic square wire, axial m       -> H_ms = 0  (N_xx = 0)
  1D-periodic square wire, transverse m  -> N_yy + N_zz = 1, N_yy = N_zz = 1/2 (square symmetry)
N is defined by  <H> = -4 pi N <M>, volume-weighted over nodes (lumped volumes).
The exact-by-symmetry parts must hold to roundoff; N_zz and N_yy carry the O(h) error of
the point-charge + Z0 discretisation.
"""
import numpy as np
import pytest

from oracle.heff import OracleModel
from synth import kuhn_voxel_mesh

MS = 637.0


def _model(mask, h, periodic, wrap, grid, ring=1, build_aim=True, s=2.0):
    m = kuhn_voxel_mesh(mask, h, wrap=wrap, jitter=0.1, seed=11)
    L = tuple(mask.shape[a] * h if periodic[a] else 0.0 for a in range(3))
    return OracleModel(m.xyz, m.tets, periodic, L, grid, Ms=MS, Aex=1.4e-6, z0_ring=ring,
                       build_aim=build_aim, rer_scale=s)


def _navg(mo, H, direction):
    Vt = mo.ops["Vt"]
    Hav = (Vt[:, None] * H).sum(axis=0) / Vt.sum()
    return -Hav / (4 * np.pi * MS)


def test_filled_cell_uniform_zero():
    mo = _model(np.ones((4, 4, 4), bool), 1e-6, (1, 1, 1), (True,) * 3, (10, 10, 10), ring=0)
    m = np.tile([0.36, 0.48, 0.8], (mo.n_parents, 1))
    for method in ("aim", "bf"):
        H = mo.demag(m, method)
        assert np.abs(H).max() < 1e-9 * 4 * np.pi * MS


@pytest.fixture(scope="module")
def film():
    # 8 x 8 x 4 cells, T-PBC in x and y, h = 2.5 nm
    return _model(np.ones((8, 8, 4), bool), 2.5e-7, (1, 1, 0), (True, True, False), (16, 16, 5))


def test_film_in_plane_zero(film):
    m = np.tile([0.8, 0.6, 0.0], (film.n_parents, 1))
    for method in ("aim", "bf"):
        H = film.demag(m, method)
        assert np.abs(H).max() < 1e-9 * 4 * np.pi * MS


def test_film_out_of_plane_nzz(film):
    m = np.tile([0.0, 0.0, 1.0], (film.n_parents, 1))
    Hb = film.demag(m, "bf")
    N = _navg(film, Hb, 2)
    assert abs(N[0]) < 1e-9 and abs(N[1]) < 1e-9          # exact by symmetry
    assert N[2] == pytest.approx(1.0, abs=0.02)            # N_zz = 1, O(h/t) discretisation
    Ha = film.demag(m, "aim")
    assert _navg(film, Ha, 2)[2] == pytest.approx(1.0, abs=0.02)


@pytest.fixture(scope="module")
def wire():
    # square 4 x 4 section, 8 cells along the periodic x axis
    return _model(np.ones((8, 4, 4), bool), 2.5e-7, (1, 0, 0), (True, False, False), (16, 8, 8))


def test_wire_axial_zero(wire):
    m = np.tile([1.0, 0.0, 0.0], (wire.n_parents, 1))
    H = wire.demag(m, "bf")
    assert np.abs(H).max() < 1e-9 * 4 * np.pi * MS


def test_wire_transverse_half():
    # N_yy = N_zz by square symmetry; tr N -> 1 with O(h) discretisation error (surface-node
    # point-charge error): Richardson-extrapolate from 4 and 6 cells across.
    tr = []
    for n in (4, 6):
        w = _model(np.ones((8, n, n), bool), 1e-6 / n, (1, 0, 0), (True, False, False),
                   (16, 2 * n, 2 * n), build_aim=False)
        Ny = _navg(w, w.demag(np.tile([0.0, 1.0, 0.0], (w.n_parents, 1)), "bf"), 1)[1]
        Nz = _navg(w, w.demag(np.tile([0.0, 0.0, 1.0], (w.n_parents, 1)), "bf"), 2)[2]
        assert Ny == pytest.approx(Nz, abs=1e-3)
        tr.append(Ny + Nz)
    assert abs(1 - tr[1]) < abs(1 - tr[0]) < 0.06
    extrap = tr[1] + (tr[1] - tr[0]) / (1 / 4 - 1 / 6) / 6
    assert extrap == pytest.approx(1.0, abs=0.02)
