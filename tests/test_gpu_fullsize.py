"""GPU parity at BASELINE.json's full size, in the launch configuration bench.py times (C2,
bench.DEFAULTS AIM parameters): H_eff at sampled nodes against the oracle computed for those
nodes only (the oracle's Z0 and C_box rows are built for the samples' 1-rings; the grid part
and the local operators are global), plus full-field properties that hold at any size."""
import numpy as np
import pytest

from oracle import fem, mesh as omesh
from oracle.heff import OracleModel
from synth import make_config, m_random, m_uniform
from helpers import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    import bench
    from paper_2409_13958_b200 import Context
    aim = bench.DEFAULTS["C2"]
    cfg = make_config("C2")
    mesh = cfg["mesh"]
    ctx = Context(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"], Aex=cfg["Aex"],
                  device=0, **aim)
    ctx.build_pgf()
    return cfg, aim, ctx


def _gpu(ctx, fn, m_user, rank):
    import torch
    md = torch.tensor(m_user[rank], dtype=torch.float32, device="cuda:0")
    H = getattr(ctx, fn)(md)
    torch.cuda.synchronize()
    out = np.zeros_like(m_user)
    out[rank] = H.double().cpu().numpy()
    return out


def test_fullsize_sampled_heff(c2):
    cfg, aim, ctx = c2
    mesh = cfg["mesh"]
    pm = omesh.PeriodicMesh(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"])
    ops = fem.assemble(pm, cfg["Ms"], cfg["Aex"])
    rng = np.random.default_rng(2024)
    x = pm.xyz[pm.parent]
    L = cfg["lattice"][0]
    r = np.hypot(x[:, 0] - L / 2, x[:, 1] - L / 2)
    # samples: random interior + hole rim + periodic-face nodes + top/bottom surface
    cand = [rng.choice(pm.n_parents, 8, replace=False),
            np.argsort(r)[:4], np.nonzero(np.isclose(x[:, 0], 0.0))[0][:3],
            np.nonzero(np.isclose(x[:, 2], x[:, 2].max()))[0][:3]]
    samples = np.unique(np.concatenate(cand))
    S = ops["S"].tocsr()
    rows = np.unique(np.concatenate([S.indices[S.indptr[n]:S.indptr[n + 1]] for n in samples] + [samples]))
    om = OracleModel(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"],
                     Aex=cfg["Aex"], rows=rows, **{"order": aim["order"], "rer_scale": aim["rer_scale"],
                                                   "z0_ring": aim["z0_ring"]})
    rank = ctx.internal_to_parent_rank()
    m = m_random(pm.n_parents, seed=77)
    H = _gpu(ctx, "heff", m, rank)
    u = om.potential_aim(m)
    ref = fem.gradient_field(om.ops, u) + om.exchange(m)
    err = rel_l2(H[samples], ref[samples])
    print("full-size C2 sampled rel L2 = %.3e over %d nodes" % (err, samples.size))
    assert err <= 1e-5
    # exchange field: complete (every node) vs the oracle
    assert rel_l2(_gpu(ctx, "exchange", m, rank), om.exchange(m)) <= 1e-5


def test_fullsize_properties(c2):
    cfg, aim, ctx = c2
    Np = ctx.n_parents
    rank = ctx.internal_to_parent_rank()
    # uniform m: exchange exactly zero; linearity of H_ms
    assert np.abs(_gpu(ctx, "exchange", m_uniform(Np, (0.6, 0.0, 0.8)), rank)).max() == 0.0
    a = m_random(Np, seed=1)
    b = m_random(Np, seed=2)
    Ha = _gpu(ctx, "demag", a, rank)
    Hb = _gpu(ctx, "demag", b, rank)
    assert rel_l2(_gpu(ctx, "demag", a + b, rank), Ha + Hb) <= 1e-5
    # 2D film: uniform in-plane m sees no film-face charge; only the hole rim is charged, so the
    # volume-averaged in-plane demag factor is small and positive, N_zz for m_z is near 1
    Hz = _gpu(ctx, "demag", m_uniform(Np, (0, 0, 1.0)), rank)
    Nzz = -Hz[:, 2].mean() / (4 * np.pi * cfg["Ms"])
    assert 0.9 < Nzz < 1.05
