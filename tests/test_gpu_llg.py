"""GPU LLG RK4 (pmfem_llg_rk4, NEXT-2) vs the oracle integrator (oracle/llg.py) and the macrospin
closed form.  fp32 state: relative L2 of m after a few steps <= 1e-5."""
import numpy as np
import pytest

from helpers import oracle_model, lib_context, rel_l2
from oracle import llg
from synth import m_uniform

pytestmark = pytest.mark.gpu


def _dev(ctx, m_user, rank):
    import torch
    return torch.tensor(m_user[rank], dtype=torch.float32, device="cuda:0")


def _user(ctx, t, rank, n):
    out = np.zeros((n, 3))
    out[rank] = t.double().cpu().numpy()
    return out


@pytest.mark.parametrize("stream", ["default", "graph"])
def test_macrospin_filled_cell(stream):
    # filled 3D-periodic cell, uniform m: H_ex = H_ms = 0, every node is a macrospin in H_ap
    import torch
    ctx = lib_context("C1r0", device=0)
    ctx.build_pgf()
    n = ctx.n_parents
    rank = ctx.internal_to_parent_rank()
    H0, alpha = 2000.0, 0.05
    th0 = 0.6
    m0 = np.tile(llg.macrospin(th0, 0.0, 0.0, H0, alpha), (n, 1))
    period = 2 * np.pi * (1 + alpha ** 2) / (llg.GAMMA * H0)
    steps, dt = 400, 2 * period / 400
    s = torch.cuda.Stream() if stream == "graph" else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        m = _dev(ctx, m0, rank)
        ctx.llg_rk4(m, steps // 2, dt, alpha, H_applied=(0, 0, H0))
        ctx.llg_rk4(m, steps - steps // 2, dt, alpha, H_applied=(0, 0, H0))   # graph replay path
        s.synchronize()
    got = _user(ctx, m, rank, n)
    ref = llg.macrospin(th0, 0.0, steps * dt, H0, alpha)
    assert np.abs(got - ref[None, :]).max() < 2e-5


def test_rk4_parity_with_oracle():
    import torch
    key = "C5p2"
    om = oracle_model(key)
    ctx = lib_context(key, device=0)
    ctx.build_pgf()
    rank = ctx.internal_to_parent_rank()
    x = om.xw
    L = om.lattice[0]
    th = 0.5 + 0.3 * np.sin(2 * np.pi * x[:, 0] / L)
    m0 = np.stack([np.cos(th), np.sin(th) * np.cos(4 * np.pi * x[:, 0] / L),
                   np.sin(th) * np.sin(4 * np.pi * x[:, 0] / L)], 1)
    alpha, dt, steps, Hap = 0.02, 2e-14, 5, (0.0, 50.0, 0.0)
    m_ref = m0.copy()
    for _ in range(steps):
        m_ref = llg.rk4_step(lambda v: om.heff(v, "aim"), m_ref, dt, alpha, Hap)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        m = _dev(ctx, m0, rank)
        ctx.llg_rk4(m, steps, dt, alpha, H_applied=Hap)
        s.synchronize()
    got = _user(ctx, m, rank, om.n_parents)
    # the change over the run carries the fp32 rounding of m (~6e-8) relative to |dm| (~1e-3)
    assert rel_l2(got - m0, m_ref - m0) <= 1e-3
    assert rel_l2(got, m_ref) <= 1e-6
    assert np.abs(np.linalg.norm(got, axis=1) - 1).max() < 1e-6


@pytest.mark.parametrize("kind,K,axis", [(1, 3e5, (0.2, 0.3, 0.93)), (2, -2e5, (0, 0, 1))])
def test_rk4_anisotropy_parity(kind, K, axis):
    """pmfem_set_anisotropy (NEXT-2: uniaxial / cubic H_an of Eq. heff) in the RK4 stages vs
    the oracle's anisotropy_field in its RK4 (same parity bar as test_rk4_parity_with_oracle)."""
    import torch
    key = "C5p2"
    om = oracle_model(key)
    ctx = lib_context(key, device=0)
    ctx.build_pgf()
    ctx.set_anisotropy(kind, K, axis)
    rank = ctx.internal_to_parent_rank()
    x = om.xw
    L = om.lattice[0]
    th = 0.7 + 0.3 * np.sin(2 * np.pi * x[:, 0] / L)
    m0 = np.stack([np.cos(th), np.sin(th) * np.cos(2 * np.pi * x[:, 0] / L),
                   np.sin(th) * np.sin(2 * np.pi * x[:, 0] / L)], 1)
    alpha, dt, steps = 0.05, 2e-14, 5
    Ms = 637.0
    m_ref = m0.copy()
    for _ in range(steps):
        m_ref = llg.rk4_step(lambda v: om.heff(v, "aim"), m_ref, dt, alpha, anis=(kind, K, Ms, axis))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        m = _dev(ctx, m0, rank)
        ctx.llg_rk4(m, steps, dt, alpha)
        s.synchronize()
    got = _user(ctx, m, rank, om.n_parents)
    assert rel_l2(got - m0, m_ref - m0) <= 1e-3
    assert rel_l2(got, m_ref) <= 1e-6


def test_am2_fixed_step_parity():
    """pmfem_llg_am2 at a fixed step (tol = inf, dt_max = dt) vs the oracle's am2_integrate: the
    same AB2 predictor / AM2 corrector sequence."""
    import torch
    key = "C5p2"
    om = oracle_model(key)
    ctx = lib_context(key, device=0)
    ctx.build_pgf()
    rank = ctx.internal_to_parent_rank()
    x = om.xw
    L = om.lattice[0]
    th = 0.5 + 0.3 * np.sin(2 * np.pi * x[:, 0] / L)
    m0 = np.stack([np.cos(th), np.sin(th) * np.cos(4 * np.pi * x[:, 0] / L),
                   np.sin(th) * np.sin(4 * np.pi * x[:, 0] / L)], 1)
    alpha, dt, n, Hap = 0.02, 2e-14, 6, (0.0, 50.0, 0.0)
    m_ref, acc, rej = llg.am2_integrate(lambda v: om.heff(v, "aim"), m0, n * dt, dt, np.inf, alpha, Hap, dt_max=dt)
    assert acc == n
    with torch.cuda.stream(torch.cuda.Stream()):
        m = _dev(ctx, m0, rank)
        a, r = ctx.llg_am2(m, n * dt, dt, 1e30, alpha, H_applied=Hap, dt_max=dt)
        torch.cuda.synchronize()
    assert a == n and r == 0
    got = _user(ctx, m, rank, om.n_parents)
    assert rel_l2(got - m0, m_ref - m0) <= 1e-3
    assert rel_l2(got, m_ref) <= 1e-6


def test_am2_adaptive_macrospin():
    """Adaptive AM2 on the filled 3D-periodic cell (every node a macrospin in H_ap): the result
    matches the macrospin closed form to the tolerance level, with step-size control active."""
    import torch
    ctx = lib_context("C1r0", device=0)
    ctx.build_pgf()
    n = ctx.n_parents
    rank = ctx.internal_to_parent_rank()
    H0, alpha, th0 = 1500.0, 0.05, 0.8
    period = 2 * np.pi * (1 + alpha ** 2) / (llg.GAMMA * H0)
    m0 = np.tile(llg.macrospin(th0, 0.0, 0.0, H0, alpha), (n, 1))
    with torch.cuda.stream(torch.cuda.Stream()):
        m = _dev(ctx, m0, rank)
        a, r = ctx.llg_am2(m, period, period / 200, 1e-6, alpha, H_applied=(0, 0, H0))
        torch.cuda.synchronize()
    got = _user(ctx, m, rank, n)
    ref = llg.macrospin(th0, 0.0, period, H0, alpha)
    assert a > 20
    assert np.abs(got - ref[None, :]).max() < 2e-4


@pytest.mark.parametrize("theta", [np.pi / 2, 0.0])
def test_kalinikos_dispersion(theta):
    """Spin waves in a continuous 2D-periodic Permalloy film: a small standing wave
    of wavelength 200 nm (the cell) on the uniform state precesses, undamped, at the Kalinikos-Slavin
    frequency of Eq. sw_disp (oracle/llg.kalinikos_omega, exact P) for k perpendicular (theta =
    90 deg) and parallel (theta = 0) to M.  Frequency from the zero crossings of the mode amplitude
    over ~3 periods; the bar (3 %) covers the mesh (h = 2.5 nm vs l_ex = 7.4 nm), the lowest-mode
    approximation of the theory and the AIM error."""
    import torch
    from synth import make_config
    from paper_2409_13958_b200 import Context
    cfg = make_config("K1")
    mesh = cfg["mesh"]
    ctx = Context(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"],
                  Aex=cfg["Aex"], order=2, rer_scale=3.0, z0_ring=1, device=0)
    ctx.build_pgf()
    n = ctx.n_parents
    rank = ctx.internal_to_parent_rank()
    parents = ctx.export("parent")
    x = mesh.xyz[parents]
    L = cfg["lattice"][0]
    k = 2 * np.pi / L
    d = 10e-7
    m0dir = np.array([0.0, 1.0, 0.0]) if theta > 0 else np.array([1.0, 0.0, 0.0])   # k along x
    eps = 0.01
    m0 = np.tile(m0dir, (n, 1))
    m0[:, 2] = eps * np.cos(k * x[:, 0])
    m0 /= np.linalg.norm(m0, axis=1, keepdims=True)
    w_th = llg.kalinikos_omega(k, d, theta, cfg["Ms"], cfg["Aex"])
    T = 2 * np.pi / w_th
    dt = 5e-14
    chunk = max(1, int(round(T / dt / 40)))
    nrec = int(3.2 * T / (chunk * dt))
    cosw = np.cos(k * x[:, 0])
    amp = []
    with torch.cuda.stream(torch.cuda.Stream()):
        m = _dev(ctx, m0, rank)
        for _ in range(nrec + 1):
            mu = _user(ctx, m, rank, n)
            amp.append(float((mu[:, 2] * cosw).sum() / (cosw * cosw).sum()))
            ctx.llg_rk4(m, chunk, dt, 0.0)
        torch.cuda.synchronize()
    a = np.array(amp)
    t = np.arange(a.size) * chunk * dt
    zc = [t[i] - a[i] * (t[i + 1] - t[i]) / (a[i + 1] - a[i]) for i in range(a.size - 1) if a[i] * a[i + 1] < 0]
    assert len(zc) >= 4
    w_num = np.pi / np.mean(np.diff(zc))
    print("theta %.2f: omega numeric %.4e, Kalinikos %.4e (rel %.3f)" % (theta, w_num, w_th, w_num / w_th - 1))
    assert abs(w_num / w_th - 1) < 0.03
