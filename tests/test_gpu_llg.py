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
