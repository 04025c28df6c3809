"""GPU parity of the NEXT-4 complex Bloch field path (pmfem_build_bloch + pmfem_*_bloch through
the C ABI) against the oracle's Bloch AIM (oracle/bloch_heff.py, pinned exactly to the static
brute force on supercells in test_oracle_bloch_heff.py) on the same seeded complex inputs; the
bars are the static path's (rel L2 1e-5, per node 1e-4: the same fp32 operators and FFT, two of
each)."""
import numpy as np
import pytest

from helpers import SMALL, lib_context, bloch_oracle, bloch_k0, rel_l2, max_node_rel

pytestmark = pytest.mark.gpu

TOL = 1e-5
NODE_TOL = 1e-4
KEYS = [k for k in sorted(SMALL) if not k.startswith("N")]      # periodic configs only


@pytest.fixture(scope="module", params=KEYS)
def pair(request):
    key = request.param
    bm = bloch_oracle(key)
    ctx = lib_context(key, device=0)
    ctx.build_bloch(bloch_k0(key))
    return key, bm, ctx


def _run(ctx, fn, m_user, rank):
    import torch
    mi = m_user[rank]
    re = torch.tensor(np.ascontiguousarray(mi.real), dtype=torch.float32, device="cuda:0")
    im = torch.tensor(np.ascontiguousarray(mi.imag), dtype=torch.float32, device="cuda:0")
    Hr, Hi = getattr(ctx, fn)(re, im)
    torch.cuda.synchronize()
    out = np.zeros(m_user.shape, complex)
    out[rank] = Hr.double().cpu().numpy() + 1j * Hi.double().cpu().numpy()
    return out


def test_bloch_random(pair):
    key, bm, ctx = pair
    rank = ctx.internal_to_parent_rank()
    rng = np.random.default_rng(77)
    m = rng.standard_normal((bm.n_parents, 3)) + 1j * rng.standard_normal((bm.n_parents, 3))
    ref_ms = bm.demag(m, "aim")
    ref_ex = bm.exchange(m)
    H_ms = _run(ctx, "demag_bloch", m, rank)
    H_ex = _run(ctx, "exchange_bloch", m, rank)
    H = _run(ctx, "heff_bloch", m, rank)
    print(key, rel_l2(H_ms, ref_ms), max_node_rel(H_ms, ref_ms), rel_l2(H_ex, ref_ex))
    assert rel_l2(H_ms, ref_ms) <= TOL and max_node_rel(H_ms, ref_ms) <= NODE_TOL
    assert rel_l2(H_ex, ref_ex) <= TOL
    assert rel_l2(H, ref_ms + ref_ex) <= TOL and max_node_rel(H, ref_ms + ref_ex) <= NODE_TOL


def test_bloch_mode(pair):
    """A smooth Bloch mode: m = (0.9, 0.4 e^{-j k0.r}, 0.4 j e^{-j k0.r})."""
    key, bm, ctx = pair
    rank = ctx.internal_to_parent_rank()
    w = np.exp(-1j * (bm.r @ bm.k3))
    m = np.stack([np.full(bm.n_parents, 0.9 + 0j), 0.4 * w, 0.4j * w], 1)
    ref = bm.heff(m, "aim")
    H = _run(ctx, "heff_bloch", m, rank)
    assert rel_l2(H, ref) <= TOL and max_node_rel(H, ref) <= NODE_TOL


def test_bloch_linear_and_static_unaffected(pair):
    """Linearity in the complex amplitude (H(c m) = c H(m), c complex) and the static path still
    evaluates after a Bloch build."""
    key, bm, ctx = pair
    import torch
    rank = ctx.internal_to_parent_rank()
    rng = np.random.default_rng(5)
    m = rng.standard_normal((bm.n_parents, 3)) + 1j * rng.standard_normal((bm.n_parents, 3))
    c = 0.6 - 0.8j
    Ha = _run(ctx, "heff_bloch", m, rank)
    Hb = _run(ctx, "heff_bloch", c * m, rank)
    assert rel_l2(Hb, c * Ha) <= 1e-5
    ctx.build_pgf()
    md = torch.tensor(np.ones((bm.n_parents, 3)) / np.sqrt(3), dtype=torch.float32, device="cuda:0")
    H = ctx.exchange(md)
    torch.cuda.synchronize()
    assert float(H.abs().max()) == 0.0
