"""Test helpers: build the oracle and the library context on the same seeded inputs."""
import functools

import numpy as np

from oracle.heff import OracleModel
from synth import make_config, kuhn_voxel_mesh

# small configs (name, kwargs) used by the parity tests; each spans several FFT tiles and has
# a ragged tail (grid and node counts are not multiples of the CUDA tile sizes)
SMALL = {
    "C1r0": dict(cfg=("C1", 2), grid=(16, 16, 16), order=1, s=2.0, ring=0),
    "C1r1": dict(cfg=("C1", 2), grid=(16, 16, 16), order=1, s=2.0, ring=1),
    "C2p2": dict(cfg=("C2", 8), grid=(32, 32, 4), order=2, s=2.0, ring=1),
    "C3p1": dict(cfg=("C3", 12), grid=(64, 8, 8), order=1, s=2.0, ring=0),
    "C4p3": dict(cfg=("C4", 40), grid=(16, 16, 16), order=3, s=1.5, ring=0),
    "C5p2": dict(cfg=("C5", 16), grid=(128, 8, 4), order=2, s=2.0, ring=0),
    # non-periodic mode (NEXT-3): isolated cube, free-space kernel, 2N padding on every axis
    "N1p2": dict(cfg=("N1", 2), grid=(16, 16, 16), order=2, s=2.0, ring=1),
    # other periodic axes: the z-periodic rod of P:277 and a y-periodic strip
    "R1p2": dict(cfg=("R1", 2), grid=(8, 8, 16), order=2, s=1.5, ring=1),
    "Y1p2": dict(cfg=("Y1", 2), grid=(8, 32, 4), order=2, s=2.0, ring=0),
}


def config(key):
    spec = SMALL[key]
    name, coarsen = spec["cfg"]
    cfg = make_config(name, coarsen=coarsen)
    return cfg, spec


@functools.lru_cache(maxsize=None)
def oracle_model(key):
    """The oracle for a SMALL config (cached: the model is read-only for the tests)."""
    cfg, spec = config(key)
    m = cfg["mesh"]
    return OracleModel(m.xyz, m.tets, cfg["periodic"], cfg["lattice"], spec["grid"], Ms=cfg["Ms"],
                       Aex=cfg["Aex"], order=spec["order"], rer_scale=spec["s"], z0_ring=spec["ring"])


def lib_context(key, device):
    from paper_2409_13958_b200 import Context
    cfg, spec = config(key)
    m = cfg["mesh"]
    return Context(m.xyz, m.tets, cfg["periodic"], cfg["lattice"], spec["grid"], Ms=cfg["Ms"],
                   Aex=cfg["Aex"], order=spec["order"], rer_scale=spec["s"], z0_ring=spec["ring"],
                   device=device)


def dense(ctx, prefix, nv, n):
    rp = ctx.export(prefix + "_rowptr")
    col = ctx.export(prefix + "_col")
    val = ctx.export(prefix + "_val").reshape(-1, nv)
    A = np.zeros((n, n, nv))
    rows = np.repeat(np.arange(n), np.diff(rp))
    np.add.at(A, (rows, col), val)
    return A


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def max_node_rel(a, b):
    """Per-node bound: max_n |a_n - b_n| / rms_n |b_n| (rows = nodes)."""
    a = np.asarray(a).reshape(len(a), -1)
    b = np.asarray(b).reshape(len(b), -1)
    return float(np.max(np.linalg.norm(a - b, axis=1)) / np.sqrt(np.mean(np.sum(np.abs(b) ** 2, axis=1))))


# NEXT-4: Bloch wave vectors of the parity tests (rad/cm, off the reciprocal lattice, generic
# fractions of the reciprocal vectors so no phase is real)
def bloch_k0(key):
    cfg, _ = config(key)
    out = np.zeros(3)
    fr = iter((0.3, 0.2, 0.1))
    for a in range(3):
        if cfg["periodic"][a]:
            out[a] = 2 * np.pi / cfg["lattice"][a] * next(fr)
    return out


@functools.lru_cache(maxsize=None)
def bloch_oracle(key):
    from oracle.bloch_heff import BlochModel
    cfg, spec = config(key)
    m = cfg["mesh"]
    return BlochModel(m.xyz, m.tets, cfg["periodic"], cfg["lattice"], spec["grid"], bloch_k0(key), Ms=cfg["Ms"],
                      Aex=cfg["Aex"], order=spec["order"], rer_scale=spec["s"], z0_ring=spec["ring"])


def dense_c(ctx, prefix, nv, n):
    """Dense [n, n, nv] complex matrix of a complex CSR export (values interleaved re/im)."""
    rp = ctx.export(prefix + "_rowptr")
    col = ctx.export(prefix + "_col")
    v = ctx.export(prefix + "_val").reshape(-1, nv, 2)
    A = np.zeros((n, n, nv), complex)
    rows = np.repeat(np.arange(n), np.diff(rp))
    np.add.at(A, (rows, col), v[..., 0] + 1j * v[..., 1])
    return A
