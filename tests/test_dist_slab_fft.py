"""Slab-decomposed FFT convolution on CPU with world_size-2 gloo processes:
each rank holds its z slab of the anterpolated grid -- the planes [Z_r, Z_r+1) of the library's
row partition (pmfem_export "dist_planes", variable thickness balancing the rows) -- transforms
x and y, sends rank p the k0 columns the library assigns it ("slab_kranges"), transforms z,
multiplies by the spectrum, transforms back, returns the blocks and finishes y and x -- the
same block layout the NCCL path of device.cu sends ([nz_r][P1][H_p] blocks landing at plane
offset Z_r of the receiver's [P2][P1][H_p] x slab).  The gathered result must equal the
single-process FFT convolution (circular on periodic axes, zero-padded on the others)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import config


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _alltoall(blocks, rank, world):
    """blocks[p] (numpy complex) -> list of the blocks every rank sent to me."""
    out = [None] * world
    reqs = []
    recv = {}
    for p in range(world):
        if p == rank:
            out[p] = blocks[p]
            continue
        sh = torch.tensor(blocks[p].shape, dtype=torch.int64)
        dist.send(sh, p) if rank < p else None
        r = torch.empty(3, dtype=torch.int64)
        dist.recv(r, p)
        if rank > p:
            dist.send(sh, p)
        buf = torch.empty(tuple(r.tolist()) + (2,), dtype=torch.float64)
        recv[p] = buf
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(
            np.stack([blocks[p].real, blocks[p].imag], -1))), p))
        reqs.append(dist.irecv(buf, p))
    for q in reqs:
        q.wait()
    for p, buf in recv.items():
        b = buf.numpy()
        out[p] = b[..., 0] + 1j * b[..., 1]
    return out


def _worker(rank, world, port, key, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2409_13958_b200 import Context
    cfg, spec = config(key)
    m = cfg["mesh"]
    ctx = Context(m.xyz, m.tets, cfg["periodic"], cfg["lattice"], spec["grid"], Ms=cfg["Ms"], Aex=cfg["Aex"],
                  order=spec["order"], rer_scale=spec["s"], z0_ring=spec["ring"], device=-1, rank=rank,
                  world=world)
    n0, n1, n2 = ctx.query()["grid"]                          # internal frame (slab axis = z)
    P = ctx.query()["fft"]
    P0, P1, P2 = P
    H0 = P0 // 2 + 1
    kr = ctx.export("slab_kranges").reshape(world, 2)
    assert kr[:, 1].sum() == H0 and kr[0, 0] == 0 and np.all(kr[1:, 0] == np.cumsum(kr[:, 1])[:-1])
    rng = np.random.default_rng(5)
    Q = rng.standard_normal((n2, n1, n0))                      # [z][y][x], same on every rank
    G = rng.standard_normal((P2, P1, H0))                      # a real spectrum [k2][k1][k0]
    Z = ctx.export("dist_planes")
    assert Z[0] == 0 and Z[-1] == n2 and np.all(np.diff(Z) > 0)
    # z slab: X (real -> half spectrum, padded to P0) and Y (padded to P1)
    Cz = np.fft.rfft(Q[Z[rank]:Z[rank + 1]], n=P0, axis=2)
    Cz = np.fft.fft(Cz, n=P1, axis=1)                          # [nzl][P1][H0]
    blocks = [Cz[:, :, kr[p, 0]:kr[p, 0] + kr[p, 1]] for p in range(world)]
    got = _alltoall(blocks, rank, world)
    h, hn = kr[rank]
    Cx = np.zeros((P2, P1, hn), complex)                       # x slab: planes Z_q.. from rank q
    for q in range(world):
        Cx[Z[q]:Z[q + 1]] = got[q]
    Cx = np.fft.ifft(np.fft.fft(Cx, axis=0) * G[:, :, h:h + hn], axis=0)
    back = _alltoall([Cx[Z[q]:Z[q + 1]] for q in range(world)], rank, world)
    for p in range(world):
        Cz[:, :, kr[p, 0]:kr[p, 0] + kr[p, 1]] = back[p]
    Us = np.fft.irfft(np.fft.ifft(Cz, axis=1)[:, :n1], n=P0, axis=2)[:, :, :n0]
    # reference on the full grid
    ref = np.fft.irfftn(np.fft.fftn(np.fft.rfft(Q, n=P0, axis=2), s=(P2, P1), axes=(0, 1)) * G,
                        s=(P2, P1, P0), axes=(0, 1, 2))[:, :n1, :n0]
    out[rank] = float(np.abs(Us - ref[Z[rank]:Z[rank + 1]]).max() / np.abs(ref).max())
    dist.destroy_process_group()


@pytest.mark.parametrize("key", ["C2p2", "C4p3", "C5p2"])
def test_slab_fft_two_ranks(key):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), key, out), nprocs=world, join=True)
    assert max(out.values()) < 1e-12
