"""Multi-GPU host logic on CPU: world_size-2 gloo processes build the library's distributed
plan (host-only contexts, pmfem_setup_dist with cuda_device = -1), exchange halos with
torch.distributed (gloo) exactly as the library does with NCCL (same index lists), and check
that every rank's rows of q = D m, u_loc = Z0 m, C_box q and G u computed from owned + halo
values equal the single-process products bit for bit.  The partition is slab-aligned
(SURVEY 8(e)): a rank owns the rows anchored in its z planes [Z_r, Z_r+1) (the FFT's z slab),
its q halo holds every row K2's stencils need below the slab, and its U ghost planes (the p
planes above the slab K4 reads) come from their owners."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import config


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _csr_internal(ctx, prefix, nv, perm, iperm):
    rp = ctx.export(prefix + "_rowptr")
    col = ctx.export(prefix + "_col")
    val = ctx.export(prefix + "_val").reshape(-1, nv)
    rows = []
    for i in range(len(perm)):
        r = perm[i]
        rows.append((iperm[col[rp[r]:rp[r + 1]]], val[rp[r]:rp[r + 1]]))
    return rows


def _worker(rank, world, port, key, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_2409_13958_b200 import Context
    cfg, spec = config(key)
    m = cfg["mesh"]
    ctx = Context(m.xyz, m.tets, cfg["periodic"], cfg["lattice"], spec["grid"], Ms=cfg["Ms"], Aex=cfg["Aex"],
                  order=spec["order"], rer_scale=spec["s"], z0_ring=spec["ring"], device=-1, rank=rank,
                  world=world)
    b = ctx.export("dist_bounds")
    lo, hi = int(b[rank]), int(b[rank + 1])
    perm = ctx.export("perm")
    Np = perm.size
    iperm = np.empty(Np, dtype=np.int64)
    iperm[perm] = np.arange(Np)
    plans = {}
    for k in "mqu":
        plans[k] = {"%s_%s" % (d, t): ctx.export("%s_%s_%s" % (d, k, t))
                    for d in ("send", "recv") for t in ("ptr", "idx")}
    # consistency: my send list to p == p's receive list from me
    allp = [None] * world
    dist.all_gather_object(allp, {k: {nm: plans[k][nm].tolist() for nm in plans[k]} for k in plans})
    ok = True
    fails = []
    for k in "mqu":
        for p in range(world):
            if p == rank:
                continue
            sp, si = np.array(allp[rank][k]["send_ptr"]), np.array(allp[rank][k]["send_idx"])
            rp, ri = np.array(allp[p][k]["recv_ptr"]), np.array(allp[p][k]["recv_idx"])
            ok &= np.array_equal(si[sp[p]:sp[p + 1]], ri[rp[rank]:rp[rank + 1]])
            if not ok and "lists" not in fails:
                fails.append("lists")

    def halo(k, v):
        """exchange owned rows of v into the full-length local copy (what device halo() does)."""
        P = plans[k]
        reqs = []
        bufs = []
        for p in range(world):
            if p == rank:
                continue
            s0, s1 = P["send_ptr"][p], P["send_ptr"][p + 1]
            r0, r1 = P["recv_ptr"][p], P["recv_ptr"][p + 1]
            if s1 > s0:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(v[P["send_idx"][s0:s1]])), p))
            if r1 > r0:
                buf = torch.empty((r1 - r0,) + v.shape[1:], dtype=torch.float64)
                reqs.append(dist.irecv(buf, p))
                bufs.append((P["recv_idx"][r0:r1], buf))
        for r in reqs:
            r.wait()
        for idx, buf in bufs:
            v[idx] = buf.numpy()

    rng = np.random.default_rng(5)
    m_full = rng.normal(size=(Np, 3))
    q_full = rng.normal(size=Np)
    u_full = rng.normal(size=Np)
    ring1 = _csr_internal(ctx, "ring1", 7, perm, iperm)
    z0 = _csr_internal(ctx, "z0", 3, perm, iperm)
    cb = _csr_internal(ctx, "cbox", 1, perm, iperm)
    m_loc = np.full((Np, 3), np.nan); m_loc[lo:hi] = m_full[lo:hi]
    q_loc = np.full(Np, np.nan); q_loc[lo:hi] = q_full[lo:hi]
    u_loc = np.full(Np, np.nan); u_loc[lo:hi] = u_full[lo:hi]
    halo("m", m_loc)
    halo("q", q_loc)
    halo("u", u_loc)
    ok0 = ok
    for i in range(lo, hi):
        c, v = ring1[i]
        ok &= np.array_equal(v[:, 1:4] * (m_loc[c] - m_loc[i]), v[:, 1:4] * (m_full[c] - m_full[i]))
        ok &= np.array_equal(v[:, 4:7] * (u_loc[c] - u_loc[i])[:, None], v[:, 4:7] * (u_full[c] - u_full[i])[:, None])
        c, v = z0[i]
        ok &= np.array_equal(v * m_loc[c], v * m_full[c])
        c, v = cb[i]
        ok &= np.array_equal(v[:, 0] * q_loc[c], v[:, 0] * q_full[c])
    if ok0 and not ok:
        fails.append("products")
    # slab alignment: own rows are exactly those anchored in [Z_r, Z_r+1)
    Z = ctx.export("dist_planes")
    ap = ctx.export("axis_perm")                 # internal axis i = user axis ap[i] (slab axis -> z)
    n2 = spec["grid"][ap[2]]
    perz = cfg["periodic"][ap[2]]
    ok &= n2 == max(spec["grid"])
    az = ctx.export("stencil_s").reshape(-1, 3)[perm, 2]
    if perz:
        az = az % n2
    own = (az >= Z[rank]) & (az < Z[rank + 1])
    okp = bool(np.all(own[lo:hi])) and not bool(np.any(own[:lo])) and not bool(np.any(own[hi:]))
    ok &= okp
    if not okp:
        fails.append("slab rows")
    # K2 reads q of every row anchored in the p planes below the slab (halo), all present
    p_ = spec["order"]
    below = [(Z[rank] - d) % n2 if perz else Z[rank] - d for d in range(1, p_ + 1)]
    need = np.isin(az, [z for z in below if 0 <= z < n2])
    okq = bool(np.all(np.isfinite(q_loc[need])))
    ok &= okq
    if not okq:
        fails.append("K2 q halo")
    # U ghost planes: what I receive = the planes above my slab that K4's stencils reach
    g = ctx.export("dist_ghost").reshape(world, 8)
    got = set()
    for pp in range(world):
        for k in range(2):
            z0_, nz_ = g[pp, 4 + 2 * k], g[pp, 5 + 2 * k]
            got.update(range(int(z0_), int(z0_ + nz_)))
    want = set()
    for d in range(p_):
        z = Z[rank + 1] + d
        z = z % n2 if perz else z
        if z < n2 and not (Z[rank] <= z < Z[rank + 1]):
            want.add(int(z))
    ok &= got == want
    if got != want:
        fails.append("ghost %s vs %s" % (sorted(got), sorted(want)))
    allg = [None] * world
    dist.all_gather_object(allg, g.tolist())
    for pp in range(world):                      # my sends to pp == pp's receives from me
        ok &= all(allg[rank][pp][k] == allg[pp][rank][4 + k] for k in range(4))
    out[rank] = (bool(ok), lo, hi, int(sum(len(plans[k]["recv_idx"]) for k in plans)), fails)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("key", ["C1r1", "C3p1", "C5p2", "C2p2", "R1p2", "C4p3"])
def test_dist_plan_world2(key):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), key, out), nprocs=world, start_method="spawn")
    res = [out[r] for r in range(world)]
    assert all(r[0] for r in res), res
    # contiguous, covering partition
    assert res[0][1] == 0 and res[0][2] == res[1][1]
    assert res[0][3] > 0 and res[1][3] > 0           # real halos exist on both ranks
