"""Full-size AIM accuracy ("controllable error", "relative error level 1e-3"):
H_eff from the GPU path for several (p, s) against the oracle's brute force (exact PGF pair
sums, O12) at sampled nodes of the full BASELINE config.

    python scripts/calibrate_fullsize.py [--config C2] [--samples 12]

The GPU path equals the oracle AIM to ~1e-6 (tests/test_gpu_*), so this measures the AIM
discretisation error itself.  The brute force is evaluated only at the samples' 1-rings.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--samples", type=int, default=12)
    ap.add_argument("--settings", default="1,2;2,3;2,4;3,3;3,4")
    ap.add_argument("--ring", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2409_13958_b200 import Context
    from oracle import fem, mesh as omesh, z0 as oz0
    from oracle.pgf import PgfSpec, pgf_potential, pgf_self
    from synth import make_config, m_random

    cfg = make_config(a.config)
    mesh = cfg["mesh"]
    t0 = time.time()
    pm = omesh.PeriodicMesh(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"])
    ops = fem.assemble(pm, cfg["Ms"], cfg["Aex"])
    rng = np.random.default_rng(7)
    samples = np.sort(rng.choice(pm.n_parents, a.samples, replace=False))
    S = ops["S"].tocsr()
    rows = np.unique(np.concatenate([S.indices[S.indptr[n]:S.indptr[n + 1]] for n in samples] + [samples]))
    z0 = oz0.assemble_z0(pm, ops, np.full(pm.tets.shape[0], cfg["Ms"]), a.ring, rows=rows)
    m = m_random(pm.n_parents, seed=77)
    q = fem.charges(ops, m)
    xw = pm.wrapped_parent_xyz()
    lat = tuple(float(cfg["lattice"][i]) if cfg["periodic"][i] else 0.0 for i in range(3))
    spec = PgfSpec(cfg["periodic"], lat)
    u = np.zeros(pm.n_parents)
    u[rows] = pgf_potential(xw[rows], xw, q, spec) + pgf_self(spec) * q[rows]
    u[rows] += z0["Zx"][rows] @ m[:, 0] + z0["Zy"][rows] @ m[:, 1] + z0["Zz"][rows] @ m[:, 2]
    H_bf = fem.gradient_field(ops, u)[samples] + fem.exchange_field(ops, m)[samples]
    print("oracle brute force at %d samples (%d rows): %.1f s" % (samples.size, rows.size, time.time() - t0),
          flush=True)
    out = []
    for st in a.settings.split(";"):
        p, s = st.split(",")
        p, s = int(p), float(s)
        t0 = time.time()
        ctx = Context(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"],
                      Aex=cfg["Aex"], order=p, rer_scale=s, z0_ring=a.ring, device=0)
        ctx.build_pgf()
        rank = ctx.internal_to_parent_rank()
        md = torch.tensor(m[rank], dtype=torch.float32, device="cuda")
        H = ctx.heff(md)
        torch.cuda.synchronize()
        Hu = np.zeros_like(m)
        Hu[rank] = H.double().cpu().numpy()
        err = float(np.linalg.norm(Hu[samples] - H_bf) / np.linalg.norm(H_bf))
        q_ = ctx.query()
        rec = {"p": p, "s": s, "rel_l2_H_vs_bruteforce": err, "nnz_cbox_per_row": q_["nnz_cbox"] / q_["n_parents"],
               "bytes_per_eval": q_["bytes_per_eval_algorithmic"], "setup_s": time.time() - t0}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        ctx.close()
    print(json.dumps({"config": a.config, "ring": a.ring, "samples": int(samples.size), "results": out}))


if __name__ == "__main__":
    main()
