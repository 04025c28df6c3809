"""Full-size AIM accuracy, oracle only ("controllable error", "relative error level
of 1e-3"; reading R19): the oracle's AIM H_eff vs the oracle's brute force at sampled
nodes of a BASELINE workload, for a sweep of (p, s).  Calls only oracle/ and synth/.

    python scripts/calibrate_fullsize.py --config C2 [--coarsen 1] [--samples 12]
        [--settings "1,3;2,3;2,4;3,4"] [--out profiles/calib_C2.json]

Brute force (O12): u_n = sum_{k != n} G_p(r_n - r_k) q_k + G_p^reg(0) q_n + (Z0 m)_n with the
C pair sums of oracle/bf.c, at the samples' 1-rings (H = -G u needs u there).  AIM (E2-E5):
P^T F^-1(G_hat F P q) + C_box q + Z0 m on the full grid, with C_box built for those rows only.
Both share q, Z0 and G, so the difference is the AIM discretisation error alone.  The GPU path
matches the oracle AIM to ~1e-6 (tests/test_gpu_*), so these numbers hold for the product.
Samples: random nodes plus surface nodes (lumped volume < 0.6 x median) and periodic-face nodes
(LCA components with more than one copy).  Two m fields: random unit vectors (white-noise
charges, the stress case) and the smooth physical field m = (cos t, sin t cos kx, sin t sin kx).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def pick_samples(pm, ops, n_random, seed=7):
    rng = np.random.default_rng(seed)
    Np = pm.n_parents
    out = list(rng.choice(Np, n_random, replace=False))
    Vt = ops["Vt"]
    surf = np.nonzero(Vt < 0.6 * np.median(Vt))[0]
    if surf.size:
        out += list(rng.choice(surf, min(4, surf.size), replace=False))
    ncopy = np.bincount(pm.pid, minlength=Np)
    face = np.nonzero(ncopy > 1)[0]
    if face.size:
        out += list(rng.choice(face, min(4, face.size), replace=False))
    return np.unique(np.array(out, dtype=np.int64))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--coarsen", type=float, default=1.0)
    ap.add_argument("--samples", type=int, default=12)
    ap.add_argument("--settings", default="2,3;2,4;3,3;3,4")
    ap.add_argument("--ring", type=int, default=1)
    ap.add_argument("--out", default=None)
    ap.add_argument("--alpha-scale", type=float, default=None,
                    help="Ewald splitting of the brute force (alpha-independent, tests/test_oracle_bf.py); "
                         "default 3 for 3D periodicity (shorter real-space sum), 1 otherwise")
    a = ap.parse_args()
    from oracle import aim, bf, fem
    from oracle.heff import OracleModel
    from synth import make_config, m_random

    t00 = time.time()
    cfg = make_config(a.config, coarsen=a.coarsen)
    mesh = cfg["mesh"]
    # operators + Z0 only at the sampled rows (build_aim=False: the grid is set up per setting)
    om = OracleModel(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"],
                     Aex=cfg["Aex"], z0_ring=a.ring, build_aim=False, rows=np.zeros(0, np.int64))
    pm, ops = om.pm, om.ops
    samples = pick_samples(pm, ops, a.samples)
    S = ops["S"].tocsr()
    rows = np.unique(np.concatenate([S.indices[S.indptr[n]:S.indptr[n + 1]] for n in samples] + [samples]))
    from oracle import z0 as oz0
    om.z0 = oz0.assemble_z0(pm, ops, om.Ms_tet, a.ring, rows=rows)
    om.rows = rows
    t_setup = time.time() - t00
    print("%s x%g: N'=%d, %d samples, %d rows, oracle setup %.1f s" % (a.config, a.coarsen, pm.n_parents,
                                                                       samples.size, rows.size, t_setup), flush=True)
    xw = om.xw
    L = max(v for v in cfg["lattice"] if v)
    k = 2 * np.pi / L
    ax = [i for i in range(3) if cfg["periodic"][i]][0]
    th = 0.3
    m_smooth = np.stack([np.full(pm.n_parents, np.cos(th)), np.sin(th) * np.cos(k * xw[:, ax]),
                         np.sin(th) * np.sin(k * xw[:, ax])], axis=1)
    fields = {"random": m_random(pm.n_parents, seed=77), "smooth": m_smooth}
    # brute force at the rows (C pair sums) -> H at the samples
    from oracle.pgf import PgfSpec
    import math
    asc = a.alpha_scale if a.alpha_scale is not None else (3.0 if om.spec.dim == 3 else 1.0)
    bf_spec = PgfSpec(om.periodic, om.lattice, alpha=asc * math.sqrt(math.pi) / om.spec.L.min())
    ref, hex_ = {}, {}
    t0 = time.time()
    for name, m in fields.items():
        q = om.charges(m)
        u = np.zeros(pm.n_parents)
        u[rows] = bf.potential(xw[rows], xw, q, bf_spec) + bf.pgf_self(bf_spec) * q[rows] + om.u_loc(m)[rows]
        ref[name] = fem.gradient_field(ops, u)[samples]
        hex_[name] = om.exchange(m)[samples]
    t_bf = time.time() - t0
    print("brute force: %.1f s" % t_bf, flush=True)
    grid = aim.Grid(cfg["grid"], om.periodic, om.lattice, xw)
    Ghat = aim.kernel_spectrum(aim.kernel_table(grid, om.spec))
    om.grid, om.Ghat = grid, Ghat
    results = []
    for st in a.settings.split(";"):
        p, s = st.split(",")
        p, s = int(p), float(s)
        t0 = time.time()
        try:
            om.S, om.W = aim.stencils(grid, xw, p)
            om.P = aim.projection_matrix(grid, om.S, om.W)
            om.C = aim.precorrection(grid, xw, om.lattice, om.S, om.W, s, p, rows)
        except ValueError as e:
            print(p, s, "invalid:", e, flush=True)
            continue
        rec = {"p": p, "s": s, "nnz_cbox_per_row": float(om.C.nnz / rows.size)}
        for name, m in fields.items():
            u = om.potential_aim(m)
            H = fem.gradient_field(ops, u)[samples]
            Hb = ref[name]
            dn = np.linalg.norm(H - Hb, axis=1)
            # H_ms (the field the AIM approximates) and H_eff = H_ms + H_ex (exact exchange)
            rec["rel_l2_Hms_%s" % name] = float(np.linalg.norm(H - Hb) / np.linalg.norm(Hb))
            rec["max_node_rel_Hms_%s" % name] = float(np.max(dn) / np.mean(np.linalg.norm(Hb, axis=1)))
            rec["rel_l2_Heff_%s" % name] = float(np.linalg.norm(H - Hb) / np.linalg.norm(Hb + hex_[name]))
        rec["seconds"] = time.time() - t0
        print(json.dumps(rec), flush=True)
        results.append(rec)
    out = {"config": a.config, "coarsen": a.coarsen, "n_parents": int(pm.n_parents), "grid": list(cfg["grid"]),
           "z0_ring": a.ring, "samples": int(samples.size), "rows": int(rows.size),
           "metric": "relative L2 over the samples of H_ms (and of H_eff = H_ms + H_ex, exchange exact), "
                     "oracle AIM vs oracle brute force; max_node_rel = max_n |dH_n| / mean_n |H_ms,n|",
           "oracle_setup_s": t_setup, "bruteforce_s": t_bf, "results": results}
    print(json.dumps(out))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
