"""AIM calibration study: oracle AIM vs oracle brute force.

Sweeps stencil order p and precorrection radius s (r_ER = s * Delta) on tiny
analogues of the BASELINE configs and prints relative L2 of H_ms (and of u after
mean removal) for a random m (white-noise charges, the worst case) and a smooth m
with non-zero divergence.  Calls only oracle/ and synth/.

    python scripts/calibrate_aim.py C2 4 [z0_ring]
"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from synth import make_config, m_random            # noqa: E402
from oracle.heff import OracleModel                # noqa: E402
from oracle import aim, fem                        # noqa: E402


def main():
    name = sys.argv[1]
    coarsen = float(sys.argv[2])
    ring = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    cfg = make_config(name, coarsen=coarsen)
    m = cfg["mesh"]
    t = time.time()
    om = OracleModel(m.xyz, m.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"],
                     Aex=cfg["Aex"], z0_ring=ring)
    print(name, coarsen, "N'", om.n_parents, "grid", cfg["grid"],
          "nodes/box %.2f" % (om.n_parents / np.prod(cfg["grid"])), "setup %.1fs" % (time.time() - t),
          flush=True)
    L = max(cfg["lattice"])
    k = 2 * np.pi / L
    ms = np.stack([np.cos(k * om.xw[:, 0]), np.sin(k * om.xw[:, 0]), 0 * om.xw[:, 0]], 1)
    fields = [("random", m_random(om.n_parents, 7)), ("smooth", ms)]
    t = time.time()
    ref = [(om.potential_bf(f)) for _, f in fields]
    print("bf %.1fs" % (time.time() - t), flush=True)
    Href = [fem.gradient_field(om.ops, u) for u in ref]
    for p in (1, 2, 3):
        for s in (1.5, 2, 3, 4):
            try:
                om.S, om.W = aim.stencils(om.grid, om.xw, p)
                om.P = aim.projection_matrix(om.grid, om.S, om.W)
                om.C = aim.precorrection(om.grid, om.xw, om.lattice, om.S, om.W, s, p)
            except ValueError as e:
                print(p, s, "invalid:", e)
                continue
            out = []
            for (nm, f), ub, Hb in zip(fields, ref, Href):
                ua = om.potential_aim(f)
                Ha = fem.gradient_field(om.ops, ua)
                du = (ua - ua.mean()) - (ub - ub.mean())
                out.append("%s u %.2e H %.2e" % (nm, np.linalg.norm(du) / np.linalg.norm(ub - ub.mean()),
                                                  np.linalg.norm(Ha - Hb) / np.linalg.norm(Hb)))
            print("p=%d s=%.1f nnz/row %.1f | %s" % (p, s, om.C.nnz / om.n_parents, " | ".join(out)), flush=True)


if __name__ == "__main__":
    main()
