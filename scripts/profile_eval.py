"""Set up one config and run a few pmfem_heff evaluations (for ncu / compute-sanitizer).

    python scripts/profile_eval.py [--config C2] [--coarsen 1] [--evals 3] [--order 2] [--rer-scale 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--coarsen", type=float, default=1)
    ap.add_argument("--evals", type=int, default=3)
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--rer-scale", type=float, default=3.0)
    ap.add_argument("--z0-ring", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2409_13958_b200 import Context
    from synth import make_config
    cfg = make_config(a.config, coarsen=a.coarsen)
    m = cfg["mesh"]
    t = time.time()
    ctx = Context(m.xyz, m.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"], Aex=cfg["Aex"],
                  order=a.order, rer_scale=a.rer_scale, z0_ring=a.z0_ring, device=0)
    ctx.build_pgf()
    print("setup %.1fs" % (time.time() - t), ctx.query(), flush=True)
    Np = ctx.n_parents
    mm = torch.randn(Np, 3, device="cuda")
    mm = (mm / mm.norm(dim=1, keepdim=True)).contiguous()
    H = torch.empty_like(mm)
    for _ in range(a.evals):
        ctx.heff(mm, H)
    torch.cuda.synchronize()
    print("done", float(H.abs().max()))


if __name__ == "__main__":
    main()
