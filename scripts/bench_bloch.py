"""Time the NEXT-4 complex Bloch field path next to the static one on the same context.

    python scripts/bench_bloch.py [--config C2] [--coarsen 2] [--steps 50]

Prints one JSON line: ms per H_eff evaluation of the static path (pmfem_heff) and of the Bloch
path (pmfem_heff_bloch: complex K1, two K2 + FFT pairs, complex K4/K5), CUDA events on the
evaluation stream after warm-up; and the host build time of the Bloch operators.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--coarsen", type=float, default=2)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    import numpy as np
    import torch
    import bench
    from paper_2409_13958_b200 import Context
    from synth import make_config
    cfg = make_config(a.config, coarsen=a.coarsen)
    mesh = cfg["mesh"]
    aim = bench.DEFAULTS[a.config]
    ctx = Context(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"], Aex=cfg["Aex"],
                  device=0, **aim)
    ctx.build_pgf()
    k0 = np.array([2 * np.pi / cfg["lattice"][a_] * f if cfg["periodic"][a_] else 0.0
                   for a_, f in zip(range(3), (0.3, 0.2, 0.1))])
    t0 = time.time()
    ctx.build_bloch(k0)
    t_build = time.time() - t0
    n = ctx.n_parents
    g = torch.Generator(device="cpu").manual_seed(1)
    mr = torch.randn(n, 3, generator=g).cuda()
    mi = torch.randn(n, 3, generator=g).cuda()
    st = torch.cuda.Stream()

    def timed(fn):
        with torch.cuda.stream(st):
            for _ in range(a.warmup):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(a.steps):
                fn()
            e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.steps

    H = torch.empty_like(mr)
    Hr, Hi = torch.empty_like(mr), torch.empty_like(mi)
    ms_static = timed(lambda: ctx.heff(mr, H, stream=st))
    ms_bloch = timed(lambda: ctx.heff_bloch(mr, mi, Hr, Hi, stream=st))
    print(json.dumps({"config": a.config, "coarsen": a.coarsen, "n_parents": n, "aim": aim,
                      "k0_fraction_of_reciprocal": [0.3, 0.2, 0.1], "ms_heff_static": ms_static,
                      "ms_heff_bloch": ms_bloch, "bloch_over_static": ms_bloch / ms_static,
                      "bloch_build_s": t_build, "steps": a.steps}))


if __name__ == "__main__":
    main()
