"""Config C5 of BASELINE.json: 1D-periodic waveguide spin-wave LLG run, full H_eff (exchange +
periodic demag) for 1000 RK4 steps (NEXT-2).  Prints one JSON line.

    python scripts/bench_llg.py [--config C5] [--steps 1000] [--dt 5e-14] [--alpha 0.02]
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
    ap.add_argument("--config", default="C5")
    ap.add_argument("--coarsen", type=float, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dt", type=float, default=5e-14)
    ap.add_argument("--alpha", type=float, default=0.02)
    ap.add_argument("--integrator", default="rk4", choices=["rk4", "am2"])
    ap.add_argument("--tol", type=float, default=1e-5, help="AM2 local error tolerance")
    a = ap.parse_args()
    import torch
    import bench
    from paper_2409_13958_b200 import Context
    from synth import make_config
    torch.cuda.set_stream(torch.cuda.Stream())
    aim = bench.aim_params(argparse.Namespace(config=a.config, order=None, rer_scale=None, z0_ring=None))
    cfg = make_config(a.config, coarsen=a.coarsen)
    mesh = cfg["mesh"]
    t0 = time.time()
    ctx = Context(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"], Aex=cfg["Aex"],
                  device=0, **aim)
    ctx.build_pgf()
    t_setup = time.time() - t0
    n = ctx.n_parents
    rng = np.random.default_rng(1005)
    pert = np.deg2rad(1.0) * rng.normal(size=(n, 2))
    m0 = np.stack([np.ones(n), pert[:, 0], pert[:, 1]], 1)
    m0 /= np.linalg.norm(m0, axis=1, keepdims=True)
    m = torch.tensor(m0, dtype=torch.float32, device="cuda")
    ctx.llg_rk4(m, a.warmup, a.dt, a.alpha)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    if a.integrator == "am2":
        # the paper's adaptive AB2/AM2 predictor-corrector over the same simulated time
        t0 = time.time()
        acc, rej = ctx.llg_am2(m, a.steps * a.dt, a.dt, a.tol, a.alpha)
        torch.cuda.synchronize()
        ms = (time.time() - t0) * 1e3
        norm_dev = float((m.norm(dim=1) - 1).abs().max())
        print(json.dumps({"metric": "LLG AM2 adaptive predictor-corrector", "simulated_ns": a.steps * a.dt * 1e9,
                          "total_s": ms / 1e3, "accepted_steps": acc, "rejected_steps": rej, "tol": a.tol,
                          "heff_evals": 2 * acc + rej + 1, "heff_evals_per_s": (2 * acc + rej + 1) / (ms / 1e3),
                          "n_parents": n, "setup_s": t_setup, "max_norm_deviation": norm_dev,
                          "config": {"workload": "%s: %s" % (a.config, cfg["desc"]), **aim}}), flush=True)
        return
    e0.record(s)
    ctx.llg_rk4(m, a.steps, a.dt, a.alpha)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    norm_dev = float((m.norm(dim=1) - 1).abs().max())
    print(json.dumps({"metric": "LLG RK4 steps/s (4 H_eff per step)", "value": a.steps / (ms / 1e3),
                      "unit": "steps/s", "steps": a.steps, "total_s": ms / 1e3, "ms_per_step": ms / a.steps,
                      "heff_evals_per_s": 4 * a.steps / (ms / 1e3), "n_parents": n, "dt_s": a.dt,
                      "alpha": a.alpha, "simulated_ns": a.steps * a.dt * 1e9, "setup_s": t_setup,
                      "max_norm_deviation": norm_dev,
                      "config": {"workload": "%s: %s" % (a.config, cfg["desc"]), **aim}}), flush=True)


if __name__ == "__main__":
    main()
