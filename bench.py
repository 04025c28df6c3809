"""Benchmark: periodic H_eff evaluations/s (and mesh nodes/s) of the B200-native PM-FEM path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl pmfem|reference]

Default workload: C4, the 3D-periodic BCC sphere lattice of 10.2M nodes on a 256^3 AIM grid (the
BJ target size), at the calibrated accuracy p = 3, s = 4, z0_ring = 1.

One step = one pmfem_heff evaluation (K1 local_in -> K2 anterpolation -> K3 FFT convolution
-> K4 interpolation + precorrection -> K5 gradient + sum) over the whole synthetic mesh, inputs
resident in HBM.  L2 is flushed (256 MiB write) between timed steps, outside the timed events.
Prints ONE JSON line (rank 0).  --impl reference times the fp64 CPU oracle (oracle/) on a
bounded sample of the same workload (the tier's reference arm).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "periodic H_eff evals/s and mesh nodes/s at 1/2/4/8 B200; % HBM roofline"
# AIM settings per workload: the cheapest (p, s) whose oracle AIM meets the paper's 1e-3 level
# (reading R19: relative L2 of H_ms vs the oracle's brute force) at full size for both the
# random and the smooth m field (scripts/calibrate_fullsize.py -> profiles/calib_*.json)
DEFAULTS = {"C2": dict(order=3, rer_scale=4.0, z0_ring=1), "C3": dict(order=3, rer_scale=4.0, z0_ring=1),
            "C5": dict(order=3, rer_scale=4.0, z0_ring=1), "C4": dict(order=3, rer_scale=4.0, z0_ring=1),
            "C1": dict(order=1, rer_scale=2.0, z0_ring=1)}
CPU_SAMPLE = {"C1": 1, "C2": 8, "C3": 12, "C4": 20, "C5": 16}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    # the target workload (BJ: 10M nodes, 256^3): the largest single-GPU config
    ap.add_argument("--config", default="C4")
    ap.add_argument("--coarsen", type=float, default=1)
    ap.add_argument("--order", type=int, default=None)
    ap.add_argument("--rer-scale", type=float, default=None)
    ap.add_argument("--z0-ring", type=int, default=None)
    ap.add_argument("--impl", default="pmfem", choices=["pmfem", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    return ap.parse_args()


def aim_params(a):
    p = dict(DEFAULTS[a.config])
    if a.order is not None:
        p["order"] = a.order
    if a.rer_scale is not None:
        p["rer_scale"] = a.rer_scale
    if a.z0_ring is not None:
        p["z0_ring"] = a.z0_ring
    return p


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + ",".join(self.FIELDS),
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            out = self.p.communicate(timeout=5)[0]
        except Exception:
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


NNZ_CBOX_FULL = {"C2": 210505380, "C3": 353942100, "C4": 6553170681, "C5": 1903449600}


def cpu_baseline(cfg_name, aim, seconds, n_full, grid_full, fft_full, nnz_cbox_full=None):
    """The oracle (fp64 NumPy/SciPy, as it stands) timed on this box's host cores.

    The oracle's setup does not fit the bench's minutes at the full workload (its Z0 quadrature and
    precorrection double sums run for hours at 10^6-10^7 nodes), so one evaluation is EXTRAPOLATED
    from two measured parts:
      * the grid FFT convolution (E3), timed at the FULL padded grid (values do not change its cost);
      * the C_box product (E5), timed on a coarsened sample of the same geometry (h and the grid
        scaled together) and scaled by nnz(C_box)_full / nnz(C_box)_sample (by N' when the full nnz
        is unknown: the reference arm has no GPU context to count it);
      * everything else (sparse D/Z0/L/G products, P, P^T: linear in N' at fixed (p, ring)), timed
        on the same sample and scaled by N'_full / N'_sample.
    Both at all cores (scipy.fft workers = cores, BLAS threads = cores; scipy.sparse matvecs are
    single-threaded) and at 1 thread.  The sample's setup uses the oracle's Z0 quadrature at
    nquad = 6 (Z0 values do not change the evaluation's cost, only its sparsity)."""
    import types
    from threadpoolctl import threadpool_limits
    from oracle.heff import OracleModel
    from oracle import aim as oaim
    from synth import make_config, m_random
    c = CPU_SAMPLE[cfg_name]
    cfg = make_config(cfg_name, coarsen=c)
    m = cfg["mesh"]
    t0 = time.time()
    om = OracleModel(m.xyz, m.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"], Aex=cfg["Aex"],
                     order=aim["order"], rer_scale=aim["rer_scale"], z0_ring=aim["z0_ring"], nquad=6,
                     build_aim=False)
    # AIM parts of the sample: stencils and P at the bench order; C_box on the same near set
    # (r_ER = s max Delta does not depend on p) with p = 1 values -- the product's cost depends on
    # the sparsity only, and the p = 3 double stencil sum of the oracle's setup takes minutes
    om.grid = oaim.Grid(cfg["grid"], om.periodic, om.lattice, om.xw)
    om.S, om.W = oaim.stencils(om.grid, om.xw, aim["order"])
    om.P = oaim.projection_matrix(om.grid, om.S, om.W)
    om.Ghat = oaim.kernel_spectrum(oaim.kernel_table(om.grid, om.spec))
    S1, W1 = oaim.stencils(om.grid, om.xw, 1)
    om.C = oaim.precorrection(om.grid, om.xw, om.lattice, S1, W1, aim["rer_scale"], 1)
    t_setup = time.time() - t0
    mm = m_random(om.n_parents, seed=3)
    ncores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(0)
    gfull = types.SimpleNamespace(n=np.array(grid_full), fft=np.array(fft_full))
    Gh_full = rng.standard_normal(tuple(fft_full))
    Q_full = rng.standard_normal(tuple(grid_full))
    Q_s = rng.standard_normal(tuple(om.grid.n))

    def timed(fn, budget, min_reps=2):
        n, t0 = 0, time.time()
        while n < min_reps or time.time() - t0 < budget:
            fn()
            n += 1
        return (time.time() - t0) / n, n

    out = {}
    for threads in (ncores, 1):
        with threadpool_limits(threads):
            oaim.FFT_WORKERS = threads
            t_eval, n_ev = timed(lambda: om.heff(mm, "aim"), seconds / 4)
            t_conv_s, _ = timed(lambda: oaim.convolve(om.grid, om.Ghat, Q_s), seconds / 16)
            q_s = om.charges(mm)
            t_cbox_s, _ = timed(lambda: om.C @ q_s, seconds / 16)
            t_conv_f, n_cf = timed(lambda: oaim.convolve(gfull, Gh_full, Q_full), seconds / 8, 1)
        oaim.FFT_WORKERS = 1
        t_rest = max(t_eval - t_conv_s - t_cbox_s, 0.0)
        c_ratio = (nnz_cbox_full / om.C.nnz) if nnz_cbox_full else n_full / om.n_parents
        t_full = t_conv_f + t_cbox_s * c_ratio + t_rest * n_full / om.n_parents
        out[threads] = dict(s_per_eval=t_full, t_sample_eval=t_eval, n_sample_evals=n_ev, t_conv_full=t_conv_f,
                            t_cbox_sample=t_cbox_s, c_ratio=c_ratio)
    a, b = out[ncores], out[1]
    sample = ("EXTRAPOLATED to %s N'=%d: grid FFT convolution timed at the full %s padded grid (%.3f s at %d "
              "threads, %.3f s at 1), sparse operators timed on %s coarsened x%g (N'=%d, grid %s, %d AIM H_eff "
              "evals, %.3f s/eval at %d threads; C_box product %.4f s for %d nnz, scaled x%.1f by %s, the rest by "
              "N'); oracle sample setup %.1f s (nquad 6, C_box sparsity of the bench r_ER with p = 1 values) not included"
              % (cfg_name, n_full, "x".join(map(str, fft_full)), a["t_conv_full"], ncores, b["t_conv_full"],
                 cfg_name, c, om.n_parents, "x".join(map(str, cfg["grid"])), a["n_sample_evals"],
                 a["t_sample_eval"], ncores, a["t_cbox_sample"], om.C.nnz, a["c_ratio"],
                 "nnz(C_box)" if nnz_cbox_full else "N'", t_setup))
    return dict(s_per_eval=a["s_per_eval"], s_per_eval_1thread=b["s_per_eval"], cores=ncores, sample=sample,
                n_sample=om.n_parents, setup_s=t_setup)


def run_reference(a):
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and rank != 0:
        return
    from synth import make_config
    aim = aim_params(a)
    full = make_config(a.config, coarsen=a.coarsen)
    per_step = max(1.0, min(20.0, 120.0 / max(1, a.steps + a.warmup)))
    from oracle.mesh import PeriodicMesh
    fm = full["mesh"]
    n_full = PeriodicMesh(fm.xyz, fm.tets, full["periodic"], full["lattice"]).n_parents   # N' as the GPU arm
    grid = list(full["grid"])
    fft = [g if p else 2 * g for g, p in zip(grid, full["periodic"])]
    # the full-size nnz(C_box) the library counts at the DEFAULTS setting (the reference arm has
    # no GPU context; measured: profiles/ab/r02c2*_bench_*.json config.nnz_cbox), so both arms
    # extrapolate the C_box product the same way; other settings fall back to N' scaling
    nnz_full = NNZ_CBOX_FULL.get(a.config) if (a.coarsen == 1 and aim == DEFAULTS.get(a.config)) else None
    cb = cpu_baseline(a.config, aim, per_step * max(1, a.steps), n_full, grid, fft, nnz_full)
    value = 1.0 / cb["s_per_eval"]
    nodes_per_s = value * n_full
    line = {"metric": METRIC, "value": value, "unit": "evals/s", "impl": "reference", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "%s: %s" % (a.config, full["desc"]), "n_nodes_full": n_full, **aim},
            "nodes_per_s": nodes_per_s,
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cb["cores"], "kind": "oracle",
                             "sample": cb["sample"], "value_1thread": 1.0 / cb["s_per_eval_1thread"]},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    # a dedicated (non-default) stream: the library captures each evaluation into a CUDA graph
    torch.cuda.set_stream(torch.cuda.Stream())
    dev = local
    from paper_2409_13958_b200 import Context, KERNELS
    from synth import make_config

    aim = aim_params(a)
    cfg = make_config(a.config, coarsen=a.coarsen)
    mesh = cfg["mesh"]
    nccl_id = None
    if world > 1:
        from paper_2409_13958_b200 import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    t0 = time.time()
    ctx = Context(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"], Aex=cfg["Aex"],
                  device=dev, rank=rank, world=world, nccl_id=nccl_id, **aim)
    t_setup = time.time() - t0
    t0 = time.time()
    ctx.build_pgf()
    t_pgf = time.time() - t0
    info = ctx.query()
    Np = info["n_parents"]
    Nloc = info["n_parents_local"]
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    m = torch.randn(Nloc, 3, device="cuda", generator=g)
    m = (m / m.norm(dim=1, keepdim=True)).contiguous()
    H = torch.empty_like(m)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MiB > L2 (126 MB)
    stream = torch.cuda.current_stream()
    for _ in range(max(3, a.warmup)):
        ctx.heff(m, H)
    torch.cuda.synchronize()
    # clocks: sample during a >= 1 s run of the same step right before and through the timed region
    clk = ClockSampler(dev)
    clk.start()
    t_end = time.time() + 1.0
    while time.time() < t_end:
        ctx.heff(m, H)
        torch.cuda.synchronize()
    ctx.set_timing(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, kern_ms = [], {k: [] for k in KERNELS}
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    for _ in range(a.steps):
        flush.zero_()
        ev0.record(stream)
        ctx.heff(m, H)
        ev1.record(stream)
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
        for k, v in ctx.timing().items():
            kern_ms[k].append(v)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ctx.set_timing(False)
    tot_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    # one distributed evaluation covers the whole mesh: evals/s of the job = steps / max time
    value = a.steps / (tot_ms / 1e3)

    # end to end through the public API with host buffers (pinned), copies inside the timed region
    m_h = m.cpu().pin_memory()
    H_h = torch.empty_like(m_h).pin_memory()
    for _ in range(3):
        ctx.heff_host(m_h, H_h)
    e2e_ms = []
    for _ in range(a.steps):
        flush.zero_()
        torch.cuda.synchronize()
        ev0.record(stream)
        ctx.heff_host(m_h, H_h)
        ev1.record(stream)
        ev1.synchronize()
        e2e_ms.append(ev0.elapsed_time(ev1))
    e2e_tot = float(sum(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_tot], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_tot = float(t.item())
    e2e_value = a.steps / (e2e_tot / 1e3)

    peaks, peak_src = load_peaks()
    kb = info["kernel_bytes"]
    kernels = {}
    for i, k in enumerate(KERNELS):
        ms = float(np.mean(kern_ms[k]))
        kernels[k] = {"ms": ms, "bytes": kb[i], "GBps": kb[i] / (ms * 1e-3) / 1e9 if ms > 0 else None}
    dom = max(KERNELS, key=lambda k: kernels[k]["ms"])
    ach = kernels[dom]["GBps"]
    for k in KERNELS:
        if kernels[k]["GBps"] is not None:
            kernels[k]["frac_hbm"] = kernels[k]["GBps"] / peaks["hbm_gbs"]
    # traffic: DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    # capture of this config (profiles/traffic.json, written by scripts/ncu_traffic.py)
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(a.config, {}).get(dom)
        if tr is not None and world == 1:
            traffic, traffic_src = tr["dram_bytes"], "%s (%s)" % (tr["report"], tr["note"])
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes": kb[KERNELS.index(dom)], "peak_source": peak_src,
                "share_of_step": kernels[dom]["ms"] / float(np.mean(step_ms))}
    alg_total = sum(kb[:5])
    line = {"metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": tot_ms / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "%s: %s" % (a.config, cfg["desc"]), "n_nodes": info["n_nodes"],
                       "n_parents": Np, "grid": info["grid"], "fft": info["fft"], **aim,
                       "nnz_ring1": info["nnz_ring1"], "nnz_z0": info["nnz_z0"], "nnz_cbox": info["nnz_cbox"],
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "parallelism": "single GPU" if world == 1 else
                       ("slab-partitioned rows over %d GPUs: NCCL halos (m, q, u) + slab-decomposed FFT "
                        "(reduce-scatter, 2 all-to-all transposes, all-gather)" % world if info["slab_world"] > 1 else
                        "slab-partitioned rows over %d GPUs: NCCL halos (m, q, u) + all-reduce of the "
                        "anterpolated grid, replicated FFT" % world), "n_parents_local": Nloc,
                       "k2_tile": info["k2_tile"],
                       "cbox_format": ["C4x", "B4", "SEG", "U4", "?", "W4"][info["cbox_format"]],
                       "cbox_packed_units": info["cbox_packed_units"]},
            "nodes_per_s": value * Np, "setup_s": t_setup, "build_pgf_s": t_pgf,
            "bytes_per_eval_algorithmic": alg_total,
            "eval_GBps_algorithmic": alg_total / (tot_ms / a.steps * 1e-3) / 1e9,
            "kernels": kernels, "roofline": roofline,
            "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": int(m_h.numel() * 4),
                    "d2h_bytes_per_step": int(H_h.numel() * 4)},
            "gpu_launches": info["launches_per_eval"] * a.steps, "clocks": clocks,
            "comm_bytes_per_eval_rank": info["comm_bytes_per_eval"]}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cb = cpu_baseline(a.config, aim, a.cpu_seconds, Np, info["grid"], info["fft"], info["nnz_cbox"])
        line["cpu_baseline"] = {"value": 1.0 / cb["s_per_eval"], "unit": "evals/s", "cores": cb["cores"],
                                "kind": "oracle", "sample": cb["sample"],
                                "value_1thread": 1.0 / cb["s_per_eval_1thread"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
