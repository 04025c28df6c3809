"""Diagnose a GPU-vs-oracle parity failure stage by stage for a SMALL config (tests/helpers.py):
device spectrum vs the host/oracle spectrum, device C_box vs host, H under FFT plan variants."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main():
    import torch
    from helpers import oracle_model, lib_context, rel_l2
    from synth import m_random
    for key in sys.argv[1:]:
        om = oracle_model(key)
        host = lib_context(key, device=-1)
        host.build_pgf()
        dev = lib_context(key, device=0)
        dev.build_pgf()
        P = om.grid.fft
        sd = dev.export("spectrum_device").reshape(P[2], P[1], P[0] // 2 + 1)
        sh = host.export("spectrum").reshape(P[2], P[1], P[0] // 2 + 1)
        print(key, "fft", list(P), "spectrum dev vs host max rel %.3e" % (np.abs(sd - sh).max() / np.abs(sh).max()),
              flush=True)
        rank = dev.internal_to_parent_rank()
        m = m_random(om.n_parents, seed=1000 + len(key))
        ref = om.demag(m, "aim")
        for env in ({}, {"PMFEM_FFT_SPLIT": "1"}, {"PMFEM_YZ_TILE": "1"}, {"PMFEM_CBOX_FORMAT": "c4x"},
                    {"PMFEM_K2_TILE": "%d,%d,%d" % tuple(om.grid.n)}):
            for k, v in env.items():
                os.environ[k] = v
            ctx = lib_context(key, device=0)
            ctx.build_pgf()
            md = torch.tensor(m[rank], dtype=torch.float32, device="cuda:0")
            H = ctx.demag(md)
            torch.cuda.synchronize()
            out = np.zeros_like(m)
            out[rank] = H.double().cpu().numpy()
            print("  ", env, "rel L2 H_ms %.3e" % rel_l2(out, ref), "fused", ctx.query()["fft_fused"],
                  "fmt", ctx.query()["cbox_format"], flush=True)
            ctx.close()
            for k in env:
                del os.environ[k]


if __name__ == "__main__":
    main()
