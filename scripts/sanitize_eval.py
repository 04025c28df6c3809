"""One small H_eff evaluation per fused-FFT tile for compute-sanitizer (memcheck / racecheck /
synccheck): K1, K2 (shared-memory fixed-point atomics), the fused YZ FFT (tile 1, 2, 4), K4, K5.

    compute-sanitizer --tool racecheck python scripts/sanitize_eval.py [C2p2]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ.setdefault("PMFEM_NO_GRAPH", "1")


def main():
    import torch
    from helpers import lib_context
    keys = sys.argv[1:] or ["C2p2", "C5p2"]
    for key in keys:
        for tile in ("1", "2", "4"):
            os.environ["PMFEM_YZ_TILE"] = tile
            ctx = lib_context(key, device=0)
            ctx.build_pgf()
            m = torch.nn.functional.normalize(torch.randn(ctx.n_parents, 3, device="cuda:0"), dim=1).contiguous()
            H = ctx.heff(m)
            torch.cuda.synchronize()
            print(key, "tile", tile, "k2_tile", ctx.query()["k2_tile"], "|H| = %.4e" % float(H.norm()), flush=True)
            ctx.close()


if __name__ == "__main__":
    main()
