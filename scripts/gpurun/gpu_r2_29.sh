#!/bin/bash
# round 2, call 29: at C4, C4x with 4 batched chunks per lane at 8 lanes per row; K2 tile 32x16x16
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c29; mkdir -p $O
PMFEM_K4_KB=4 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_kb4.json 2> $O/bench_C4_kb4.err
PMFEM_K2_TILE=32,16,16 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_k2t32.json 2> $O/bench_C4_k2t32.err
