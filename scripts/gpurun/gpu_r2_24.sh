#!/bin/bash
# round 2, call 24: K4 lanes per row at C4 (C4x, G = 16 / 8 vs the default 32)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c24; mkdir -p $O
for gsel in 16 8; do
  PMFEM_K4_GROUP=$gsel timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_g$gsel.json 2> $O/bench_C4_g$gsel.err
done
timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_g32.json 2> $O/bench_C4_g32.err
