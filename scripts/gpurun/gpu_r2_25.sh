#!/bin/bash
# round 2, call 25: K4 lanes per row (G = 4/8/16/32) per config and format
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c25; mkdir -p $O
PMFEM_LIB=checked PMFEM_K4_GROUP=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cbox_formats and (c4x or w4 or u4)" > $O/pytest_g4_checked.log 2>&1
for gsel in 4 8; do
  PMFEM_K4_GROUP=$gsel timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_g$gsel.json 2> $O/bench_C4_g$gsel.err
done
for c in C5 C2 C3; do
  for gsel in 4 8 16 32; do
    PMFEM_K4_GROUP=$gsel timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_${c}_g$gsel.json 2> $O/bench_${c}_g$gsel.err
  done
done
