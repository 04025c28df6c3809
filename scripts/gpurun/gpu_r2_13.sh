#!/bin/bash
# round 2, call 13: W4 A/B benches (the bench label for format 5 was missing in call 12)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c13; mkdir -p $O
for c in C2 C5 C3; do
  PMFEM_CBOX_FORMAT=w4 timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_${c}_w4.json 2> $O/bench_${c}_w4.err
done
PMFEM_CBOX_FORMAT=w4 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_w4.json 2> $O/bench_C4_w4.err
PMFEM_CBOX_FORMAT=w4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_win -c 1 -o $O/k4_c5_w4 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c5.log 2>&1
