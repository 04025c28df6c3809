#!/bin/bash
# round 2, call 15: W4 window cap A/B at C4 (the bench default) and C3, next to C4x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c15; mkdir -p $O
for w in 4096 2048 6144; do
  PMFEM_W4_WMAX=$w PMFEM_CBOX_FORMAT=w4 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_w4_$w.json 2> $O/bench_C4_w4_$w.err
done
PMFEM_CBOX_FORMAT=c4x timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_c4x.json 2> $O/bench_C4_c4x.err
for w in 2048 4096; do
  PMFEM_W4_WMAX=$w PMFEM_CBOX_FORMAT=w4 timeout 600 python bench.py --config C3 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C3_w4_$w.json 2> $O/bench_C3_w4_$w.err
  PMFEM_W4_WMAX=$w PMFEM_CBOX_FORMAT=w4 timeout 600 python bench.py --config C5 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C5_w4_$w.json 2> $O/bench_C5_w4_$w.err
done
PMFEM_CBOX_FORMAT=w4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_win -c 1 -o $O/k4_c4_w4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1
