#!/bin/bash
# round 2, call 1: box facts, C5/C4 setup breakdown and eval time at the accurate AIM settings
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c01; mkdir -p $O
(nproc; lscpu | head -20; free -g; nvidia-smi) > $O/box.txt 2>&1
for cfg in C5 C4; do
  PMFEM_VERBOSE=1 timeout 1500 python bench.py --config $cfg --order 3 --rer-scale 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_${cfg}_p3s4.json 2> $O/bench_${cfg}_p3s4.err
done
PMFEM_VERBOSE=1 timeout 600 python bench.py --config C5 --order 2 --rer-scale 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C5_p2s4.json 2> $O/bench_C5_p2s4.err
