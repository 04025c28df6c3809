#!/bin/bash
# round 2, call 19: W4 rows with every operand in shared memory and the chunk batch issued before
# the interpolation; same-box A/B against the default formats; ncu of the Z0 integration kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c19; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_setup.py -q -k "w4" > $O/pytest_w4.log 2>&1
PMFEM_LIB=checked timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cbox_formats and w4" > $O/pytest_w4_checked.log 2>&1
for c in C5 C2; do
  for w in 4096 6144; do
    PMFEM_W4_WMAX=$w PMFEM_CBOX_FORMAT=w4 timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_${c}_w4_$w.json 2> $O/bench_${c}_w4_$w.err
  done
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_${c}_auto.json 2> $O/bench_${c}_auto.err
done
for w in 4096 6144; do
  PMFEM_W4_WMAX=$w PMFEM_CBOX_FORMAT=w4 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_w4_$w.json 2> $O/bench_C4_w4_$w.err
done
timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_auto.json 2> $O/bench_C4_auto.err
PMFEM_W4_WMAX=4096 PMFEM_CBOX_FORMAT=w4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_win -c 1 -o $O/k4_c4_w4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_z0_warp -c 1 -o $O/z0_c5 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_z0.log 2>&1
