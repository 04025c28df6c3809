#!/bin/bash
# round 2, call 18: W4 with the window copy flattened over the CTA (run table in shared memory)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c18; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_setup.py -q -k "w4" > $O/pytest_w4.log 2>&1
PMFEM_LIB=checked timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cbox_formats and w4" > $O/pytest_w4_checked.log 2>&1
for w in 6144 4096 8192; do
  PMFEM_W4_WMAX=$w PMFEM_CBOX_FORMAT=w4 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_w4_$w.json 2> $O/bench_C4_w4_$w.err
done
for c in C5 C2 C3; do
  for w in 4096 6144; do
    PMFEM_W4_WMAX=$w PMFEM_CBOX_FORMAT=w4 timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_${c}_w4_$w.json 2> $O/bench_${c}_w4_$w.err
  done
done
PMFEM_W4_WMAX=6144 PMFEM_CBOX_FORMAT=w4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_win -c 1 -o $O/k4_c4_w4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1
