#!/bin/bash
# round 2, call 12: W4 windowed C_box (shared-memory q window per tile): parity + A/B benches
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c12; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cbox_formats and w4" > $O/pytest_w4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_setup.py -q -k "w4" > $O/pytest_w4_setup.log 2>&1
PMFEM_LIB=checked timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cbox_formats and w4" > $O/pytest_w4_checked.log 2>&1
for c in C2 C5 C3; do
  PMFEM_VERBOSE=1 PMFEM_CBOX_FORMAT=w4 timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_${c}_w4.json 2> $O/bench_${c}_w4.err
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_${c}.json 2> $O/bench_${c}.err
done
PMFEM_VERBOSE=1 PMFEM_CBOX_FORMAT=w4 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_w4.json 2> $O/bench_C4_w4.err
