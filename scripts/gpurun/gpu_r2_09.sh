#!/bin/bash
# round 2, call 9: Z0 warp-parallel subdivision (device vs host Z0), C4 setup timing, format
# auto-selection; then the default bench (C4 + cpu baseline) and the ncu launch list of it
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c09; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_setup.py -q -k "z0" > $O/pytest_z0.log 2>&1
PMFEM_VERBOSE=1 timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in C2 C3 C5; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
