#!/bin/bash
# round 2, call 20: Z0 kernel POP=8 / 5 CTAs per SM vs POP=16; W4 auto-selection (C2, C5)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c20; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_setup.py -q -k "z0" > $O/pytest_z0.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "heff_random or w4" > $O/pytest_parity.log 2>&1
PMFEM_VERBOSE=1 timeout 600 python bench.py --config C5 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
PMFEM_Z0_POP=16 PMFEM_VERBOSE=1 timeout 600 python bench.py --config C5 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C5_pop16.json 2> $O/bench_C5_pop16.err
timeout 600 python bench.py --config C2 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
PMFEM_VERBOSE=1 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
