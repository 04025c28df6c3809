#!/bin/bash
# round 2, call 5: U4 C_box format (unaligned 4-column blocks + q4 gathers); full-size sampled parity
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c05; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_setup.py tests/test_gpu_parity.py -q -k "cbox" > $O/pytest_cbox.log 2>&1
for c in C2 C5 C3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_${c}_u4.json 2> $O/bench_${c}_u4.err
done
PMFEM_VERBOSE=1 timeout 1200 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C4_u4.json 2> $O/bench_C4_u4.err
PMFEM_CBOX_FORMAT=c4x timeout 1200 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C4_c4x.json 2> $O/bench_C4_c4x.err
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s > $O/pytest_fullsize.log 2>&1
