#!/bin/bash
# round 2, call 8: batched K4 gathers (index/value loads first, then the dependent q gathers);
# checked build (device bounds asserts) over the GPU parity / setup / LLG tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c08; mkdir -p $O
for f in u4 c4x; do
  PMFEM_VERBOSE=1 PMFEM_CBOX_FORMAT=$f timeout 900 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_$f.json 2> $O/bench_C4_$f.err
done
for f in b4 u4 c4x; do
  PMFEM_CBOX_FORMAT=$f timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C5_$f.json 2> $O/bench_C5_$f.err
  PMFEM_CBOX_FORMAT=$f timeout 600 python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C3_$f.json 2> $O/bench_C3_$f.err
done
PMFEM_LIB=checked timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_setup.py tests/test_gpu_llg.py tests/test_gpu_nonperiodic.py -q -x > $O/pytest_checked.log 2>&1
