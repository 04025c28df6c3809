#!/bin/bash
# round 2, call 30: C4x KB = 4 as the default -- parity (normal + checked) and the default bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c30; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "heff_random or cbox_formats or fullsize" > $O/pytest.log 2>&1
PMFEM_LIB=checked timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cbox_formats and c4x" > $O/pytest_checked.log 2>&1
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --config C3 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
