#!/bin/bash
# round 2, call 26: C4x K4 (8 lanes per row) with __launch_bounds__(256, 5): 48 registers, 5 CTAs per SM
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c26; mkdir -p $O
timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_lb5.json 2> $O/bench_C4_lb5.err
timeout 600 python bench.py --config C3 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C3_lb5.json 2> $O/bench_C3_lb5.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "heff_random or (cbox_formats and c4x)" > $O/pytest.log 2>&1
