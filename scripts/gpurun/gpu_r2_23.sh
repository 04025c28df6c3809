#!/bin/bash
# round 2, call 23: W4 with the tile's chunk block staged by cp.async.bulk (PMFEM_W4_TMA=1); the
# C_box format parity tests with the K4 variants now read per context
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c23; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "cbox_formats" > $O/pytest_formats.log 2>&1
PMFEM_LIB=checked timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cbox_formats and (tma or stream)" > $O/pytest_checked.log 2>&1
PMFEM_W4_TMA=1 PMFEM_CBOX_FORMAT=w4 PMFEM_VERBOSE=1 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_w4tma.json 2> $O/bench_C4_w4tma.err
PMFEM_W4_TMA=1 timeout 600 python bench.py --config C5 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C5_w4tma.json 2> $O/bench_C5_w4tma.err
timeout 600 python bench.py --config C5 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C5_w4.json 2> $O/bench_C5_w4.err
PMFEM_W4_TMA=1 timeout 600 python bench.py --config C2 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C2_w4tma.json 2> $O/bench_C2_w4tma.err
PMFEM_W4_TMA=1 PMFEM_CBOX_FORMAT=w4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_win -c 1 -o $O/k4_c4_w4tma python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1
