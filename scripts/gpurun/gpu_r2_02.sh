#!/bin/bash
# round 2, call 2: Z0 warp-per-task kernel (device vs host Z0, C4 setup time), new parity cases
# (fused-YZ tiles 2/4, z- and y-periodic), compute-sanitizer on K2 + fused FFT
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c02; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_setup.py -x -q -k "z0" > $O/pytest_z0.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "yz_fused_tiles or R1p2 or Y1p2" > $O/pytest_new.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_eval.py C2p2 C5p2 > $O/sanitizer_$tool.log 2>&1
done
PMFEM_VERBOSE=1 timeout 1500 python bench.py --config C4 --order 3 --rer-scale 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C4_p3s4.json 2> $O/bench_C4_p3s4.err
