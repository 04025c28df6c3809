#!/bin/bash
# round 2, call 10: persistent Z0 pipeline buffers (setup timing), Bloch device kernel, C_box
# format parity incl. the row-range streaming K4 variants, and K4 stream vs default benches
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c10; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_setup.py -q -k "z0 or bloch" > $O/pytest_setup.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cbox_formats" > $O/pytest_formats.log 2>&1
PMFEM_VERBOSE=1 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
PMFEM_K4_STREAM=1 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_stream.json 2> $O/bench_C4_stream.err
for c in C2 C5; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  PMFEM_K4_STREAM=1 timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_${c}_stream.json 2> $O/bench_${c}_stream.err
done
