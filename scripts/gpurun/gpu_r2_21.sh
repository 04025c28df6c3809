#!/bin/bash
# round 2, call 21: Z0 pipeline with pinned parallel staging; full GPU suite + smoke (Bloch in
# smoke); default bench with setup timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c21; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
PMFEM_VERBOSE=1 timeout 600 python bench.py --config C5 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
PMFEM_VERBOSE=1 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
