set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
python scripts/profile_eval.py --config C2 --coarsen 4 --evals 1 > gpurun_out/plain_small.log 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --leak-check no python scripts/profile_eval.py --config C2 --coarsen 4 --evals 1 > gpurun_out/memcheck.log 2>&1; echo memcheck=$?
