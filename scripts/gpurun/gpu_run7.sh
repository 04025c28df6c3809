set -x
export PMFEM_VERBOSE=1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo bench3=$?
timeout 900 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo bench5=$?
timeout 3000 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo bench4=$?
