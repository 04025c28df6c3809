set -x
export PMFEM_VERBOSE=1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo bench3=$?
timeout 900 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo bench5=$?
python scripts/profile_eval.py --config C3 --evals 2 > gpurun_out/plain_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_eval.py --config C3 --evals 2 > gpurun_out/ncu_c3.log 2>&1; echo ncu=$?
timeout 3000 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo bench4=$?
