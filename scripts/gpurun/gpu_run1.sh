set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv
nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config C2 --coarsen 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2c2.log 2>&1; echo b1=$?
timeout 1500 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo b2=$?
