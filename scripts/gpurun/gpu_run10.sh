# round-1 session 3: health check of the committed path, bench lines, launch list, K4 --set full
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1; echo launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k4_interp|k1_local|k2_|k5_grad|fft_" -c 8 -o gpurun_out/prof_c2 python scripts/profile_eval.py --evals 1 > gpurun_out/ncu_full_c2.log 2>&1; echo full2=$?
timeout 900 python bench.py --config C3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
