set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
python scripts/profile_eval.py --evals 2 > gpurun_out/plain_prof.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c2.csv python scripts/profile_eval.py --evals 3 > gpurun_out/ncu_launch.log 2>&1; echo launch=$?
ncu --set full --clock-control none --import-source on -k regex:"k1_local|k4_interp|k5_grad|fft_yz|fft_x_|k2_anterp" -s 1 -c 7 -o gpurun_out/prof_c2 python scripts/profile_eval.py --evals 1 > gpurun_out/ncu_full.log 2>&1; echo full=$?
