# round-1 session 2: health check of the committed path + K4 --set full traffic for C3 and C2
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
python scripts/profile_eval.py --evals 3 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k4_interp|k1_local|k2_p2g|k5_grad|fft_" -s 0 -c 8 -o gpurun_out/prof_c2 python scripts/profile_eval.py --evals 1 > gpurun_out/ncu_full_c2.log 2>&1; echo full2=$?
python scripts/profile_eval.py --config C3 --evals 2 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k4_interp|k1_local|k2_p2g|k5_grad|fft_" -c 8 -o gpurun_out/prof_c3 python scripts/profile_eval.py --config C3 --evals 1 > gpurun_out/ncu_full_c3.log 2>&1; echo full3=$?
