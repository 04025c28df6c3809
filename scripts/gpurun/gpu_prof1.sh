set -x
python scripts/profile_eval.py --evals 3 > gpurun_out/plain_prof.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c2.csv python scripts/profile_eval.py --evals 3 > gpurun_out/ncu_launch.log 2>&1; echo launch=$?
ncu --set full --clock-control none --import-source on -k regex:"k1_local_in|k4_interp|k5_grad|fft_strided|k2_anterp|fft_x" -c 9 -o gpurun_out/prof_c2 python scripts/profile_eval.py --evals 1 > gpurun_out/ncu_full.log 2>&1; echo full=$?
