# round-1 session 3: evidence for the committed path: C2 launch list + --set full (traffic), C4 bench
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1; echo launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_local|k2_tile|k4_interp|k5_grad|fft_" -s 10 -c 7 -o gpurun_out/prof_c2_all -f python scripts/profile_eval.py --evals 3 > gpurun_out/ncu_c2_all.log 2>&1; echo full2=$?
timeout 2400 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo c4=$?
