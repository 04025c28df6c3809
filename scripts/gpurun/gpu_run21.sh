# round-1 session 3 final evidence: tests, default bench (+ oracle baseline), reference arm,
# C2 launch list + --set full (traffic), C3 --set full, C3/C5/C4 benches, LLG
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1; echo launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_local|k2_tile|k4_interp|k5_grad|fft_.*float" -s 7 -c 7 -o gpurun_out/prof_c2_all -f python scripts/profile_eval.py --evals 2 > gpurun_out/ncu_c2_all.log 2>&1; echo full2=$?
timeout 900 python bench.py --config C3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_local|k2_tile|k4_interp|k5_grad|fft_.*float" -s 7 -c 7 -o gpurun_out/prof_c3_all -f python scripts/profile_eval.py --config C3 --evals 2 > gpurun_out/ncu_c3_all.log 2>&1; echo full3=$?
timeout 900 python bench.py --config C5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 900 python scripts/bench_llg.py > gpurun_out/bench_llg.log 2>&1; echo llg=$?
timeout 2400 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo c4=$?
