# round-1 session 3: tiled K2; K4/K2 --set full captures (traffic), bench C2/C3/C5
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python bench.py --config C3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 900 python bench.py --config C5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k4_interp|k2_tile|k1_local|k5_grad" -s 4 -c 4 -o gpurun_out/prof_c2_k -f python scripts/profile_eval.py --evals 2 > gpurun_out/ncu_full_c2.log 2>&1; echo full2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k4_interp|k2_tile|k1_local|k5_grad|fft_.*float" -s 7 -c 7 -o gpurun_out/prof_c3_k -f python scripts/profile_eval.py --config C3 --evals 2 > gpurun_out/ncu_full_c3.log 2>&1; echo full3=$?
