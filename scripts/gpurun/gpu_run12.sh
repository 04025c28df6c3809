# round-1 session 3: fixed-point tiled K2, C4x C_box (K4), slab FFT (simulated ranks); profiles
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python bench.py --config C3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 900 python bench.py --config C5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo c5=$?
for k in k2_tile k4_interp fft_yz k1_local; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_c3_$k -f python scripts/profile_eval.py --config C3 --evals 1 > gpurun_out/ncu_c3_$k.log 2>&1; echo full3_$k=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_tile|k4_interp" -c 2 -o gpurun_out/prof_c2 -f python scripts/profile_eval.py --evals 1 > gpurun_out/ncu_c2.log 2>&1; echo full2=$?
timeout 2400 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo c4=$?
