# round-1 session 3: Stockham FFT thread counts, non-periodic mode (NEXT-3), K4/K1 reverted
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python bench.py --config C3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 900 python bench.py --config C5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_yz -s 1 -c 1 -o gpurun_out/prof_c3_fft_yz -f python scripts/profile_eval.py --config C3 --evals 2 > gpurun_out/ncu_c3_fft_yz.log 2>&1; echo full3=$?
