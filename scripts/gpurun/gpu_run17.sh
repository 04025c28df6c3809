# round-1 session 3: radix-4 DIT FFT restored (Stockham regressed), non-periodic parity, variance check
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python bench.py --config C3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 900 python bench.py --config C3 --steps 40 --no-cpu-baseline > gpurun_out/bench_c3b.log 2>&1; echo c3b=$?
timeout 900 python bench.py --config C5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo c5=$?
