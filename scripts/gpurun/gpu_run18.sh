# round-1 session 3: B4 C_box format, K1/K5 row split
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
PMFEM_CBOX_FORMAT=c4x timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_c2_c4x.log 2>&1; echo bench=$?
PMFEM_ROW_SPLIT=1 timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_c2_rs1.log 2>&1; echo bench=$?
timeout 900 python bench.py --config C3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
PMFEM_CBOX_FORMAT=c4x timeout 900 python bench.py --config C3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c3_c4x.log 2>&1; echo c3=$?
timeout 900 python bench.py --config C5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo c5=$?
PMFEM_CBOX_FORMAT=b4 timeout 900 python bench.py --config C5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5_b4.log 2>&1; echo c5=$?
