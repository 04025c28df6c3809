# restored-checkout check + A/B: streaming-load hint (-DPMFEM_STREAM_CS) and K4 C4x vector gathers (PMFEM_K4_VEC=1, C3 uses C4x)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_default.log 2>&1; echo build=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
for v in default cs; do
if [ $v = cs ]; then export PMFEM_EXTRA_NVCC=-DPMFEM_STREAM_CS; python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$v.log 2>&1; echo build=$?; fi
timeout 900 python bench.py --steps 40 --no-cpu-baseline > gpurun_out/bench_c2_$v.log 2>&1; echo c2=$?
timeout 900 python bench.py --config C3 --steps 30 --no-cpu-baseline > gpurun_out/bench_c3_$v.log 2>&1; echo c3=$?
PMFEM_K4_VEC=1 timeout 900 python bench.py --config C3 --steps 30 --no-cpu-baseline > gpurun_out/bench_c3vec_$v.log 2>&1; echo c3vec=$?
timeout 900 python bench.py --config C5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5_$v.log 2>&1; echo c5=$?
done
