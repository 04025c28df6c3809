# K4 C4x vector gathers A/B (C3, C2 forced C4x), parity subset
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "cbox_formats or heff_random" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for v in 0 1; do
PMFEM_K4_VEC=$v timeout 900 python bench.py --config C3 --steps 30 --no-cpu-baseline > gpurun_out/bench_c3_vec$v.log 2>&1; echo c3_$v=$?
PMFEM_K4_VEC=$v PMFEM_CBOX_FORMAT=c4x timeout 900 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/bench_c2_vec$v.log 2>&1; echo c2_$v=$?
done
PMFEM_K4_VEC=1 PMFEM_CBOX_FORMAT=c4x timeout 900 python bench.py --config C5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5_vec1.log 2>&1; echo c5=$?
