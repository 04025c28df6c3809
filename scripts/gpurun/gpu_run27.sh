# batched FFT loads (default now) + __ldcs K1/K5 streams; A/B: PMFEM_YZ_HALF=1, PMFEM_YZ_THREADS=1024, -DPMFEM_K2_UNROLL
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_default.log 2>&1; echo build=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
B="timeout 900 python bench.py --no-cpu-baseline"
$B --config C3 --steps 30 > gpurun_out/c3_base.log 2>&1; echo $?
PMFEM_YZ_HALF=1 $B --config C3 --steps 30 > gpurun_out/c3_half.log 2>&1; echo $?
PMFEM_YZ_THREADS=1024 $B --config C3 --steps 30 > gpurun_out/c3_t1024.log 2>&1; echo $?
$B --steps 40 > gpurun_out/c2_base.log 2>&1; echo $?
PMFEM_YZ_HALF=1 $B --steps 40 > gpurun_out/c2_half.log 2>&1; echo $?
$B --config C5 --steps 20 > gpurun_out/c5_base.log 2>&1; echo $?
export PMFEM_EXTRA_NVCC=-DPMFEM_K2_UNROLL
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_unroll.log 2>&1; echo build=$?
PMFEM_YZ_HALF=1 $B --config C3 --steps 30 > gpurun_out/c3_unroll_half.log 2>&1; echo $?
$B --steps 40 > gpurun_out/c2_unroll.log 2>&1; echo $?
unset PMFEM_EXTRA_NVCC
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_default2.log 2>&1; echo build=$?
$B --config C4 --steps 10 --warmup 3 > gpurun_out/c4_base.log 2>&1; echo $?
