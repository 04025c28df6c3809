# streaming-load hint A/B: default build vs -DPMFEM_STREAM_CS
set -x
for v in default cs; do
if [ $v = cs ]; then export PMFEM_EXTRA_NVCC=-DPMFEM_STREAM_CS; fi
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$v.log 2>&1; echo build=$?
timeout 900 python bench.py --steps 40 --no-cpu-baseline > gpurun_out/bench_c2_$v.log 2>&1; echo c2=$?
timeout 900 python bench.py --config C3 --steps 30 --no-cpu-baseline > gpurun_out/bench_c3_$v.log 2>&1; echo c3=$?
timeout 900 python bench.py --config C5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5_$v.log 2>&1; echo c5=$?
done
