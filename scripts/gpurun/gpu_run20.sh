# round-1 session 3: K2 tile-size exploration, C4 bench, LLG C5 bench
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
for t in 8,8,8 8,8,4 8,4,4 16,8,4; do
PMFEM_K2_TILE=$t timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_c2_t$t.log 2>&1; echo c2_$t=$?
done
for t in 16,16,8 16,8,8 8,8,8 32,8,8; do
PMFEM_K2_TILE=$t timeout 600 python bench.py --config C3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3_t$t.log 2>&1; echo c3_$t=$?
done
timeout 900 python scripts/bench_llg.py > gpurun_out/bench_llg.log 2>&1; echo llg=$?
timeout 2400 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo c4=$?
