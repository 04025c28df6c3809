#!/bin/bash
# round 2, final call: smoke, the default bench (C4, CPU baseline), the per-config lines, the ncu
# launch list of the default command and a --set full capture of its K4, then the GPU suite
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2final; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in C2 C3 C5; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_to_m4|k1_local|k2_tile|fft_|k4_|k5_grad|k_q4" -c 300 --csv --log-file $O/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_interp_corr -c 1 -o $O/k4_c4_c4x python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_k4.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
