#!/bin/bash
# round 2, call 22: C4x KB=4 A/B at C4; W4 traffic captures (C5, C2); default bench with the CPU
# baseline, the reference arm, and the ncu launch list of the default command
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c22; mkdir -p $O
PMFEM_K4_KB=4 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_kb4.json 2> $O/bench_C4_kb4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_win -c 1 -o $O/k4_c5_w4 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_win -c 1 -o $O/k4_c2_w4 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_to_m4|k1_local|k2_tile|fft_|k4_|k5_grad|k_q4" -c 300 --csv --log-file $O/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
