#!/bin/bash
# round 2, call 31: ncu launch list of the default command at the final K4 setting
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c31; mkdir -p $O
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_to_m4|k1_local|k2_tile|fft_|k4_|k5_grad|k_q4" -c 300 --csv --log-file $O/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
