# round-1 session 3: --set full of every hot kernel (C2, C3) -- ncu -k matches base names
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_local|k2_tile|k4_interp|k5_grad|fft_x|fft_yz" -s 8 -c 7 -o gpurun_out/prof_c2_all -f python scripts/profile_eval.py --evals 2 > gpurun_out/ncu_c2_all.log 2>&1; echo full2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_local|k2_tile|k4_interp|k5_grad|fft_x|fft_yz" -s 8 -c 7 -o gpurun_out/prof_c3_all -f python scripts/profile_eval.py --config C3 --evals 2 > gpurun_out/ncu_c3_all.log 2>&1; echo full3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k4_interp" -s 1 -c 1 -o gpurun_out/prof_c5_k4 -f python scripts/profile_eval.py --config C5 --evals 2 > gpurun_out/ncu_c5_k4.log 2>&1; echo full5=$?
