# --set full of every hot kernel of one C2 / C3 evaluation (graph off so each kernel is a plain launch)
set -x
export PMFEM_NO_GRAPH=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_local|k2_tile|k4_interp|k5_grad|fft_.*float" -c 7 -o gpurun_out/prof_c2_all -f python scripts/profile_eval.py --evals 1 > gpurun_out/ncu_c2_all.log 2>&1; echo full2=$?
python scripts/ncu_traffic.py --rep gpurun_out/prof_c2_all.ncu-rep --config C2 --note "run29, commit 6575840+" > gpurun_out/traffic_c2.log 2>&1; echo traffic=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_local|k2_tile|k4_interp|k5_grad|fft_.*float" -c 7 -o gpurun_out/prof_c3_all -f python scripts/profile_eval.py --config C3 --evals 1 > gpurun_out/ncu_c3_all.log 2>&1; echo full3=$?
python scripts/ncu_traffic.py --rep gpurun_out/prof_c3_all.ncu-rep --config C3 --note "run29, commit 6575840+" > gpurun_out/traffic_c3.log 2>&1; echo traffic=$?
cp profiles/traffic.json gpurun_out/traffic.json
