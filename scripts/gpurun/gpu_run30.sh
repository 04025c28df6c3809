# --set full of the fp32 FFT passes of one C2 / C3 evaluation (demangled names: the template argument is in the name)
set -x
export PMFEM_NO_GRAPH=1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fft_.*<float" -c 3 -o gpurun_out/prof_c2_fft -f python scripts/profile_eval.py --evals 1 > gpurun_out/ncu_c2_fft.log 2>&1; echo fft2=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fft_.*<float" -c 3 -o gpurun_out/prof_c3_fft -f python scripts/profile_eval.py --config C3 --evals 1 > gpurun_out/ncu_c3_fft.log 2>&1; echo fft3=$?
