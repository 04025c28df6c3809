#!/bin/bash
# round 2, call 7: U4 with 4 shifted q copies (dense gathers); format A/B on all configs; ncu of K4 U4 at C4
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c07; mkdir -p $O
for c in C2 C5 C3; do
  for f in u4 b4 c4x; do
    PMFEM_CBOX_FORMAT=$f timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_${c}_$f.json 2> $O/bench_${c}_$f.err
  done
done
PMFEM_CBOX_FORMAT=u4 timeout 900 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_u4.json 2> $O/bench_C4_u4.err
PMFEM_CBOX_FORMAT=u4 timeout 300 python scripts/profile_eval.py --config C4 --order 3 --rer-scale 4 --evals 2 > $O/plain_c4.log 2>&1 && \
PMFEM_CBOX_FORMAT=u4 ncu --set full --clock-control none --import-source on -k regex:k4_interp -s 1 -c 1 -o $O/k4_c4_u4 python scripts/profile_eval.py --config C4 --order 3 --rer-scale 4 --evals 2 > $O/ncu_c4_u4.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_setup.py tests/test_gpu_parity.py -q -k "cbox or heff_random" > $O/pytest_cbox.log 2>&1
