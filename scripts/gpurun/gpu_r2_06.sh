#!/bin/bash
# round 2, call 6: new GPU tests (NEXT-2 LLG, axis permutation, slab simulation); C3 format A/B;
# ncu --set full of K4 at C5 (B4, U4) and C4 (C4x)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c06; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_llg.py tests/test_gpu_parity.py -q -k "llg or anisotropy or am2 or kalinikos or axis_perm or slab or rk4 or macrospin" -s > $O/pytest_new.log 2>&1
for f in c4x b4 u4; do
  PMFEM_CBOX_FORMAT=$f timeout 600 python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C3_$f.json 2> $O/bench_C3_$f.err
done
PMFEM_CBOX_FORMAT=b4 timeout 300 python scripts/profile_eval.py --config C5 --order 3 --rer-scale 4 --evals 2 > $O/plain_c5.log 2>&1 && \
PMFEM_CBOX_FORMAT=b4 ncu --set full --clock-control none --import-source on -k regex:k4_interp -s 1 -c 1 -o $O/k4_c5_b4 python scripts/profile_eval.py --config C5 --order 3 --rer-scale 4 --evals 2 > $O/ncu_c5_b4.log 2>&1
PMFEM_CBOX_FORMAT=u4 timeout 300 python scripts/profile_eval.py --config C5 --order 3 --rer-scale 4 --evals 2 > $O/plain_c5u.log 2>&1 && \
PMFEM_CBOX_FORMAT=u4 ncu --set full --clock-control none --import-source on -k regex:k4_interp -s 1 -c 1 -o $O/k4_c5_u4 python scripts/profile_eval.py --config C5 --order 3 --rer-scale 4 --evals 2 > $O/ncu_c5_u4.log 2>&1
PMFEM_CBOX_FORMAT=c4x timeout 300 python scripts/profile_eval.py --config C4 --order 3 --rer-scale 4 --evals 2 > $O/plain_c4.log 2>&1 && \
PMFEM_CBOX_FORMAT=c4x ncu --set full --clock-control none --import-source on -k regex:k4_interp -s 1 -c 1 -o $O/k4_c4_c4x python scripts/profile_eval.py --config C4 --order 3 --rer-scale 4 --evals 2 > $O/ncu_c4_c4x.log 2>&1
