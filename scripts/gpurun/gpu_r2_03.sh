#!/bin/bash
# round 2, call 3: SEG C_box format (K4 without column indices), R1/Y1 parity diagnosis
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c03; mkdir -p $O
timeout 600 python scripts/diag_parity.py R1p2 Y1p2 C3p1 C2p2 > $O/diag.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_setup.py tests/test_gpu_parity.py -q --maxfail=20 > $O/pytest.log 2>&1
for f in seg b4; do
  PMFEM_CBOX_FORMAT=$f timeout 600 python bench.py --config C5 --order 3 --rer-scale 4 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C5_$f.json 2> $O/bench_C5_$f.err
  PMFEM_CBOX_FORMAT=$f timeout 600 python bench.py --config C2 --order 3 --rer-scale 4 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C2_$f.json 2> $O/bench_C2_$f.err
done
for g in 8 32; do
  PMFEM_K4_GROUP=$g timeout 600 python bench.py --config C5 --order 3 --rer-scale 4 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C5_seg_g$g.json 2> $O/bench_C5_seg_g$g.err
done
PMFEM_VERBOSE=1 timeout 1200 python bench.py --config C4 --order 3 --rer-scale 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C4_seg.json 2> $O/bench_C4_seg.err
