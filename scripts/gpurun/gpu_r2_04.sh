#!/bin/bash
# round 2, call 4: PGF fix; full GPU suite; SEG vs packed C_box formats; K4 group sizes; C4 setup
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c04; mkdir -p $O
timeout 600 python scripts/diag_parity.py R1p2 Y1p2 > $O/diag.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --maxfail=20 > $O/pytest.log 2>&1
for f in seg b4; do
  for c in C2 C5; do
    PMFEM_CBOX_FORMAT=$f timeout 600 python bench.py --config $c --order 3 --rer-scale 4 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_${c}_$f.json 2> $O/bench_${c}_$f.err
  done
done
for g in 8 32; do
  PMFEM_K4_GROUP=$g timeout 600 python bench.py --config C5 --order 3 --rer-scale 4 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C5_seg_g$g.json 2> $O/bench_C5_seg_g$g.err
done
PMFEM_VERBOSE=1 timeout 1200 python bench.py --config C4 --order 3 --rer-scale 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C4_seg.json 2> $O/bench_C4_seg.err
