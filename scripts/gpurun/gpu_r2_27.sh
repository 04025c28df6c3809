#!/bin/bash
# round 2, call 27: C2 / C3 lines again (the final call's showed ~0.2 ms outside the kernels) and the
# reference arm with the library's full-size nnz in its extrapolation
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c27; mkdir -p $O
for c in C2 C3; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
