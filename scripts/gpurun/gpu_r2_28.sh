#!/bin/bash
# round 2, call 28: NEXT-4 complex Bloch path timing next to the static path
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c28; mkdir -p $O
timeout 900 python scripts/bench_bloch.py --config C2 --coarsen 2 > $O/bloch_C2c2.json 2> $O/bloch_C2c2.err
timeout 900 python scripts/bench_bloch.py --config C5 --coarsen 4 > $O/bloch_C5c4.json 2> $O/bloch_C5c4.err
