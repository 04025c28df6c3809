# default bench line with the refreshed traffic.json (call 29 capture) + LLG on C5 at the final commit
set -x
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python scripts/bench_llg.py > gpurun_out/bench_llg.log 2>&1; echo llg=$?
