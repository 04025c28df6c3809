timeout 300 python scripts/dbg_stream.py > gpurun_out/dbg.log 2>&1; echo dbg=$?
