# setup timing breakdown (C3, C5) + torchrun N=1 launch of bench.py
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
PMFEM_VERBOSE=1 timeout 900 python scripts/profile_eval.py --config C3 --evals 1 > gpurun_out/setup_c3.log 2>&1; echo c3=$?
PMFEM_VERBOSE=1 timeout 900 python scripts/profile_eval.py --config C5 --evals 1 > gpurun_out/setup_c5.log 2>&1; echo c5=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_torchrun1.log 2>&1; echo tr=$?
