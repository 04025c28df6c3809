#!/bin/bash
# round 2, call 11: NEXT-4 complex Bloch field path parity (normal + checked build), static
# parity re-check after the Z0 / C_box host refactor, Z0 setup timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c11; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_bloch.py -q -s > $O/pytest_bloch.log 2>&1
PMFEM_LIB=checked timeout 900 python -m pytest tests/test_gpu_bloch.py -q -k "C2p2 or R1p2" > $O/pytest_bloch_checked.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "heff_random" > $O/pytest_parity.log 2>&1
