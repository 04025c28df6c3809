set -x
export PMFEM_VERBOSE=1
timeout 600 cuda-gdb -batch -ex run -ex bt --args python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/gdb.log 2>&1; echo gdb=$?
