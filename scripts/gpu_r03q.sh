#!/bin/bash
# r03q: after removing the untested group sweep kernel: whole GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r03q_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r03q_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
