#!/bin/bash
# r03p: flow kernel as a cooperative launch inside the PCG graph too: solver tests + ICCG timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_gpu_solver_contract.py -m gpu -q -x 2>&1 | tail -2
for c in 2 3 5; do timeout 1200 python scripts/ab.py $c "coop:" > gpurun_out/r03p_ab_c$c.log 2>&1; tail -1 gpurun_out/r03p_ab_c$c.log; done
