#!/bin/bash
# r02q: item-pipelined dataflow precond (flow2.cuh) A/B vs the persistent dataflow kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x > gpurun_out/r02q_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r02q_pytest.log
for c in 2 5 3; do
  timeout 900 python scripts/ab.py $c "old:TB_FLOW2=0" "flow2:TB_FLOW2=1" > gpurun_out/r02q_ab_c$c.log 2>&1; echo ab$c rc=$?
  cat gpurun_out/r02q_ab_c$c.log | tail -6
done
