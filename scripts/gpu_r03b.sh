#!/bin/bash
# r03b: short-slice path of the generalised flow kernel restored to the direct per-step issue: regression check
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 5 2 3; do
  timeout 1200 python scripts/ab.py $c "noflow:TB_FLOW2=0" "flow:TB_FLOW2=1" > gpurun_out/r03b_ab_c$c.log 2>&1; echo ab$c rc=$?
  tail -2 gpurun_out/r03b_ab_c$c.log
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x > gpurun_out/r03b_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r03b_pytest.log
