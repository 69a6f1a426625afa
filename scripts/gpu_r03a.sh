#!/bin/bash
# r03a: flow kernel generalised to long slices (chunked ring stages): config 3 A/B, regression A/B on configs 2, 5, parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x > gpurun_out/r03a_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r03a_pytest.log
for c in 3 2 5 4; do
  timeout 1200 python scripts/ab.py $c "noflow:TB_FLOW2=0" "flow:TB_FLOW2=1" > gpurun_out/r03a_ab_c$c.log 2>&1; echo ab$c rc=$?
  tail -4 gpurun_out/r03a_ab_c$c.log
done
