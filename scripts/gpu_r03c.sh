#!/bin/bash
# r03c: flow kernel with long dependency lists (kNN): new test, config 4 A/B, parity suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_full.py -m gpu -q -x -k "flow_kernel" > gpurun_out/r03c_pytest_flow.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r03c_pytest_flow.log
timeout 1200 python scripts/ab.py 4 "noflow:TB_FLOW2=0" "flow:TB_FLOW2=1" > gpurun_out/r03c_ab_c4.log 2>&1; echo ab4 rc=$?
tail -4 gpurun_out/r03c_ab_c4.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x > gpurun_out/r03c_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r03c_pytest.log
