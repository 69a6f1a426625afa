#!/bin/bash
# r02p: re-entry check: GPU tests on the restored tree + the reference's own
# tests against the public API (baseline/_ref is a git-ignored copy).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02p_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r02p_pytest_gpu.log
bash scripts/gpu_refsuite.sh gpurun_out/r02p_reference_suite_against_public_api.txt
