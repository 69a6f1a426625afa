#!/bin/bash
# Re-entry evidence run: round script + A/B of the sweep scheduling variants.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; free -g >> gpurun_out/gpu.txt
timeout 900 python scripts/ab.py 2 "barrier:TB_DATAFLOW=0" "flow:" "flow_apair:TB_APAIR=1" > gpurun_out/ab.log 2>&1; echo ab_rc=$?
tail -8 gpurun_out/ab.log
bash scripts/gpu_round.sh
