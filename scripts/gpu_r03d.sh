#!/bin/bash
# r03d: config 4 (kNN 4M) through the flow kernel (dependency lists up to 734 entries)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python scripts/ab.py 4 "noflow:TB_FLOW2=0" "flow:TB_FLOW2=1" > gpurun_out/r03d_ab_c4.log 2>&1; echo ab4 rc=$?
tail -4 gpurun_out/r03d_ab_c4.log
