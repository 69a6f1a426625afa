#!/bin/bash
# r03g: config 5: wavefront item order (TB_FLOW2_LAG) x L2 eviction hints (TB_FLOW2_HINT), 4 plans per process (31 GB each)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python scripts/ab.py 5 "base:TB_FLOW2_LAG=0,TB_FLOW2_HINT=0" "hint:TB_FLOW2_LAG=0,TB_FLOW2_HINT=3" "lag4k:TB_FLOW2_LAG=4096,TB_FLOW2_HINT=0" "lag4k_hint:TB_FLOW2_LAG=4096,TB_FLOW2_HINT=3" > gpurun_out/r03g_ab_c5_a.log 2>&1; echo ab5a rc=$?
tail -8 gpurun_out/r03g_ab_c5_a.log
timeout 1500 python scripts/ab.py 5 "hint:TB_FLOW2_LAG=0,TB_FLOW2_HINT=3" "lag2k_hint:TB_FLOW2_LAG=2048,TB_FLOW2_HINT=3" "lag8k_hint:TB_FLOW2_LAG=8192,TB_FLOW2_HINT=3" "lag4k_h1:TB_FLOW2_LAG=4096,TB_FLOW2_HINT=1" > gpurun_out/r03g_ab_c5_b.log 2>&1; echo ab5b rc=$?
tail -8 gpurun_out/r03g_ab_c5_b.log
