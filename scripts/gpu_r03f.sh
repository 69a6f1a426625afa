#!/bin/bash
# r03f: wavefront item order (TB_FLOW2_LAG) and L2 eviction hints (TB_FLOW2_HINT) for the flow kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python scripts/ab.py 5 "base:TB_FLOW2_LAG=0,TB_FLOW2_HINT=0" "hint:TB_FLOW2_LAG=0,TB_FLOW2_HINT=3" "lag4k:TB_FLOW2_LAG=4096,TB_FLOW2_HINT=0" "lag4k_hint:TB_FLOW2_LAG=4096,TB_FLOW2_HINT=3" "lag2k_hint:TB_FLOW2_LAG=2048,TB_FLOW2_HINT=3" "lag8k_hint:TB_FLOW2_LAG=8192,TB_FLOW2_HINT=3" "lag4k_h1:TB_FLOW2_LAG=4096,TB_FLOW2_HINT=1" > gpurun_out/r03f_ab_c5.log 2>&1; echo ab5 rc=$?
tail -14 gpurun_out/r03f_ab_c5.log
timeout 1200 python scripts/ab.py 3 "base:TB_FLOW2_LAG=0,TB_FLOW2_HINT=0" "hint:TB_FLOW2_LAG=0,TB_FLOW2_HINT=3" "lag1k_hint:TB_FLOW2_LAG=1024,TB_FLOW2_HINT=3" "lag512_hint:TB_FLOW2_LAG=512,TB_FLOW2_HINT=3" > gpurun_out/r03f_ab_c3.log 2>&1; echo ab3 rc=$?
tail -8 gpurun_out/r03f_ab_c3.log
timeout 1200 python scripts/ab.py 2 "base:TB_FLOW2_LAG=0,TB_FLOW2_HINT=0" "hint:TB_FLOW2_LAG=0,TB_FLOW2_HINT=3" "h1:TB_FLOW2_LAG=0,TB_FLOW2_HINT=1" > gpurun_out/r03f_ab_c2.log 2>&1; echo ab2 rc=$?
tail -6 gpurun_out/r03f_ab_c2.log
