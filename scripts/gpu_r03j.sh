#!/bin/bash
# r03j: flow kernel grid size (CTAs per SM) at the small config 2 and at config 3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/ab.py 2 "c5:TB_FLOW2_CTAS=5" "c4:TB_FLOW2_CTAS=4" "c3:TB_FLOW2_CTAS=3" "c2:TB_FLOW2_CTAS=2" > gpurun_out/r03j_ab_c2.log 2>&1; tail -4 gpurun_out/r03j_ab_c2.log
timeout 900 python scripts/ab.py 3 "c4:TB_FLOW2_CTAS=4" "c3:TB_FLOW2_CTAS=3" "c2:TB_FLOW2_CTAS=2" > gpurun_out/r03j_ab_c3.log 2>&1; tail -3 gpurun_out/r03j_ab_c3.log
