#!/bin/bash
# r03r: operand-prefetch variant of the flow kernel (columns one stage ahead, L2 prefetch of the next step's gathers)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python scripts/ab.py 5 "ring:TB_FLOW2_OPF=0" "opf:TB_FLOW2_OPF=1" > gpurun_out/r03r_ab_c5.log 2>&1; tail -4 gpurun_out/r03r_ab_c5.log
timeout 900 python scripts/ab.py 2 "ring:TB_FLOW2_OPF=0" "opf:TB_FLOW2_OPF=1" > gpurun_out/r03r_ab_c2.log 2>&1; tail -4 gpurun_out/r03r_ab_c2.log
