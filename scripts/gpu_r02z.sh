#!/bin/bash
# r02z: gather-ahead variant (select-merged in-block operands, 128-register cap) vs the ring kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 5 2; do
  timeout 1200 python scripts/ab.py $c "ring:TB_FLOW2_GA=0" "ga:TB_FLOW2_GA=1" > gpurun_out/r02z_ab_c$c.log 2>&1; echo ab$c rc=$?
  tail -4 gpurun_out/r02z_ab_c$c.log
done
TB_FLOW2_GA=1 ncu --set full --clock-control none --import-source on -k regex:precond_ga_kernel -s 2 -c 1 \
    -o gpurun_out/r02z_ga_c5 python scripts/prof_kernels.py precond c5:256 1 > gpurun_out/r02z_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02z_ga_c5.ncu-rep
