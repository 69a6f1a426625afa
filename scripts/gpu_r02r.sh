#!/bin/bash
# r02r: flow2 with / without the L2 bulk prefetch vs the persistent dataflow kernel; ncu of both flow2 modes (config 2) 
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 2 5; do
  timeout 900 python scripts/ab.py $c "old:TB_FLOW2=0" "flow2pf:TB_FLOW2=1,TB_FLOW2_PF=1" "flow2:TB_FLOW2=1,TB_FLOW2_PF=0" > gpurun_out/r02r_ab_c$c.log 2>&1; echo ab$c rc=$?
  tail -3 gpurun_out/r02r_ab_c$c.log
done
for pf in 0 1; do
TB_FLOW2_PF=$pf ncu --set full --clock-control none --import-source on -k regex:precond_kernel -s 2 -c 1 \
    -o gpurun_out/r02r_flow2_pf${pf}_c2 python scripts/prof_kernels.py precond 2 1 > gpurun_out/r02r_ncu_$pf.log 2>&1
tail -1 gpurun_out/r02r_ncu_$pf.log
python scripts/ncu_summary.py gpurun_out/r02r_flow2_pf${pf}_c2.ncu-rep
done
TB_FLOW2=0 ncu --set full --clock-control none --import-source on -k regex:pcg_persistent -s 2 -c 1 \
    -o gpurun_out/r02r_old_c2 python scripts/prof_kernels.py precond 2 1 > gpurun_out/r02r_ncu_old.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02r_old_c2.ncu-rep
