#!/bin/bash
# r02t: flow2 v3 (item order: backward ascending inside a color; per-lane L2 line prefetch; release after the next item's first loads)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x > gpurun_out/r02t_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r02t_pytest.log
for c in 2 5; do
  timeout 900 python scripts/ab.py $c "old:TB_FLOW2=0" "f2_nopf:TB_FLOW2_PF=0" "f2_d2:TB_FLOW2_PFD=2" "f2_d4:TB_FLOW2_PFD=4" "f2_d8:TB_FLOW2_PFD=8" > gpurun_out/r02t_ab_c$c.log 2>&1; echo ab$c rc=$?
  tail -5 gpurun_out/r02t_ab_c$c.log
done
for pf in 0 1; do
TB_FLOW2_PF=$pf ncu --set full --clock-control none --import-source on -k regex:precond_kernel -s 2 -c 1 \
    -o gpurun_out/r02t_flow2_pf${pf}_c2 python scripts/prof_kernels.py precond 2 1 > gpurun_out/r02t_ncu_$pf.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02t_flow2_pf${pf}_c2.ncu-rep
done
