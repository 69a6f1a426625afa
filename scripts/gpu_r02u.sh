#!/bin/bash
# r02u: flow2 v4 (nested chain branches, no prefetch code) and its occupancy variants (3 / 4 CTAs per SM with spills)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x > gpurun_out/r02u_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r02u_pytest.log
for c in 2 5; do
  timeout 900 python scripts/ab.py $c "old:TB_FLOW2=0" "flow2:TB_FLOW2=1" > gpurun_out/r02u_ab_c$c.log 2>&1; echo ab$c rc=$?
  tail -2 gpurun_out/r02u_ab_c$c.log
  for m in 3 4; do
    scripts/with_variant.sh minb$m timeout 900 python scripts/ab.py $c "flow2_minb$m:TB_FLOW2=1" > gpurun_out/r02u_ab_c${c}_minb$m.log 2>&1
    tail -1 gpurun_out/r02u_ab_c${c}_minb$m.log
  done
done
ncu --set full --clock-control none --import-source on -k regex:precond_kernel -s 2 -c 1 \
    -o gpurun_out/r02u_flow2_c2 python scripts/prof_kernels.py precond 2 1 > gpurun_out/r02u_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02u_flow2_c2.ncu-rep
