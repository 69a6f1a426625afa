#!/bin/bash
# r02x: ring with gather-ahead and lazy flag publication vs the plain ring
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x > gpurun_out/r02x_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r02x_pytest.log
for c in 2 5; do
  timeout 1200 python scripts/ab.py $c "ring3:TB_FLOW2_GA=0" "ga3:TB_FLOW2_LAZY=0" "ga3lazy:TB_FLOW2_LAZY=1" "ga4lazy:TB_FLOW2_D=4" > gpurun_out/r02x_ab_c$c.log 2>&1; echo ab$c rc=$?
  tail -8 gpurun_out/r02x_ab_c$c.log
done
ncu --set full --clock-control none --import-source on -k regex:ringga_kernel -s 2 -c 1 \
    -o gpurun_out/r02x_ga3_c2 python scripts/prof_kernels.py precond 2 1 > gpurun_out/r02x_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02x_ga3_c2.ncu-rep
