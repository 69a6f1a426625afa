#!/bin/bash
# r03h: L2 evict-first policy on the TMA SpMV's matrix stream: A/B (variant library without the hint) + ICCG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 2 3 4 c5:512; do
  echo "== $c hint" ; timeout 900 python scripts/spmv_ab.py $c "hint:" 2>&1 | tail -1
  echo "== $c nohint"; scripts/with_variant.sh nohint timeout 900 python scripts/spmv_ab.py $c "nohint:" 2>&1 | tail -1
done > gpurun_out/r03h_spmv_ab.log 2>&1
cat gpurun_out/r03h_spmv_ab.log
timeout 900 python -m pytest tests/test_gpu_spmv_contract.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
