#!/bin/bash
# r02v: timing probes of flow2 (not bitwise): no operand loads / no value stream / no global operand loads
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 2 5; do
  for m in 1 2 3; do
    scripts/with_variant.sh probe$m timeout 900 python scripts/ab.py $c "probe$m:TB_FLOW2=1" > gpurun_out/r02v_ab_c${c}_probe$m.log 2>&1
    tail -1 gpurun_out/r02v_ab_c${c}_probe$m.log
  done
done
