#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
timeout 300 python scripts/ab.py 2 "pre4:" "old:TB_PRE_CTAS=0" "pre2:TB_PRE_CTAS=2" 2>&1 | tail -3
TB_LIB_OVERRIDE=scratch_libs/libhbmc_pre3.so timeout 300 python scripts/ab.py 2 "pre3:" 2>&1 | tail -1
done
timeout 600 python -m pytest tests -m gpu -q -x -k "pcg or sweep or smoke or full_config_iccg_matches_reference and 2" > gpurun_out/pyt.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pyt.log
