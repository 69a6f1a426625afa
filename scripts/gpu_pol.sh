#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -x -k "split or spmv or full_config_iccg" > gpurun_out/pyt.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pyt.log
for c in 2 3 4; do python scripts/spmv_ab.py $c "default:" "old:TB_SPMV_TMA=0" 2>&1 | tail -2; done
python scripts/iccg_ab.py 3 "default:" "persist:TB_PCG_SPLIT=0" 2>&1 | tail -2
python scripts/iccg_ab.py 4 "default:" 2>&1 | tail -1
