#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_full.py -m gpu -q -x -k "spmv or ic0" > gpurun_out/pytest_new.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_new.log
python scripts/spmv_ab.py 2 "old:TB_SPMV_TMA=0" "tma:" "tma_d6:TB_SPMV_D=6,TB_SPMV_KB=200" "tma_s4:TB_SPMV_S=4" "tma_s16:TB_SPMV_S=16,TB_SPMV_KB=200" 2>&1 | tail -5
python scripts/spmv_ab.py c5:256 "old:TB_SPMV_TMA=0" "tma:" "tma_d6:TB_SPMV_D=6,TB_SPMV_KB=200" 2>&1 | tail -3
python scripts/spmv_ab.py 3 "old:TB_SPMV_TMA=0" "tma:" 2>&1 | tail -2
python scripts/spmv_ab.py 4 "old:TB_SPMV_TMA=0" "tma:" 2>&1 | tail -2
