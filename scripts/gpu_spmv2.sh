#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_full.py -m gpu -q -x -k "spmv" > gpurun_out/pyt.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pyt.log
python scripts/spmv_ab.py 2 "s8d4:" "s16d2:TB_SPMV_S=16,TB_SPMV_D=2" "s16d3:TB_SPMV_S=16,TB_SPMV_D=3,TB_SPMV_KB=200" "s32d2:TB_SPMV_S=32,TB_SPMV_D=2,TB_SPMV_KB=200" "s8d3:TB_SPMV_D=3" "old:TB_SPMV_TMA=0" 2>&1 | tail -6
python scripts/spmv_ab.py c5:256 "s8d4:" "s16d2:TB_SPMV_S=16,TB_SPMV_D=2" "s16d3:TB_SPMV_S=16,TB_SPMV_D=3,TB_SPMV_KB=200" "s8d3:TB_SPMV_D=3" 2>&1 | tail -4
