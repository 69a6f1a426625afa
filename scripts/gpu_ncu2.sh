#!/bin/bash
# ncu --set full of the TMA SpMV (config 2, config 5 at 256^3) and the persistent precond at config 5 256^3.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/prof_kernels.py spmv 2 > gpurun_out/pk_spmv2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 2 -c 1 \
  -o gpurun_out/spmv_tma_c2 -f python scripts/prof_kernels.py spmv 2 > gpurun_out/ncu_spmv2.log 2>&1; echo spmv2_rc=$?
python scripts/prof_kernels.py spmv c5:256 > gpurun_out/pk_spmv5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 2 -c 1 \
  -o gpurun_out/spmv_tma_c5_256 -f python scripts/prof_kernels.py spmv c5:256 > gpurun_out/ncu_spmv5.log 2>&1; echo spmv5_rc=$?
python scripts/prof_kernels.py precond c5:256 > gpurun_out/pk_pre5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_persistent -s 2 -c 1 \
  -o gpurun_out/precond_c5_256 -f python scripts/prof_kernels.py precond c5:256 > gpurun_out/ncu_pre5.log 2>&1; echo pre5_rc=$?
tail -2 gpurun_out/ncu_*.log
