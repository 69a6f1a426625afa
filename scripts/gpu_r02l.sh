#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p /tmp/rep
# phase b0 of the 3rd application: 2 x 30 warm-up launches + 29 -> launch index 89
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 89 -c 1 \
  -o /tmp/rep/c4_b0 python scripts/prof_kernels.py precond 4 1 > gpurun_out/r02l_ncu.log 2>&1
tail -1 gpurun_out/r02l_ncu.log
ncu -i /tmp/rep/c4_b0.ncu-rep --page raw --csv > gpurun_out/r02l_c4_b0_raw.csv
ncu -i /tmp/rep/c4_b0.ncu-rep --page source --csv > gpurun_out/r02l_c4_b0_source.csv
