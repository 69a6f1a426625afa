#!/bin/bash
# r02d: ncu of the lean dataflow precond vs the streamed one, configs 2 and 3
# (reports converted to CSV on the box; the .ncu-rep files stay there)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p /tmp/rep
for c in 2 3; do
  for v in 0 1; do
    TB_STREAM=$v ncu --set full --clock-control none --import-source on \
      -k regex:"pcg_persistent|precond_stream" -s 2 -c 1 -o /tmp/rep/r02d_c${c}_s$v \
      python scripts/prof_kernels.py precond $c 1 > gpurun_out/r02d_c${c}_s$v.log 2>&1
    tail -1 gpurun_out/r02d_c${c}_s$v.log
    ncu -i /tmp/rep/r02d_c${c}_s$v.ncu-rep --page raw --csv > gpurun_out/r02d_c${c}_s${v}_raw.csv
    ncu -i /tmp/rep/r02d_c${c}_s$v.ncu-rep --page details --csv > gpurun_out/r02d_c${c}_s${v}_details.csv
    ncu -i /tmp/rep/r02d_c${c}_s$v.ncu-rep --page source --csv > gpurun_out/r02d_c${c}_s${v}_source.csv
  done
done
ls -la gpurun_out
