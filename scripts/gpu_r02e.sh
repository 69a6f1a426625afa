#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for c in 2 3 5; do
  timeout 600 python scripts/ab.py $c "lean:TB_STREAM=0" "stream:TB_STREAM=1" > gpurun_out/r02e_ab_c$c.log 2>&1
  echo "== config $c rc=$?"; tail -4 gpurun_out/r02e_ab_c$c.log
done
mkdir -p /tmp/rep
TB_STREAM=1 ncu --set full --clock-control none --import-source on -k regex:"precond_stream" -s 2 -c 1 \
  -o /tmp/rep/s python scripts/prof_kernels.py precond 2 1 > /dev/null 2>&1
ncu -i /tmp/rep/s.ncu-rep --page raw --csv > gpurun_out/r02e_c2_s1_raw.csv
ncu -i /tmp/rep/s.ncu-rep --page source --csv > gpurun_out/r02e_c2_s1_source.csv
