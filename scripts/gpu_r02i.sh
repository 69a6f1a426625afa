#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for c in 4 3; do
  timeout 600 python scripts/ab.py $c "default:" "perphase:TB_PERSIST=0" > gpurun_out/r02i_ab_c$c.log 2>&1
  echo "== config $c rc=$?"; tail -4 gpurun_out/r02i_ab_c$c.log
done
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_bench_c4.log 2>&1
TB_PERSIST=0 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_bench_c4_pp.log 2>&1
