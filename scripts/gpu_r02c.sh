#!/bin/bash
# r02c: A/B of the streamed precond (TB_STREAM=1, default) vs the lean
# dataflow kernel (TB_STREAM=0), bitwise check, per config.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for c in 2 3 5 4; do
  timeout 600 python scripts/ab.py $c "lean:TB_STREAM=0" "stream:TB_STREAM=1" > gpurun_out/r02c_ab_c$c.log 2>&1
  echo "== config $c rc=$?"; tail -4 gpurun_out/r02c_ab_c$c.log
done
