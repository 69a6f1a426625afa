#!/bin/bash
# Config 5 at 256^3 (proxy with a reference iteration count) and full 512^3,
# under a host-memory watchdog (kill above 170 GB RSS).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
free -g | head -2
for n in ${C5_SIZES:-256 512}; do
  python scripts/run_config5.py $n 5 > gpurun_out/config5_$n.log 2>&1 &
  pid=$!
  while kill -0 $pid 2>/dev/null; do
    rss=$(ps -o rss= -p $pid 2>/dev/null | tr -d ' ')
    if [ -n "$rss" ] && [ "$rss" -gt 170000000 ]; then echo "watchdog: killing $pid at ${rss} KB"; kill -9 $pid; fi
    sleep 2
  done
  wait $pid; echo "n=$n rc=$?"
  tail -4 gpurun_out/config5_$n.log
done
