#!/bin/bash
# Round evidence: bench (+reference arm), ncu launch list of the bench command,
# config 5 full size.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
python scripts/run_config5.py 512 5 > gpurun_out/config5_512.log 2>&1 &
pid=$!
while kill -0 $pid 2>/dev/null; do
  rss=$(ps -o rss= -p $pid 2>/dev/null | tr -d ' ')
  if [ -n "$rss" ] && [ "$rss" -gt 170000000 ]; then echo "watchdog: killing $pid"; kill -9 $pid; fi
  sleep 2
done
wait $pid; echo c5_rc=$?
tail -n 1 gpurun_out/config5_512.log
