#!/bin/bash
# Round evidence on one GPU: tests, smoke, bench (+reference arm), ncu launch
# list of the bench command, one full ncu capture of the dominant kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
# launch list: the bench command (short) under ncu, per-kernel device time
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
# full capture of the dominant kernel (persistent precond launch)
python scripts/prof_sweep.py 2 4 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pcg_persistent -s 2 -c 1 \
    -o gpurun_out/persistent_full -f python scripts/prof_sweep.py 2 4 > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
