#!/bin/bash
# r02o: final-tree evidence on one B200: tests, smoke, default bench (config 5),
# reference arm, launch list of the bench command.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02o_pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/r02o_pytest_gpu.log | tail -2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o_smoke.log 2>&1; echo smoke_rc=$?
tail -1 gpurun_out/r02o_smoke.log
timeout 1500 python bench.py > gpurun_out/r02o_bench_config5.jsonl 2> gpurun_out/r02o_bench.err; echo bench_rc=$?
timeout 1500 python bench.py --impl reference > gpurun_out/r02o_bench_reference_config5.jsonl 2> gpurun_out/r02o_bench_ref.err; echo ref_rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02o_bench_launches_config5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r02o_ncu_launches.log 2>&1; echo launches_rc=$?
