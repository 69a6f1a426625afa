#!/bin/bash
# r03y: last check of the round's final tree: whole GPU suite, smoke, default bench + reference arm, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r03y_pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/r03y_pytest_gpu.log | tail -2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03y_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python bench.py > gpurun_out/r03y_bench_config5.jsonl 2> gpurun_out/r03y_bench.err; echo bench_rc=$?
timeout 1500 python bench.py --impl reference > gpurun_out/r03y_bench_reference_config5.jsonl 2> gpurun_out/r03y_bench_ref.err; echo ref_rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r03y_bench_launches_config5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r03y_ncu_launches.log 2>&1; echo launches_rc=$?
timeout 1500 python scripts/run_all_configs.py 1,2,3,4 gpurun_out/r03y_all_configs.json > gpurun_out/r03y_all_configs.log 2>&1; echo all_rc=$?
