#!/bin/bash
# r03v: final-tree evidence (after the address-instruction trims) on one B200: whole GPU suite, smoke, default bench (config 5) + reference arm,
# launch list of the bench command, all configs table, ncu capture of the config-3 flow kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r03v_pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/r03v_pytest_gpu.log | tail -2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03v_smoke.log 2>&1; echo smoke_rc=$?
tail -1 gpurun_out/r03v_smoke.log
timeout 1500 python bench.py > gpurun_out/r03v_bench_config5.jsonl 2> gpurun_out/r03v_bench.err; echo bench_rc=$?
timeout 1500 python bench.py --impl reference > gpurun_out/r03v_bench_reference_config5.jsonl 2> gpurun_out/r03v_bench_ref.err; echo ref_rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r03v_bench_launches_config5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r03v_ncu_launches.log 2>&1; echo launches_rc=$?
timeout 1500 python scripts/run_all_configs.py 1,2,3,4 gpurun_out/r03v_all_configs.json > gpurun_out/r03v_all_configs.log 2>&1; echo all_rc=$?
ncu --set full --clock-control none --import-source on -k regex:precond_kernel -s 2 -c 1 \
    -o gpurun_out/r03v_precond_c3 python scripts/prof_kernels.py precond 3 1 > gpurun_out/r03v_ncu_c3.log 2>&1
python scripts/ncu_summary.py gpurun_out/r03v_precond_c3.ncu-rep
ncu -i gpurun_out/r03v_precond_c3.ncu-rep --page raw --csv > gpurun_out/r03v_precond_c3_raw.csv
ncu --set full --clock-control none --import-source on -k regex:precond_kernel -s 2 -c 1 \
    -o gpurun_out/r03v_precond_c5 python scripts/prof_kernels.py precond c5:512 1 > gpurun_out/r03v_ncu_c5.log 2>&1
python scripts/ncu_summary.py gpurun_out/r03v_precond_c5.ncu-rep
ncu -i gpurun_out/r03v_precond_c5.ncu-rep --page raw --csv > gpurun_out/r03v_precond_c5_raw.csv
