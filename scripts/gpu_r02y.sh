#!/bin/bash
# r02y: final flow2 (ring only): whole GPU suite, config-5 ncu capture of the flow kernel, hot spots, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02y_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r02y_pytest_gpu.log
ncu --set full --clock-control none --import-source on -k regex:precond_kernel -s 2 -c 1 \
    -o gpurun_out/r02y_precond_c5 python scripts/prof_kernels.py precond c5:512 1 > gpurun_out/r02y_ncu_c5.log 2>&1
tail -1 gpurun_out/r02y_ncu_c5.log
python scripts/ncu_summary.py gpurun_out/r02y_precond_c5.ncu-rep
ncu -i gpurun_out/r02y_precond_c5.ncu-rep --page raw --csv > gpurun_out/r02y_precond_c5_raw.csv
ncu -i gpurun_out/r02y_precond_c5.ncu-rep --page details --csv > gpurun_out/r02y_precond_c5_details.csv
ncu --set full --clock-control none --import-source on -k regex:precond_kernel -s 2 -c 1 \
    -o gpurun_out/r02y_precond_c2 python scripts/prof_kernels.py precond 2 1 > gpurun_out/r02y_ncu_c2.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02y_precond_c2.ncu-rep
ncu -i gpurun_out/r02y_precond_c2.ncu-rep --page raw --csv > gpurun_out/r02y_precond_c2_raw.csv
timeout 1500 python bench.py > gpurun_out/r02y_bench_config5.jsonl 2> gpurun_out/r02y_bench.err; echo bench_rc=$?
cat gpurun_out/r02y_bench_config5.jsonl | cut -c1-1500
