#!/bin/bash
# Final round evidence: full GPU suite, smoke, bench (+ reference arm), ncu launch list of the
# bench command, ncu --set full of the headline kernel (persistent dataflow precond, config 2).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
python scripts/prof_kernels.py precond 2 3 > gpurun_out/pk_pre2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_persistent -s 2 -c 1 \
  -o gpurun_out/precond_c2_final -f python scripts/prof_kernels.py precond 2 3 > gpurun_out/ncu_pre2.log 2>&1; echo full_rc=$?
python scripts/prof_kernels.py spmv 2 3 > gpurun_out/pk_sp2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 2 -c 1 \
  -o gpurun_out/spmv_c2_final -f python scripts/prof_kernels.py spmv 2 3 > gpurun_out/ncu_sp2.log 2>&1; echo full_spmv_rc=$?
