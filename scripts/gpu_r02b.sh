#!/bin/bash
# r02b: new GPU tests (ADVICE SpMV fix), then ncu of the config-5 precond and
# SpMV (traffic for the bench's roofline) and the launch list of the bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
python -m pytest tests/test_gpu_spmv_contract.py tests/test_gpu_parity.py -q > gpurun_out/r02b_pytest.log 2>&1
tail -3 gpurun_out/r02b_pytest.log
ncu --set full --clock-control none --import-source on -k regex:pcg_persistent -s 2 -c 1 \
    -o gpurun_out/r02b_precond_c5 python scripts/prof_kernels.py precond c5:512 1 > gpurun_out/r02b_ncu_pre.log 2>&1
tail -2 gpurun_out/r02b_ncu_pre.log
ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 2 -c 1 \
    -o gpurun_out/r02b_spmv_c5 python scripts/prof_kernels.py spmv c5:512 1 > gpurun_out/r02b_ncu_spmv.log 2>&1
tail -2 gpurun_out/r02b_ncu_spmv.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r02b_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r02b_ncu_launches.log 2>&1
tail -2 gpurun_out/r02b_ncu_launches.log
