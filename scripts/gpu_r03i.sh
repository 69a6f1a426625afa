#!/bin/bash
# r03i: L2 evict-first policy on the per-phase lean sweep kernels' factor stream: config 4 (kNN) A/B, parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/ab.py 4 "hint:" > gpurun_out/r03i_ab_c4_hint.log 2>&1; tail -1 gpurun_out/r03i_ab_c4_hint.log
scripts/with_variant.sh leannohint timeout 900 python scripts/ab.py 4 "nohint:" > gpurun_out/r03i_ab_c4_nohint.log 2>&1; tail -1 gpurun_out/r03i_ab_c4_nohint.log
timeout 900 python scripts/ab.py 4 "hint:" > gpurun_out/r03i_ab_c4_hint2.log 2>&1; tail -1 gpurun_out/r03i_ab_c4_hint2.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_gpu_spmv_contract.py -m gpu -q -x 2>&1 | tail -2
