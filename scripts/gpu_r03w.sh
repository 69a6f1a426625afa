#!/bin/bash
# r03w: step loop split by copy source (compile-time: current vs next item)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 5 2 3; do timeout 1200 python scripts/ab.py $c "imm:" > gpurun_out/r03w_ab_c$c.log 2>&1; tail -1 gpurun_out/r03w_ab_c$c.log; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x 2>&1 | tail -2
