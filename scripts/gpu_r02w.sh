#!/bin/bash
# r02w: flow2 ring variant (cp.async shared-memory ring of static operands) vs register ping-pong vs the persistent dataflow kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x > gpurun_out/r02w_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r02w_pytest.log
for c in 2 5; do
  timeout 1200 python scripts/ab.py $c "old:TB_FLOW2=0" "regs:TB_FLOW2_RING=0" "ring3:TB_FLOW2_D=3" "ring4:TB_FLOW2_D=4" "ring3c4:TB_FLOW2_D=3,TB_FLOW2_CTAS=4" > gpurun_out/r02w_ab_c$c.log 2>&1; echo ab$c rc=$?
  grep -v "bitwise vs old: True" gpurun_out/r02w_ab_c$c.log | tail -6
done
ncu --set full --clock-control none --import-source on -k regex:ring_kernel -s 2 -c 1 \
    -o gpurun_out/r02w_ring3_c2 python scripts/prof_kernels.py precond 2 1 > gpurun_out/r02w_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02w_ring3_c2.ncu-rep
