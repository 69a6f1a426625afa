#!/bin/bash
# One GPU round-trip: smoke, GPU parity tests, bench per sweep family.
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
summ() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], 'value %.0f GB/s' % d['value'], 'roof %.0f (%.2f)' % (d['roofline']['achieved'], d['roofline']['frac']), 'iccg %.2f ms it %d' % (d['iccg']['time_to_solution_ms'], d['iccg']['iterations']), 'e2e %.0f' % d['e2e']['value'], [ (p['staged'],p['warps'],p['grid'],p['max_slots']) for p in d['roofline']['phases']])
" $1 $2; }
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench_rc=$?
summ gpurun_out/bench.log default
for mode in ${SWEEP_MODES:-simple}; do
  TB_SWEEP=$mode timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$mode.log 2>&1
  summ gpurun_out/bench_$mode.log $mode
done
for cfg in ${RING_CFGS}; do
  R=${cfg%:*}; W=${cfg#*:}
  TB_RING_R=$R TB_RING_WARPS=$W timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r$R_w$W.log 2>&1
  summ gpurun_out/bench_r$R_w$W.log ring_R${R}_W${W}
done
