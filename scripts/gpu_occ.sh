#!/bin/bash
# Occupancy experiment for the persistent kernel + iteration trace + partitioned bench path.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/trace_iter.py 2 2>&1 | tail -6
for m in 3 4; do
  TB_LIB_OVERRIDE=scratch_libs/libhbmc_m$m.so TB_PERSIST_CTAS=$m timeout 300 python scripts/ab.py 2 "m$m:" 2>&1 | tail -1
  TB_LIB_OVERRIDE=scratch_libs/libhbmc_m$m.so TB_PERSIST_CTAS=$m TB_DATAFLOW=0 timeout 300 python scripts/ab.py 2 "m${m}_bar:" 2>&1 | tail -1
done
timeout 300 python scripts/ab.py 2 "base:" "bar:TB_DATAFLOW=0" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['traffic'], d['spmv'])"
timeout 600 torchrun --standalone --nproc-per-node 1 bench.py --force-partitioned --steps 10 --warmup 3 > gpurun_out/bench_part.log 2>&1; echo part_rc=$?
tail -3 gpurun_out/bench_part.log
