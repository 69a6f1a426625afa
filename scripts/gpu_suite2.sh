#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['spmv']['achieved'], d['spmv']['frac'], d['e2e']['value'], d['iccg'])"
python scripts/spmv_ab.py 3 "old:TB_SPMV_TMA=0" "s8d2:TB_SPMV_S=8,TB_SPMV_D=2,TB_SPMV_KB=200" "s16d1:TB_SPMV_S=16,TB_SPMV_D=1,TB_SPMV_KB=200" 2>&1 | tail -3
python scripts/spmv_ab.py 4 "old:TB_SPMV_TMA=0" "s8d2:TB_SPMV_S=8,TB_SPMV_D=2,TB_SPMV_KB=200" "s16d2:TB_SPMV_S=16,TB_SPMV_D=2,TB_SPMV_KB=200" 2>&1 | tail -3
