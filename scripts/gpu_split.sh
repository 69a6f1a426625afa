#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -x -k "split or spmv" > gpurun_out/pyt.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pyt.log
python scripts/iccg_ab.py 2 "persist:" "split:TB_PCG_SPLIT=1" "split8:TB_PCG_SPLIT=1,TB_PCG_SPLIT_POLL=16" "graph:TB_PERSIST=0" 2>&1 | tail -4
python scripts/iccg_ab.py c5:256 "persist:" "split:TB_PCG_SPLIT=1" "split16:TB_PCG_SPLIT=1,TB_PCG_SPLIT_POLL=16" 2>&1 | tail -3
python scripts/iccg_ab.py 3 "persist:" "split:TB_PCG_SPLIT=1" 2>&1 | tail -2
python scripts/iccg_ab.py 4 "persist:" "split:TB_PCG_SPLIT=1" 2>&1 | tail -2
