#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "pcg or split or full_config or random or smoke" > gpurun_out/pyt.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pyt.log
python scripts/iccg_ab.py 2 "graph:" "poll4:TB_PCG_SPLIT_POLL=4" "persist:TB_PCG_SPLIT=0" 2>&1 | tail -3
python scripts/iccg_ab.py c5:256 "graph:" "poll4:TB_PCG_SPLIT_POLL=4" "persist:TB_PCG_SPLIT=0" 2>&1 | tail -3
python scripts/iccg_ab.py 1 "graph:" "persist:TB_PCG_SPLIT=0" 2>&1 | tail -2
