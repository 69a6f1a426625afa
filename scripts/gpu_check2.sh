#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/ab.py 2 "main:" "bar:TB_DATAFLOW=0" 2>&1 | tail -2
python scripts/trace_iter.py 2 2>&1 | tail -5
python scripts/trace_iter.py c5:256 2>&1 | tail -5
