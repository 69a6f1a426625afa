#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
python scripts/trace_iter.py 2 2>&1 | tail -5
TB_FUSE_RZ=0 python scripts/trace_iter.py 2 2>&1 | tail -5
done
timeout 300 python scripts/ab.py 2 "fuse:" 2>&1 | tail -1
TB_FUSE_RZ=0 timeout 300 python scripts/ab.py 2 "nofuse:" 2>&1 | tail -1
