#!/bin/bash
# ncu capture of the sweep kernels on config 2 (TAG names the output).
cd $GRAFT_REPO_ROOT
TAG=${TAG:-reg}
python scripts/prof_sweep.py 2 4 > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --cache-control none --clock-control none --import-source on -k regex:sweep -s 8 -c 4 \
    -o gpurun_out/sweep_$TAG -f python scripts/prof_sweep.py 2 4 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
cat gpurun_out/prof_plain_$TAG.log
