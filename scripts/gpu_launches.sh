#!/bin/bash
# Launch list (per-kernel device time) of one ICCG solve, host-polled PCG mode.
cd $GRAFT_REPO_ROOT
CFG=${CFG:-2}
TB_PCG_NOGRAPH=8 python scripts/iccg_launches.py $CFG > gpurun_out/iccg_plain.log 2>&1 && \
TB_PCG_NOGRAPH=8 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/iccg_launches_c$CFG.csv python scripts/iccg_launches.py $CFG \
    > gpurun_out/iccg_ncu.log 2>&1
echo rc=$?
cat gpurun_out/iccg_plain.log
