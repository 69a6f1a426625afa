#!/bin/bash
# r03m: flow kernel block-size test; per-kernel launch list of a config-5 ICCG solve (host-polled split path)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -x -k "flow_kernel" 2>&1 | tail -3
TB_PCG_NOGRAPH=8 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
    --log-file gpurun_out/r03m_iccg_launches_c5.csv python scripts/iccg_launches.py 5 > gpurun_out/r03m_ncu.log 2>&1
tail -2 gpurun_out/r03m_ncu.log
python scripts/launch_table.py gpurun_out/r03m_iccg_launches_c5.csv 2>&1 | head -20
