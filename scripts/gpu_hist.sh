cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/hist_check.py 3 2>&1 | tail -4
TB_DATAFLOW=0 python scripts/hist_check.py 2 2>&1 | tail -3
TB_PERSIST=0 python scripts/hist_check.py 2 2>&1 | tail -3
