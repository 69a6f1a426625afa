#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "pcg or sweep or full_config or split" > gpurun_out/pyt.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pyt.log
for rep in 1 2; do
timeout 300 python scripts/ab.py 2 "pair:" 2>&1 | tail -1
TB_LIB_OVERRIDE=scratch_libs/libhbmc_nopair.so timeout 300 python scripts/ab.py 2 "nopair:" 2>&1 | tail -1
done
python scripts/iccg_ab.py c5:256 "pair:" 2>&1 | tail -1
TB_LIB_OVERRIDE=scratch_libs/libhbmc_nopair.so python scripts/iccg_ab.py c5:256 "nopair:" 2>&1 | tail -1
python scripts/prof_kernels.py precond c5:256 5 2>&1 | tail -1
