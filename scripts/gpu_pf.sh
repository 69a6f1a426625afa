#!/bin/bash
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
timeout 300 python scripts/ab.py 2 "main:" 2>&1 | tail -1
for v in 1 2 4; do TB_LIB_OVERRIDE=scratch_libs/libhbmc_pf$v.so timeout 300 python scripts/ab.py 2 "pf$v:" 2>&1 | tail -1; done
done
for v in 2; do TB_LIB_OVERRIDE=scratch_libs/libhbmc_pf$v.so python scripts/prof_kernels.py precond c5:256 1 > /dev/null 2>&1; done
python scripts/iccg_ab.py c5:256 "main:" 2>&1 | tail -1
TB_LIB_OVERRIDE=scratch_libs/libhbmc_pf2.so python scripts/iccg_ab.py c5:256 "pf2:" 2>&1 | tail -1
