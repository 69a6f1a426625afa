#!/bin/bash
# A/B of prebuilt library variants (scratch_libs/libhbmc_<tag>.so) on config 2 (+ config 5 256^3).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
timeout 300 python scripts/ab.py 2 "main:" 2>&1 | tail -1
for tag in ${VARIANTS}; do
  TB_LIB_OVERRIDE=scratch_libs/libhbmc_$tag.so timeout 300 python scripts/ab.py 2 "$tag:" 2>&1 | tail -1
done
done
