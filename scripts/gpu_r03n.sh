#!/bin/bash
# r03n: slice lengths / offsets passed through a warp reduction (uniform registers) vs plain shuffles
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 5 2 3; do
  timeout 1200 python scripts/ab.py $c "uniform:" > gpurun_out/r03n_ab_c${c}_u.log 2>&1; tail -1 gpurun_out/r03n_ab_c${c}_u.log
  scripts/with_variant.sh nouni timeout 1200 python scripts/ab.py $c "plain:" > gpurun_out/r03n_ab_c${c}_p.log 2>&1; tail -1 gpurun_out/r03n_ab_c${c}_p.log
done
