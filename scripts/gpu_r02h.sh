#!/bin/bash
# r02h: config 4 (kNN) evidence: ncu of the precond (barrier-mode persistent)
# and the SpMV, plus the bench line with per-phase timings.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p /tmp/rep
python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_bench_c4.log 2>&1
echo "bench rc=$?"
for k in precond spmv; do
  pat=$([ $k = precond ] && echo "pcg_persistent" || echo "spmv")
  ncu --set full --clock-control none --import-source on -k regex:$pat -s 2 -c 1 \
    -o /tmp/rep/c4_$k python scripts/prof_kernels.py $k 4 1 > gpurun_out/r02h_ncu_$k.log 2>&1
  tail -1 gpurun_out/r02h_ncu_$k.log
  ncu -i /tmp/rep/c4_$k.ncu-rep --page raw --csv > gpurun_out/r02h_${k}_c4_raw.csv
  ncu -i /tmp/rep/c4_$k.ncu-rep --page details --csv > gpurun_out/r02h_${k}_c4_details.csv
  ncu -i /tmp/rep/c4_$k.ncu-rep --page source --csv > gpurun_out/r02h_${k}_c4_source.csv
done
