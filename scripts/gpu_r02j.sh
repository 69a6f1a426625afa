#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for c in 4 3; do
  timeout 600 python scripts/ab.py $c "default:" "perphase:TB_PERSIST=0" > gpurun_out/r02j_ab_c$c.log 2>&1
  echo "== config $c rc=$?"; tail -4 gpurun_out/r02j_ab_c$c.log
done
TB_PERSIST=0 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench_c4_pp.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02j_bench_c4_pp.log'):
    if l.startswith('{'):
        d=json.loads(l)
        print(' '.join(f"{p['sweep'][0]}{p['color']}:{p['avg_us']:.0f}" for p in d['roofline']['per_phase_kernels']))
PY
