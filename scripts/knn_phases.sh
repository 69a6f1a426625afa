for wr in 24 1000; do TB_WIDE_ROWS=$wr python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print($wr, ' '.join('%s%d:%.0f' % (p['sweep'][0], p['color'], p['avg_us']) for p in d['roofline']['per_phase_kernels']))"; done
