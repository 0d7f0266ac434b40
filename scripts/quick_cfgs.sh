# quick fused-path bench of the given configs (default 2 and 5): one digest line each
for c in ${@:-2 5}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms']
print('cfg$c', 'value %.1f' % d['value'], 'ms %.4f' % d['ms_per_step'], {a: round(b, 4) for a, b in k.items() if isinstance(b, float)})"
done
