# fused / separate / list-only paths on cfg2..cfg5 (digest lines)
for c in ${@:-2 3 4 5}; do
  for path in fused list separate; do
    timeout 600 python bench.py --config $c --path $path --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms']
print('cfg$c $path'.ljust(16), 'value %.1f' % d['value'], 'ms %.4f' % d['ms_per_step'], {a: round(b, 4) for a, b in k.items() if isinstance(b, float)}, 'matches', d['config']['matches_per_step'])"
  done
done
