# cfg3/cfg4 quick bench (fused) + image info
for c in 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/big_cfg$c.err | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'][:5], round(d['value'],1), 'Gb/s', round(d['ms_per_step'],3), 'ms', {k:(round(v,4) if isinstance(v,float) else v) for k,v in d['kernels_ms'].items()}, 'frac', round(d['roofline']['frac'],3), d['config']['image'])"
done
