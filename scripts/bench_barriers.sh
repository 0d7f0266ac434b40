# Bench cfg2 without / with barriers (FASTA layout) on both paths + the barrier parity tests.
# Full JSON lines go to gpurun_out/bench_barriers_<tag>.jsonl; a short digest to stdout.
tag=${1:-x}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_barriers.py -x -q 2>&1 | tail -3
out=gpurun_out/bench_barriers_$tag.jsonl
: > $out
for extra in "" "--barriers 80" "--barriers 60 --path separate" "--barriers 80 --config 4" "--config 4"; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $extra 2>&1 | grep '^{' | tee -a $out \
    | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms']
print('$extra'.ljust(32), 'value %.1f' % d['value'], 'ms %.3f' % d['ms_per_step'], 'pack %.3f' % k['pack'],
      'match %.3f' % [v for kk, v in k.items() if kk.startswith('match')][0], 'frac %.3f' % d['roofline']['frac'],
      'e2e %.1f' % d['e2e']['value'], 'matches', d['config']['matches_per_step'])"
done
