# The all-occurrence expansion inside the timed step (cfg2, cfg5) + the plain default for comparison.
tag=${1:-x}
mkdir -p gpurun_out
out=gpurun_out/bench_expand_$tag.jsonl
: > $out
for extra in "" "--all-matches" "--config 5" "--config 5 --all-matches"; do
  timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $extra 2>&1 | grep '^{' | tee -a $out \
    | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms']
print('$extra'.ljust(28), 'value %.1f' % d['value'], 'ms %.3f' % d['ms_per_step'], json.dumps(k))"
done
