# Text-input kernel: GPU parity tests + bench lines of the text paths beside the packed ones.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_text.py -x -q > gpurun_out/text_tests.log 2>&1; tail -15 gpurun_out/text_tests.log
for c in ${CFGS:-2 3 4 5}; do
  for path in fused text list text-list; do
    timeout 600 python bench.py --config $c --path $path --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>>gpurun_out/text_bench.err | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms']
print('cfg$c $path'.ljust(16), 'value %.1f' % d['value'], 'ms %.4f' % d['ms_per_step'], {a: round(b, 4) for a, b in k.items() if isinstance(b, float)}, 'frac %.3f' % d['roofline']['frac'], 'matches', d['config']['matches_per_step'])"
  done
done
