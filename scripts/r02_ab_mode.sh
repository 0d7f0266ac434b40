# cfg2/cfg3: the 2048-position text kernel (mode 1, 28 warps) vs the 1024-position one (mode 2, 32 warps).
tag=${1:-r02ae}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
for c in 2 3; do
  for m in 1 2 1 2; do
    timeout 300 python bench.py --config $c --text-kernel $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' > /tmp/l.json
    python -c "import json;d=json.load(open('/tmp/l.json'));d['variant']='m$m';print(json.dumps(d))" >> gpurun_out/ab_mode_${tag}.jsonl
    python -c "import json;d=json.load(open('/tmp/l.json'));print('cfg$c mode $m', round(d['ms_per_step'],4), round(d['value'],1))"
  done
done
