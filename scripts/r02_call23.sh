# Dynamic slice claiming in the 1024-position text kernel (text-kernel mode 3): parity, then A/B vs mode 2.
tag=${1:-r02z}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests/test_gpu_text.py -x -q -k "dyn" > gpurun_out/tests_dyn_${tag}.log 2>&1; tail -3 gpurun_out/tests_dyn_${tag}.log
for c in 5 4 2; do
  for m in 2 3 2 3; do
    timeout 300 python bench.py --config $c --text-kernel $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/dyn_err_${c}_${m}.txt | grep '^{' > /tmp/l.json
    python -c "import json;d=json.load(open('/tmp/l.json'));d['variant']='m$m';print(json.dumps(d))" >> gpurun_out/ab_dyn_${tag}.jsonl
    python -c "import json;d=json.load(open('/tmp/l.json'));print('cfg$c mode $m', round(d['ms_per_step'],4), round(d['value'],1))"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config5_full or config2_full or fasta" > gpurun_out/tests_dynfull_${tag}.log 2>&1; tail -3 gpurun_out/tests_dynfull_${tag}.log
