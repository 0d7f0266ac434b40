# Session-3: the round-emission text kernel (pfac_set_emit_mode 1): parity, A/B vs runs, then the full
# GPU suite (no -x, failures listed) and ncu --set full per config (reports kept in /tmp on the box,
# summaries in gpurun_out/ and profiles/ copies).
tag=${1:-r02t}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests/test_gpu_text.py -x -q -k "rounds" > gpurun_out/tests_text_rounds_${tag}.log 2>&1; tail -3 gpurun_out/tests_text_rounds_${tag}.log
for c in 2 5 4 3; do
  for e in 0 1 0 1; do
    timeout 300 python bench.py --config $c --emit-mode $e --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2> gpurun_out/ab_emit_cfg${c}_e${e}_${tag}.err | grep '^{' >> gpurun_out/ab_emit_${tag}.jsonl
    python -c "import json;d=[json.loads(l) for l in open('gpurun_out/ab_emit_${tag}.jsonl')][-1];print('cfg$c emit $e', round(d['ms_per_step'],4), round(d['value'],1))"
  done
done
timeout 2400 python -m pytest tests -q -m gpu -rf > gpurun_out/tests_${tag}.log 2>&1; tail -15 gpurun_out/tests_${tag}.log
