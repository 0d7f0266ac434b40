# Session-3: round emission with relaxed sync (A/B vs runs, and a no-wait probe), then ncu --set full per config.
tag=${1:-r02u}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 600 python -m pytest tests/test_gpu_text.py -x -q -k "rounds and (vs_oracle or match_log or barriers)" > gpurun_out/tests_text_rounds_${tag}.log 2>&1; tail -1 gpurun_out/tests_text_rounds_${tag}.log
for c in 2 5 4; do
  for v in e0 e1 nowait e0 e1 nowait; do
    lib=""; em=0
    [ $v = e1 ] && em=1
    [ $v = nowait ] && em=1 && lib=paper_1811_10498_b200/_lib/alt/libpfac_rnd_nowait.so
    PFAC_LIB=$lib timeout 300 python bench.py --config $c --emit-mode $em --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' > /tmp/l.json
    python -c "import json;d=json.load(open('/tmp/l.json'));d['variant']='$v';print(json.dumps(d))" >> gpurun_out/ab_emit_${tag}.jsonl
    python -c "import json;d=json.load(open('/tmp/l.json'));print('cfg$c $v', round(d['ms_per_step'],4), round(d['value'],1))"
  done
done
bash scripts/r02_ncu_full.sh ${tag} "2 4 5"
