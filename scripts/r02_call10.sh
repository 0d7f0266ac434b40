tag=${1:-r02j}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests/test_gpu_text.py -x -q > gpurun_out/tests_${tag}.log 2>&1; tail -1 gpurun_out/tests_${tag}.log
for c in 5 2 3; do for m in 0 1 2; do
  timeout 600 python bench.py --config $c --text-kernel $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' > gpurun_out/mode_cfg${c}_m${m}_${tag}.json
  python -c "import json;d=json.load(open('gpurun_out/mode_cfg${c}_m${m}_${tag}.json'));print('cfg$c mode $m', round(d['ms_per_step'],4), d['path'], d['roofline']['kernel'][:60])"
done; done
bash scripts/ab_libs.sh $tag 2 "4" base ipl3 ipl4
