# round-2 call 2: NB chain-head J2 entries, scan-based push, per-warp match logs
tag=${1:-r02b}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/smoke_${tag}.log
timeout 900 python -m pytest tests/test_gpu_text.py -x -q -k "match_log or chain_heads" > gpurun_out/tests_new_${tag}.log 2>&1; tail -3 gpurun_out/tests_new_${tag}.log
for c in 2 3 4 5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg${c}_${tag}.json 2> gpurun_out/bench_cfg${c}_${tag}.err
  python -c "import json;d=json.load(open('gpurun_out/bench_cfg${c}_${tag}.json'));print($c, round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
done
timeout 600 python bench.py --config 5 --path fused --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5f_${tag}.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_cfg5f_${tag}.json'));print('5f', round(d['value'],1), round(d['ms_per_step'],4))"
for c in 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/match_text_cfg${c}_${tag} -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cfg${c}_${tag}.log 2>&1
done
timeout 2400 python -m pytest tests -q -m gpu --deselect tests/test_gpu_sanitizer.py > gpurun_out/tests_all_${tag}.log 2>&1; tail -3 gpurun_out/tests_all_${tag}.log
