# Session-3 first call: full GPU suite, default bench, ncu --set full of the text kernel per config
# (cfg2..cfg5) summarised into profiles/ (ncu_traffic.json, ncu_bounds.json).
tag=${1:-r02s}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/tests_${tag}.log 2>&1; tail -2 gpurun_out/tests_${tag}.log
timeout 600 python bench.py > gpurun_out/bench_default_${tag}.json 2> gpurun_out/bench_default_${tag}.err; tail -c 400 gpurun_out/bench_default_${tag}.json
for c in 2 3 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/match_text_cfg${c}_${tag} -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo ncu cfg$c rc $?
done
python scripts/ncu_config_summary.py gpurun_out/ncu_configs_${tag}.md 2=gpurun_out/match_text_cfg2_${tag}.ncu-rep 3=gpurun_out/match_text_cfg3_${tag}.ncu-rep 4=gpurun_out/match_text_cfg4_${tag}.ncu-rep 5=gpurun_out/match_text_cfg5_${tag}.ncu-rep > gpurun_out/ncu_summary_${tag}.log 2>&1; echo summary rc $?
cp profiles/ncu_bounds.json profiles/ncu_traffic.json gpurun_out/ 2>/dev/null
