# Round-2 final evidence, part 2 (after the 32-warp 1024-position kernels): GPU suite, bench lines of
# every config, and ncu --set full of the cfg4 / cfg5 text kernels.
tag=${1:-r02g}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 2400 python -m pytest tests -q -m gpu -rfs > gpurun_out/tests_${tag}.log 2>&1; tail -2 gpurun_out/tests_${tag}.log
timeout 900 python bench.py > gpurun_out/bench_default_${tag}.json 2> gpurun_out/bench_default_${tag}.err; tail -c 200 gpurun_out/bench_default_${tag}.json
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/bench_cfg${c}_${tag}.json
  python -c "import json;d=json.load(open('gpurun_out/bench_cfg${c}_${tag}.json'));print('cfg$c', round(d['ms_per_step'],4), round(d['value'],1), round(d['roofline']['frac'],3), d['roofline']['kernel'])"
done
timeout 600 python bench.py --config 5 --path text-list --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' > gpurun_out/bench_cfg5_list_${tag}.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${tag}.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo launches rc $?
bash scripts/r02_ncu_full.sh ${tag} "4 5"
