# Round-2 final evidence on the final tree: GPU suite, the default bench line, one line per config
# (cfg1..cfg5), FASTA and list-only lines, the reference arm, the ncu launch list of the default
# command and ncu --set full of the text kernel on cfg2..cfg5 (summaries only; reports removed).
tag=${1:-r02f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/smi_${tag}.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 2400 python -m pytest tests -q -m gpu -rfs > gpurun_out/tests_${tag}.log 2>&1; tail -3 gpurun_out/tests_${tag}.log
timeout 900 python bench.py > gpurun_out/bench_default_${tag}.json 2> gpurun_out/bench_default_${tag}.err; tail -c 300 gpurun_out/bench_default_${tag}.json
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/bench_cfg${c}_${tag}.json
  python -c "import json;d=json.load(open('gpurun_out/bench_cfg${c}_${tag}.json'));print('cfg$c', round(d['ms_per_step'],4), round(d['value'],1), round(d['roofline']['frac'],3), d['roofline']['kernel'])"
done
timeout 600 python bench.py --config 2 --barriers 80 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' > gpurun_out/bench_cfg2_fasta_${tag}.json
for c in 2 5; do
  timeout 600 python bench.py --config $c --path text-list --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' > gpurun_out/bench_cfg${c}_list_${tag}.json
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | grep '^{' > gpurun_out/bench_reference_${tag}.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${tag}.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo launches rc $?
bash scripts/r02_ncu_full.sh ${tag} "2 3 4 5"
ls gpurun_out | grep ${tag} | wc -l
