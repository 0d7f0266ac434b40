tag=${1:-r02n}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests/test_gpu_text.py tests/test_gpu_parity.py -x -q -k "nested or vs_oracle or config5 or kmers or edge" > gpurun_out/tests_${tag}.log 2>&1; tail -1 gpurun_out/tests_${tag}.log
for m in 1 2; do
  timeout 600 python bench.py --config 4 --text-kernel $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' > gpurun_out/mode_cfg4_m${m}_${tag}.json
  python -c "import json;d=json.load(open('gpurun_out/mode_cfg4_m${m}_${tag}.json'));print('cfg4 mode $m', round(d['ms_per_step'],4))"
done
bash scripts/ab_libs.sh ${tag}a 2 "2 5" base nofstep
bash scripts/ab_libs.sh ${tag}b 2 "3 4" base k2max10
