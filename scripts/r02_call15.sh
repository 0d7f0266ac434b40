tag=${1:-r02n}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/match_text_cfg${c}_${tag} -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
for m in 1 2; do
  timeout 600 python bench.py --config 4 --text-kernel $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' > gpurun_out/mode_cfg4_m${m}_${tag}.json
  python -c "import json;d=json.load(open('gpurun_out/mode_cfg4_m${m}_${tag}.json'));print('cfg4 mode $m', round(d['ms_per_step'],4))"
done
bash scripts/ab_libs.sh ${tag} 2 "3 4" base k2max10
