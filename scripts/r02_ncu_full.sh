# ncu --set full of the text kernel per config (reports in gpurun_out/ncu_tmp, summarised, then removed
# so gpurun_out stays under the 64 MiB copy-back limit): profiles-ready markdown, ncu_traffic.json /
# ncu_bounds.json (copied to gpurun_out), and the SASS hot spots per report.
# usage: bash scripts/r02_ncu_full.sh <tag> "<configs>" [extra bench args]
tag=$1; cfgs=${2:-"2 3 4 5"}; shift 2; extra="$*"
mkdir -p gpurun_out/ncu_tmp
specs=""
for c in $cfgs; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $extra 2>/dev/null | grep '^{' > gpurun_out/ncu_tmp/bench_cfg${c}_${tag}.json
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/ncu_tmp/match_text_cfg${c}_${tag} -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $extra > /dev/null 2>&1
  echo ncu cfg$c rc $?
  specs="$specs cfg${c}=gpurun_out/ncu_tmp/match_text_cfg${c}_${tag}.ncu-rep"
  python scripts/sass_hot.py gpurun_out/ncu_tmp/match_text_cfg${c}_${tag}.ncu-rep 40 > gpurun_out/sass_hot_cfg${c}_${tag}.txt 2>&1
  ncu -i gpurun_out/ncu_tmp/match_text_cfg${c}_${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_tmp/src_cfg${c}.csv 2>/dev/null
  gzip -c gpurun_out/ncu_tmp/src_cfg${c}.csv > gpurun_out/sass_src_cfg${c}_${tag}.csv.gz
  ncu -i gpurun_out/ncu_tmp/match_text_cfg${c}_${tag}.ncu-rep --page raw --csv > gpurun_out/ncu_raw_cfg${c}_${tag}.csv 2>/dev/null
done
python scripts/ncu_config_summary.py gpurun_out/ncu_configs_${tag}.md $specs > gpurun_out/ncu_summary_${tag}.log 2>&1; echo summary rc $?
cp profiles/ncu_bounds.json gpurun_out/ncu_bounds_${tag}.json; cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_${tag}.json
rm -rf gpurun_out/ncu_tmp/*.ncu-rep gpurun_out/ncu_tmp/src_*.csv
du -sh gpurun_out
