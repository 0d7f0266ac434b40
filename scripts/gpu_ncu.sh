# usage: bash scripts/gpu_ncu.sh <tag> [bench args...]
set -x
tag=${1:-r01}; shift
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/launches_${tag}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 3 -c 1 \
  -o gpurun_out/match_${tag} -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_match_${tag}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:compact_kernel -s 3 -c 1 \
  -o gpurun_out/compact_${tag} -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_compact_${tag}.log 2>&1
ls -la gpurun_out
