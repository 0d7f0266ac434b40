# usage: bash scripts/ncu_match.sh <tag> [bench args]  -- one ncu --set full capture of the match kernel
tag=$1; shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 3 -c 1 \
  -o gpurun_out/match_${tag} -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_match_${tag}.log 2>&1
