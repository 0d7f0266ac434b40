# usage: bash scripts/ncu_all.sh <tag> [bench args] -- launch list + one --set full capture per kernel
tag=$1; shift
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/launches_${tag}.log 2>&1
cap() {  # cap <kernel regex> <out name> <skip> <bench args...>
  local k=$1 name=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/${name}_${tag} -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_${name}_${tag}.log 2>&1
}
# skip counts: the bench's probe pass launches pack + fused match once before the 3 warm-ups
cap match_kernel match_text 4 --path text "$@"
cap pack_kernel pack_kernel 4 --path fused "$@"
cap match_kernel match_fused 4 --path fused "$@"
cap match_kernel match_kernel 4 --path separate "$@"
cap compact_kernel compact_kernel 3 --path separate "$@"
cap match_kernel match_bar 4 --path fused --barriers 80 "$@"
