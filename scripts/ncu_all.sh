# usage: bash scripts/ncu_all.sh <tag> [bench args] -- launch list + one --set full capture per kernel
tag=$1; shift
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/launches_${tag}.log 2>&1
for k in pack_kernel match_kernel compact_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/${k}_${tag} -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_${k}_${tag}.log 2>&1
done
