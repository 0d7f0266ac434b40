# round-2 first probe: baseline bench on cfg2/cfg4/cfg5 + ncu --set full of the cfg4 and cfg5 text kernels
tag=${1:-r02a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_${tag}.txt
for c in 2 4 5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg${c}_${tag}.json 2> gpurun_out/bench_cfg${c}_${tag}.err
done
for c in 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/match_text_cfg${c}_${tag} -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cfg${c}_${tag}.log 2>&1
done
ls -la gpurun_out
