# round-2 first GPU call: smoke, new tests, whole -m gpu suite (minus sanitizer), 2-rank gloo bench,
# per-config bench lines (cfg2/4/5) and ncu --set full of the cfg4 / cfg5 text kernels
tag=${1:-r02a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_${tag}.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/smoke_${tag}.log
timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_multirank.py -x -q > gpurun_out/tests_new_${tag}.log 2>&1; tail -3 gpurun_out/tests_new_${tag}.log
timeout 600 python bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gloo2_${tag}.json 2> gpurun_out/bench_gloo2_${tag}.err; tail -c 600 gpurun_out/bench_gloo2_${tag}.json
for c in 2 4 5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg${c}_${tag}.json 2> gpurun_out/bench_cfg${c}_${tag}.err
  tail -c 400 gpurun_out/bench_cfg${c}_${tag}.json
done
for c in 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/match_text_cfg${c}_${tag} -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cfg${c}_${tag}.log 2>&1
done
timeout 1800 python -m pytest tests -q -m gpu --deselect tests/test_gpu_sanitizer.py > gpurun_out/tests_all_${tag}.log 2>&1; tail -3 gpurun_out/tests_all_${tag}.log
ls gpurun_out
