tag=${1:-r02k}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests/test_gpu_text.py tests/test_gpu_list_only.py -x -q > gpurun_out/tests_${tag}.log 2>&1; tail -1 gpurun_out/tests_${tag}.log
bash scripts/ab_libs.sh $tag 2 "2 3 4 5" base nodefer
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -v > gpurun_out/tests_san_${tag}.log 2>&1; tail -7 gpurun_out/tests_san_${tag}.log
cp gpurun_out/sanitizer.log gpurun_out/sanitizer_${tag}.log 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/match_text_cfg4_${tag} -f python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cfg4_${tag}.log 2>&1
