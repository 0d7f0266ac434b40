tag=${1:-r02i}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 2400 python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_sanitizer.py > gpurun_out/tests_all_${tag}.log 2>&1; tail -2 gpurun_out/tests_all_${tag}.log
bash scripts/ab_libs.sh $tag 2 "2 3 4 5" base r01 chain16 noend nolog
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/match_text_cfg4_${tag} -f python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cfg4_${tag}.log 2>&1
