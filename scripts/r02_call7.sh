tag=${1:-r02g}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests/test_gpu_text.py tests/test_gpu_list_only.py -x -q > gpurun_out/tests_${tag}.log 2>&1; tail -1 gpurun_out/tests_${tag}.log
bash scripts/ab_libs.sh $tag 2 "2 4 5" base r01 nolog ipl1
for c in 4 5; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/match_text_cfg${c}_${tag} -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cfg${c}_${tag}.log 2>&1
done
