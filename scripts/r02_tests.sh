# GPU tests (new boundary / multi-rank / sanitizer first), then the whole -m gpu suite, a 2-rank gloo bench
tag=${1:-r02b}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; tail -1 gpurun_out/smoke_${tag}.log
timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_multirank.py -x -q > gpurun_out/tests_new_${tag}.log 2>&1; tail -3 gpurun_out/tests_new_${tag}.log
timeout 1800 python -m pytest tests/test_gpu_sanitizer.py -q > gpurun_out/tests_san_${tag}.log 2>&1; tail -3 gpurun_out/tests_san_${tag}.log
timeout 1500 python -m pytest tests -q -m gpu --deselect tests/test_gpu_sanitizer.py > gpurun_out/tests_all_${tag}.log 2>&1; tail -3 gpurun_out/tests_all_${tag}.log
timeout 600 python bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gloo2_${tag}.json 2> gpurun_out/bench_gloo2_${tag}.err; tail -c 1500 gpurun_out/bench_gloo2_${tag}.json
