tag=${1:-r02s}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 5000 python -m pytest tests/test_gpu_sanitizer.py -v > gpurun_out/tests_san_${tag}.log 2>&1; tail -8 gpurun_out/tests_san_${tag}.log
cp gpurun_out/sanitizer.log gpurun_out/sanitizer_${tag}.log 2>/dev/null
