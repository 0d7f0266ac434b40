tag=${1:-r02l}
mkdir -p gpurun_out
rm -f gpurun_out/sanitizer.log
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_sanitizer.py > gpurun_out/tests_all_${tag}.log 2>&1; tail -2 gpurun_out/tests_all_${tag}.log
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -v > gpurun_out/tests_san_${tag}.log 2>&1; tail -7 gpurun_out/tests_san_${tag}.log
cp gpurun_out/sanitizer.log gpurun_out/sanitizer_${tag}.log 2>/dev/null
bash scripts/r02_evidence.sh ${tag}
