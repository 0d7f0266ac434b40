# Full evidence pass for one tag: tests, default bench (with cpu_baseline + e2e), reference arm,
# launch list + ncu captures of the kernels, clocks during the bench.
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_${tag}.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/smi_${tag}.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; tail -1 gpurun_out/smoke_${tag}.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_${tag}.log 2>&1; tail -3 gpurun_out/gpu_tests_${tag}.log
timeout 900 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; cat gpurun_out/bench_${tag}.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_${tag}.json 2>&1; tail -1 gpurun_out/bench_ref_${tag}.json
bash scripts/ncu_all.sh ${tag}
# FASTA-like text through the default (text) path and the packed BAR path
for p in text fused; do timeout 300 python bench.py --barriers 80 --path $p --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' >> gpurun_out/bench_barriers_${tag}.jsonl; done
