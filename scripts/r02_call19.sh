# J2 prefetch (cp.async at filter time) in the 1024-position uint32 text kernels: parity, then A/B.
tag=${1:-r02v}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests/test_gpu_text.py -x -q -k "1k" > gpurun_out/tests_text1k_${tag}.log 2>&1; tail -1 gpurun_out/tests_text1k_${tag}.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config3_config4_full and 4 or large_automaton" > gpurun_out/tests_cfg4_${tag}.log 2>&1; tail -1 gpurun_out/tests_cfg4_${tag}.log
bash scripts/ab_libs.sh ${tag} 3 "4" base nojpre
