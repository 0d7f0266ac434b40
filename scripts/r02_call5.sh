tag=${1:-r02e}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests/test_gpu_text.py -x -q -k "match_log or chain_heads or vs_oracle" > gpurun_out/tests_${tag}.log 2>&1; tail -1 gpurun_out/tests_${tag}.log
bash scripts/ab_libs.sh $tag 2 "2 4 5" base r01 nolog push_ballot nolog_ballot ipl2
