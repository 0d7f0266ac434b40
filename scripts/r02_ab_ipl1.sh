# 1024-position kernels at 32 warps: one vs two drain items per lane (cfg4, cfg5).
tag=${1:-r02af}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
bash scripts/ab_libs.sh ${tag} 2 "4 5" base w32ipl1
