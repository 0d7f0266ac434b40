# 32 warps per CTA in the 1024-position text kernels: queue length and drain items per lane.
tag=${1:-r02ad}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
bash scripts/ab_libs.sh ${tag} 2 "4 5" base mt1k_q96 w28q96 w32ipl3 w32ipl4
