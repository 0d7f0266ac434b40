# CTA size of the 1024-position-slice text kernels (warps vs the L1 left by shared memory): cfg4, cfg5.
tag=${1:-r02x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
bash scripts/ab_libs.sh ${tag} 2 "4 5" base mt1k mt1k640 mt1k512
