# CTA size of the 1024-position text kernels with the shared memory kept under the 196-KB carve-out.
tag=${1:-r02ac}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
bash scripts/ab_libs.sh ${tag} 2 "4 5" base mt1k960 mt1k_q96
