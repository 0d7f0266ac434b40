# L1::no_allocate table loads (J2/HR only, or every table load) vs the L1-allocating ld.global.nc.
tag=${1:-r02y}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
bash scripts/ab_libs.sh ${tag} 2 "4 2 3 5" base j2na tabna
