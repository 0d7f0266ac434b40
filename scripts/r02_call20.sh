# JPRE follow-up: is the loss the shared-memory carve-out (probe: buffer allocated, unused) or the prefetch itself?
tag=${1:-r02w}
mkdir -p gpurun_out
bash scripts/ab_libs.sh ${tag} 2 "4" nojpre jpre_probe jpre4 base
