# usage: bash scripts/ncu_cfg.sh <tag> <config> -- ncu --set full of the fused match kernel on a config
tag=$1; c=$2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
  -o gpurun_out/match_cfg${c}_${tag} -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cfg${c}_${tag}.log 2>&1
python - <<PY
import ctypes
lib = ctypes.CDLL(None)
PY
nvidia-smi -q | grep -i -A2 "l2\|persist" | head -20
