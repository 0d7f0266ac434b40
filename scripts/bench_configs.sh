# bench every config on one GPU (fused and separate paths); JSON lines into gpurun_out/configs_<tag>.jsonl
tag=${1:-r01}
out=gpurun_out/configs_${tag}.jsonl; : > $out
for c in 1 2 3 4 5; do
  for path in fused separate; do
    timeout 900 python bench.py --config $c --path $path --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/cfg${c}_${path}.err | grep '^{' >> $out || echo "cfg$c $path failed" >> $out
  done
done
python - <<PY
import json
for l in open("$out"):
    if not l.startswith("{"): print(l.strip()); continue
    d = json.loads(l)
    print(d["config"]["workload"][:5], d["path"], round(d["value"],1), "Gb/s step", round(d["ms_per_step"],4), "ms",
          {k: (round(v,4) if isinstance(v,float) else v) for k,v in d["kernels_ms"].items()}, "match_frac", round(d["roofline"]["frac"],3))
PY
