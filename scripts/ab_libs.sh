# A/B of libpfac builds on one box: bash scripts/ab_libs.sh <tag> <reps> "<configs>" <variant>...
# (variant "base" = the in-tree library; others = paper_1811_10498_b200/_lib/alt/libpfac_<variant>.so)
# -> gpurun_out/ab_<tag>.jsonl (one bench line per run, "variant" added) and a summary on stdout
tag=$1; reps=$2; cfgs=$3; shift 3
mkdir -p gpurun_out
out=gpurun_out/ab_$tag.jsonl; : > $out
for rep in $(seq $reps); do
  for v in "$@"; do
    lib=""; [ "$v" != base ] && lib=paper_1811_10498_b200/_lib/alt/libpfac_$v.so
    for c in $cfgs; do
      PFAC_LIB=$lib timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
        | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['variant']='$v'; print(json.dumps(d))" >> $out
    done
  done
done
python - "$out" <<'PY'
import json, sys, collections
r = collections.defaultdict(list)
for l in open(sys.argv[1]):
    d = json.loads(l); r[(d["variant"], d["config"]["workload"][:4])].append(d["ms_per_step"])
for (v, c), ms in sorted(r.items(), key=lambda x: (x[0][1], x[0][0])):
    print(f"{c} {v:12s} ms/step " + " ".join(f"{m:.4f}" for m in ms))
PY
