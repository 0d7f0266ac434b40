# usage: bash scripts/ab.sh [bench args] -- runs bench.py with the default lib and each alt lib
for lib in "" $(ls paper_1811_10498_b200/_lib/alt/*.so 2>/dev/null); do
  echo "== lib: ${lib:-default}"
  PFAC_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e "$@" | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value',round(d['value'],1),'ms',round(d['ms_per_step'],4),{k:(round(v,4) if v is not None else None) for k,v in d['kernels_ms'].items()},'match_frac',round(d['roofline']['frac'],4))"
done
