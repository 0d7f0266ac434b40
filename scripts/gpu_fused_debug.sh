timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "not fused and not config2_full and not config5_full" 2>&1 | tail -3
for c in edge cfg1 short shard kmers8; do
  echo "== $c"; timeout 60 python -m pytest tests/test_gpu_parity.py -x -q -k "test_fused_match_compact and $c" 2>&1 | tail -3
done
