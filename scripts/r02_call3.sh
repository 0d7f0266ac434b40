# round-2 call 3: coalesced match-log emission/replay; A/B of the push, merged-F and ld.cg table
# variants on cfg2..cfg5 (same box); parity of the ablation builds; ncu of cfg5
tag=${1:-r02c}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 1200 python -m pytest tests/test_gpu_text.py tests/test_gpu_list_only.py -x -q > gpurun_out/tests_text_${tag}.log 2>&1; tail -2 gpurun_out/tests_text_${tag}.log
out=gpurun_out/ab_${tag}.jsonl; : > $out
for rep in 1 2; do
for lib in "" paper_1811_10498_b200/_lib/alt/libpfac_push_ballot.so paper_1811_10498_b200/_lib/alt/libpfac_merged_f.so paper_1811_10498_b200/_lib/alt/libpfac_tab_cg.so; do
  name=$(basename "${lib:-libpfac_base.so}" .so); name=${name#libpfac_}
  for c in 2 3 4 5; do
    PFAC_LIB=$lib timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
      | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['variant']='$name'; print(json.dumps(d))" >> $out
  done
done
done
TAG=$tag python - <<'PY'
import json
for l in open("gpurun_out/ab_"+__import__("os").environ["TAG"]+".jsonl"):
    d=json.loads(l); print(d["variant"], d["config"]["workload"][:5], round(d["value"],1), round(d["ms_per_step"],4))
PY
for v in merged_f tab_cg; do
  PFAC_LIB=paper_1811_10498_b200/_lib/alt/libpfac_$v.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_text.py -q \
    -k "edge_sizes or all_kmers or config2_full or config5_full or fused_match_compact or large_automaton or config1 or vs_oracle or chain_heads or nested" > gpurun_out/tests_abl_${v}_${tag}.log 2>&1
  echo $v; tail -1 gpurun_out/tests_abl_${v}_${tag}.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/match_text_cfg5_${tag} -f python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cfg5_${tag}.log 2>&1
