# B200 versions of the paper's layout/cache experiments: bench every
# ablation library (scripts/build_ablations.py) on cfg2..cfg5 (fused path) and capture a few ncu
# counters of the match kernel on cfg2 and cfg5.  Output: gpurun_out/ablations_<tag>.jsonl,
# gpurun_out/abl_ncu_<variant>_cfg<c>_<tag>.csv
tag=${1:-x}
mkdir -p gpurun_out
out=gpurun_out/ablations_$tag.jsonl
: > $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum
for lib in "" $(ls paper_1811_10498_b200/_lib/alt/libpfac_*.so); do
  name=$(basename "${lib:-libpfac_base.so}" .so); name=${name#libpfac_}
  for c in 2 3 4 5; do
    PFAC_LIB=$lib timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
      | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['variant']='$name'; print(json.dumps(d))" >> $out
  done
  for c in 2 5; do
    PFAC_LIB=$lib timeout 600 ncu --metrics $M --clock-control none -k regex:match_kernel -s 4 -c 1 --csv \
      python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abl_ncu_${name}_cfg${c}_$tag.csv 2>/dev/null
  done
done
python scripts/ablation_summary.py $tag
