# Round-2 evidence on the final tree: oracle timings, the default bench line, per-config lines,
# FASTA and list-only lines, the reference arm, the ncu launch list of the default command, ncu --set
# full of the text kernel on cfg2..cfg5, and ncu counters of the two paper-layout ablation builds.
tag=${1:-r02z}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/smi_${tag}.txt
lscpu > gpurun_out/lscpu_${tag}.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 900 python scripts/oracle_timings.py --seconds 12 > gpurun_out/oracle_timings_${tag}.json 2> gpurun_out/oracle_timings_${tag}.err; tail -5 gpurun_out/oracle_timings_${tag}.err
timeout 900 python bench.py > gpurun_out/bench_default_${tag}.json 2> gpurun_out/bench_default_${tag}.err
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg${c}_${tag}.json 2> gpurun_out/bench_cfg${c}_${tag}.err
done
timeout 600 python bench.py --config 2 --barriers 80 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_fasta_${tag}.json 2>/dev/null
for c in 2 5; do
  timeout 600 python bench.py --config $c --path text-list --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg${c}_list_${tag}.json 2>/dev/null
  timeout 600 python bench.py --config $c --path fused --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg${c}_fused_${tag}.json 2>/dev/null
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_${tag}.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${tag}.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for c in ${NCU_CFGS-2 3}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 4 -c 1 \
    -o gpurun_out/match_text_cfg${c}_${tag} -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
for v in base merged_f tab_cg; do
  lib=""; [ "$v" != base ] && lib=paper_1811_10498_b200/_lib/alt/libpfac_$v.so
  for c in 2 3 4 5; do
    PFAC_LIB=$lib timeout 600 ncu --metrics $M --clock-control none -k regex:match_kernel -s 4 -c 1 --csv \
      python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abl_ncu_${v}_cfg${c}_${tag}.csv 2>/dev/null
  done
done
bash scripts/ab_libs.sh ${tag} 2 "2 3 4 5" base merged_f tab_cg r01
ls gpurun_out | grep ${tag} | wc -l
