# Round-2 final evidence, part 3 (the final tree): FASTA and list-only lines, the reference arm, and
# ncu --set full of the cfg2 / cfg3 text kernels.
tag=${1:-r02j}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke rc $?
timeout 600 python bench.py --config 2 --barriers 80 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' > gpurun_out/bench_cfg2_fasta_${tag}.json
timeout 600 python bench.py --config 2 --path text-list --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' > gpurun_out/bench_cfg2_list_${tag}.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | grep '^{' > gpurun_out/bench_reference_${tag}.json
for f in fasta list; do python -c "import json;d=json.load(open('gpurun_out/bench_cfg2_${f}_${tag}.json'));print('$f', round(d['ms_per_step'],4), round(d['value'],1))"; done
bash scripts/r02_ncu_full.sh ${tag} "2 3"
