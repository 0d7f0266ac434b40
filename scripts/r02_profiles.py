"""Round-2 evidence from gpurun_out/ into profiles/ (committed).

usage: python scripts/r02_profiles.py <bench-tag> [cfgN=<report.ncu-rep> ...]
  reads  gpurun_out/{bench_*,oracle_timings,launches,abl_ncu_*,ab}_<tag>*
  writes profiles/r02_bench_lines.jsonl    every bench line of the evidence run (default, per config,
                                           FASTA, list-only, pack + fused, the reference arm)
         profiles/r02_oracle_timings.json  the oracle per config on the box's host cores
         profiles/r02_launches.csv         ncu gpu__time_duration.sum launch list of `python bench.py`
         profiles/r02_ablations.md         the paper's layout questions: A/B times + ncu counters
         profiles/r02_ncu_summary.md       (with cfgN=report args) via scripts/ncu_config_summary.py
"""
import csv
import glob
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def last_json(path):
    try:
        lines = [ln for ln in open(path).read().splitlines() if ln.startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except (OSError, ValueError):
        return None


def ncu_csv(path):
    """metric -> value of the single profiled kernel in an `ncu --csv --metrics` log."""
    txt = open(path).read()
    rows = [r for r in csv.reader(io.StringIO("\n".join(ln for ln in txt.splitlines() if ln.startswith('"'))))]
    if not rows:
        return {}
    hdr = rows[0]
    mi, ui, vi, ki = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value"), hdr.index("Kernel Name")
    d = {"kernel": rows[1][ki] if len(rows) > 1 else ""}
    for r in rows[1:]:
        d[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    return d


def main():
    tag = sys.argv[1]
    lines = []
    for f in sorted(glob.glob(os.path.join(OUT, f"bench_*_{tag}.json"))):
        d = last_json(f)
        if d:
            d["_file"] = os.path.basename(f)
            lines.append(d)
    with open(os.path.join(PROF, "r02_bench_lines.jsonl"), "w") as fo:
        for d in lines:
            fo.write(json.dumps(d) + "\n")
    print(f"{len(lines)} bench lines")
    src = os.path.join(OUT, f"oracle_timings_{tag}.json")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(PROF, "r02_oracle_timings.json"))
    src = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(src):
        with open(src) as fi, open(os.path.join(PROF, "r02_launches.csv"), "w") as fo:
            fo.writelines(ln for ln in fi if ln.startswith('"'))
    # ablations: A/B times (ab_<tag>.jsonl) + counters (abl_ncu_<variant>_cfg<c>_<tag>.csv)
    ab = {}
    p = os.path.join(OUT, f"ab_{tag}.jsonl")
    if os.path.exists(p):
        for ln in open(p):
            d = json.loads(ln)
            ab.setdefault((d["variant"], d["config"]["workload"][:4]), []).append(d["ms_per_step"])
    md = ["# The paper's layout questions re-asked on B200 (round 2, final tree)", "",
          "Same box, same bench (`python bench.py --config C`, the text kernel), one library per variant "
          "(`scripts/build_ablations.py`; `r01` = the round-1 tree). Times: ms per step, each of two runs "
          f"of 20 steps (`gpurun_out/ab_{tag}.jsonl`). Counters: one `ncu --metrics` launch per config "
          f"(`gpurun_out/abl_ncu_*_{tag}.csv`).", "",
          "* `merged_f` — the paper's merged array (PAPER.md:206-207, :327): F(s) stored in cell 4 of an "
          "8-cell row next to the transitions, instead of the two arrays T and F.",
          "* `tab_cg` — the paper's `-Xptxas -dlcm=cg` L1 bypass (PAPER.md:227-228, :381-382): table loads "
          "`ld.global.cg` (L2 only) instead of `ld.global.nc`.", "",
          "| config | variant | ms/step | DRAM read GB | DRAM write GB | L1 hit % (global loads) | L2 hit % | warp instr (M) | issue active % |",
          "|---|---|---|---|---|---|---|---|---|"]
    for c in ("cfg2", "cfg3", "cfg4", "cfg5"):
        for v in ("base", "merged_f", "tab_cg", "r01"):
            ms = ab.get((v, c), [])
            f = os.path.join(OUT, f"abl_ncu_{v}_{c}_{tag}.csv")
            n = ncu_csv(f) if os.path.exists(f) else {}

            def g(k, s=1.0):
                return f"{n[k][0] / s:.3f}" if k in n else "—"
            l1 = ("—" if "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum" not in n else
                  f"{100 * n['l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum'][0] / max(1, n['l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum'][0]):.1f}")
            md.append(f"| {c} | {v} | {' / '.join(f'{x:.4f}' for x in ms) or '—'} | {g('dram__bytes_read.sum', 1e9)} | "
                      f"{g('dram__bytes_write.sum', 1e9)} | {l1} | {g('lts__t_sector_hit_rate.pct')} | "
                      f"{g('smsp__inst_executed.sum', 1e6)} | {g('smsp__issue_active.avg.pct_of_peak_sustained_active')} |")
    with open(os.path.join(PROF, "r02_ablations.md"), "w") as fo:
        fo.write("\n".join(md) + "\n")
    specs = [a for a in sys.argv[2:] if "=" in a]
    if specs:
        subprocess.check_call([sys.executable, os.path.join(ROOT, "scripts", "ncu_config_summary.py"),
                               os.path.join(PROF, "r02_ncu_summary.md"), *specs])


if __name__ == "__main__":
    main()
