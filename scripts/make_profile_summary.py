"""Turn one round's gpurun_out/ captures into committed evidence under profiles/.

usage: python scripts/make_profile_summary.py <tag> [<round>]
  reads  gpurun_out/launches_<tag>.csv, gpurun_out/{pack,match,compact}_kernel_<tag>.ncu-rep,
         gpurun_out/bench_<tag>.json
  writes profiles/<round>_launches.csv  (ncu gpu__time_duration.sum launch list)
         profiles/<round>_ncu_summary.md (per-kernel metrics, shares of the step, roofline)
         profiles/ncu_traffic.json       (dram bytes per launch, read by bench.py)
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
KERNELS = ["match_text", "pack_kernel", "match_fused", "match_kernel", "compact_kernel", "match_bar"]
ALG = {"match_text": 5.0, "pack_kernel": 1.25, "match_fused": 4.25, "match_kernel": 4.25, "compact_kernel": 4.0, "match_bar": 4.375}
TITLES = {"match_text": "match_kernel<TXT=1> (pack + match + compact from ASCII, bench default)",
          "pack_kernel": "pack_kernel (--path fused)", "match_fused": "match_kernel<FUSE=1> (match + compact, --path fused)",
          "match_kernel": "match_kernel<FUSE=0> (--path separate)", "compact_kernel": "compact_kernel (--path separate)",
          "match_bar": "match_kernel<FUSE=1, BAR=1> (--barriers 80: FASTA newlines + N gaps)"}
TRAFFIC_KEY = {"match_text": "match_text", "pack_kernel": "pack", "match_fused": "match_fused", "match_kernel": "match",
               "compact_kernel": "compact", "match_bar": "match_bar"}
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp instr"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / scheduler"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3,
              "nsecond": 1e-9, "second": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def val(d, u, k):
    try:
        return float(d[k]) * UNIT_SCALE.get(u.get(k, ""), 1)
    except (KeyError, ValueError):
        return None


def main(tag, rnd="r01"):
    os.makedirs(PROF, exist_ok=True)
    bench = None
    bp = os.path.join(OUT, f"bench_{tag}.json")
    if os.path.exists(bp):
        for line in open(bp):
            if line.startswith("{"):
                bench = json.loads(line)
    n = bench["config"]["n_bases_per_rank"] if bench else 256_000_000
    lines = [f"# ncu summary — {rnd} (tag {tag}), cfg2 (256 Mbp, 1000 x 20-mers), 1x B200", ""]
    if bench and "image" in bench.get("config", {}):
        lines.append(f"Device image: {bench['config']['image']}")
        lines.append("")
    lines.append("Captured with `ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 3 -c 1` "
                 "around `python bench.py --steps 1 --warmup 3` (scripts/ncu_all.sh). Per-launch times under ncu are "
                 "cold-cache and serialised; compare shares, not absolutes.")
    lines.append("")
    traffic = {}
    for k in KERNELS:
        rep = os.path.join(OUT, f"{k}_{tag}.ncu-rep")
        if not os.path.exists(rep):
            continue
        d, u = raw(rep)
        lines.append(f"## {TITLES[k]}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, name in METRICS:
            if key in d:
                lines.append(f"| {name} (`{key}`) | {d[key]} {u.get(key, '')} |")
        rd, wr = val(d, u, "dram__bytes_read.sum"), val(d, u, "dram__bytes_write.sum")
        dur = val(d, u, "gpu__time_duration.sum")
        if rd is not None and wr is not None:
            alg = ALG[k] * n
            lines.append(f"| DRAM read+write per launch | {(rd + wr) / 1e6:.1f} MB (algorithmic {alg / 1e6:.1f} MB, "
                         f"ratio {(rd + wr) / alg:.3f}) |")
            traffic[TRAFFIC_KEY[k]] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                                                 "algorithmic_bytes": alg, "ncu_duration_s": dur, "n": n}
        st = {kk: float(vv) for kk, vv in d.items() if kk.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not kk.endswith("_not_issued") and vv not in ("", "n/a")}
        tot = sum(st.values()) or 1
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        lines.append("| top stall reasons | " + ", ".join(
            f"{kk.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%" for kk, v in top) + " |")
        lines.append("")
    # launch list: shares of the step
    lp = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(PROF, f"{rnd}_launches.csv"))
        rows = [r for r in csv.reader(open(lp)) if len(r) > 10 and r[0] != "ID"]
        tot = {}
        names = {"pack_kernel": "pack_kernel", "match_kernel": "match_kernel", "compact_kernel": "compact_kernel"}
        for r in rows:
            name = r[4]
            short = next((v for k, v in names.items() if k in name), "other: " + name[:40])
            tot.setdefault(short, []).append(float(r[-1]))
        lines.append("## Launch list (ncu `gpu__time_duration.sum`, all launches of a 2-step bench run)")
        lines.append("")
        lines.append("| kernel | launches | mean ns | share of our kernels' time |")
        lines.append("|---|---|---|---|")
        ours = sum(sum(v) for k2, v in tot.items() if not k2.startswith("other"))
        for k2, v in sorted(tot.items()):
            share = f"{100 * sum(v) / ours:.1f}%" if not k2.startswith("other") else "-"
            lines.append(f"| {k2} | {len(v)} | {sum(v) / len(v):.0f} | {share} |")
        lines.append("")
    if bench:
        kt = {k2: v for k2, v in bench["kernels_ms"].items() if isinstance(v, float) and not k2.endswith("frac")}
        tot_ms = sum(kt.values())
        lines.append("## Live bench (CUDA events, same build)")
        lines.append("")
        lines.append(f"- path {bench.get('path')}: step {bench['ms_per_step']:.4f} ms → {bench['value']:.1f} Gbases/s; "
                     f"clocks {bench['clocks']}")
        for k2, v in kt.items():
            lines.append(f"- {k2}: {v:.4f} ms ({100 * v / tot_ms:.1f}% of kernel time)")
        r = bench["roofline"]
        lines.append(f"- match roofline: {r['achieved']:.0f} GB/s of {r['peak']} GB/s measured = {r['frac']:.3f}")
        lines.append("")
    with open(os.path.join(PROF, f"{rnd}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(PROF, "ncu_traffic.json")
    allt = json.load(open(tp)) if os.path.exists(tp) else {}
    allt["cfg2"] = traffic
    allt["cfg2"]["source"] = f"profiles/{rnd}_ncu_summary.md (tag {tag})"
    json.dump(allt, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
