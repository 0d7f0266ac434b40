"""Summarise per-config `ncu --set full` captures of the bench step's dominant kernel into profiles/.

usage: python scripts/ncu_config_summary.py <out.md> <cfg>=<report.ncu-rep> [...]

For each report: duration, DRAM bytes (vs the algorithmic bytes of the text kernel: 1 B ASCII read +
4 B out[] written per base + 12 B per listed match), L2 sectors read by the SM (per base), warp
instructions (per base), issue activity, SIMT efficiency, shared-memory bank conflicts and the
warp-stall breakdown.  Also updates profiles/ncu_traffic.json (dram bytes per launch, read by
bench.py for roofline.traffic) and profiles/ncu_bounds.json (the per-base L2-sector and instruction
counts bench.py turns into the cfg4 L2-gather and cfg5 issue bounds).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PROF = os.path.join(ROOT, "profiles")

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
        ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 sectors read (SM)"),
        ("lts__t_sector_hit_rate.pct", "L2 hit rate %"), ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
        ("smsp__inst_executed.sum", "warp instructions"), ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / warp instr"),
        ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / scheduler"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
        ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"), ("launch__registers_per_thread", "registers / thread"),
        ("sm__cycles_elapsed.avg.per_second", "SM clock (Hz)")]
SCALE = {"dram__bytes_read.sum": 1e9, "dram__bytes_write.sum": 1e9}  # ncu raw csv reports GB for these


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return dict(zip(hdr, rows[2])), dict(zip(hdr, units))


def num(d, k):
    try:
        return float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")


def to_base(v, unit):
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                "msecond": 1e-3, "second": 1}.get(unit, 1)


def main():
    out_md = sys.argv[1]
    import pfac_datagen as gen
    traffic_p = os.path.join(PROF, "ncu_traffic.json")
    bounds_p = os.path.join(PROF, "ncu_bounds.json")
    traffic = json.load(open(traffic_p)) if os.path.exists(traffic_p) else {}
    bounds = json.load(open(bounds_p)) if os.path.exists(bounds_p) else {}
    lines = [f"# ncu --set full of the bench step's dominant kernel ({os.path.basename(out_md)})", ""]
    for spec in sys.argv[2:]:
        cfg, rep = spec.split("=", 1)
        ci = int(cfg.replace("cfg", ""))
        d, u = raw(rep)
        n = gen.CONFIGS[ci].n
        name = d.get("Kernel Name", "")
        dur = to_base(num(d, "gpu__time_duration.sum"), u.get("gpu__time_duration.sum"))
        rd = to_base(num(d, "dram__bytes_read.sum"), u.get("dram__bytes_read.sum"))
        wr = to_base(num(d, "dram__bytes_write.sum"), u.get("dram__bytes_write.sum"))
        bench = os.path.join(os.path.dirname(rep), f"bench_{cfg}_{os.path.basename(rep).rsplit('_', 1)[-1].split('.')[0]}.json")
        matches = None
        if os.path.exists(bench):
            try:
                matches = json.load(open(bench))["config"]["matches_per_step"]
            except Exception:  # noqa: BLE001
                matches = None
        alg = 5.0 * n + 12.0 * (matches or 0)
        sectors = num(d, "lts__t_sectors_srcunit_tex_op_read.sum")
        inst = num(d, "smsp__inst_executed.sum")
        lines += [f"## {cfg}: `{name[:110]}`", "", f"report: `{os.path.basename(rep)}`, n = {n:,} bases"
                  + (f", {matches:,} matches" if matches is not None else ""), "",
                  "| metric | value |", "|---|---|"]
        for k, label in KEYS:
            if k in d:
                lines.append(f"| {label} (`{k}`) | {d[k]} {u.get(k, '')} |")
        lines += [f"| DRAM bytes / algorithmic bytes | {(rd + wr) / alg:.3f} ({(rd + wr) / 1e9:.3f} GB vs {alg / 1e9:.3f} GB: "
                  f"5 B/base + 12 B/match) |",
                  f"| L2 sectors read per base | {sectors / n:.4f} |",
                  f"| warp instructions per base | {inst / n:.4f} |", ""]
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(d, k) for k in d
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
        st = {k: v for k, v in st.items() if v == v and v > 0}
        tot = sum(st.values()) or 1
        lines += ["stall samples: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in
                                                sorted(st.items(), key=lambda x: -x[1])[:9]), ""]
        traffic.setdefault(cfg, {})["match_text"] = {
            "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "algorithmic_bytes": alg,
            "ncu_duration_s": dur, "n": n, "report": os.path.basename(rep)}
        bounds[cfg] = {"l2_sectors_read_per_base": sectors / n, "warp_inst_per_base": inst / n,
                       "threads_per_warp_inst": num(d, "smsp__thread_inst_executed_per_inst_executed.ratio"),
                       "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                       "ncu_duration_s": dur, "report": os.path.basename(rep)}
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_p, "w") as f:
        json.dump(traffic, f, indent=1)
    with open(bounds_p, "w") as f:
        json.dump(bounds, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
