"""Summarise scripts/ablations.sh output into profiles/r01_ablations.md (usage: ablation_summary.py <tag>)."""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
WHAT = {
    "base": "product build: 4^10-bit filter in smem, J2 in an L2-persisting window, T-row window in smem, TMA-staged text",
    "text_direct": "text read straight from global memory (L1/L2) instead of TMA-staged smem slices",
    "window0": "no T rows in shared memory: every row through L2 (ld.global.nc)",
    "jtable": "uint16 images: single-level 4^8 jump table in smem instead of filter + J2 (cfg3/cfg4 unaffected)",
    "nopersist": "no L2 access-policy window over J2",
}
KEYS = [("gpu__time_duration.sum", "ncu us"), ("dram__bytes_read.sum", "DRAM rd"),
        ("dram__bytes_write.sum", "DRAM wr"), ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("l1tex__t_sector_hit_rate.pct", "L1 hit %"), ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
        ("smsp__inst_executed.sum", "warp instr")]


def ncu(path):
    if not os.path.exists(path):
        return {}
    rows = list(csv.reader(io.StringIO(open(path).read())))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"]
    if not hdr:
        return {}
    rows = [r for r in rows[hdr[0]:] if len(r) == len(rows[hdr[0]])]
    h = rows[0]
    im, iv, iu = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    return {r[im]: f"{r[iv]} {r[iu]}".strip() for r in rows[1:]}


def main(tag):
    res = {}
    for line in open(os.path.join(OUT, f"ablations_{tag}.jsonl")):
        d = json.loads(line)
        c = d["config"]["workload"][:4]
        k = [v for kk, v in d["kernels_ms"].items() if kk.startswith("match")][0]
        res.setdefault(d["variant"], {})[c] = (k, d["roofline"]["frac"])
    cfgs = ["cfg2", "cfg3", "cfg4", "cfg5"]
    L = [f"# Layout / cache ablations on B200 (tag {tag}) — SURVEY.md §8(f) NEXT 4", "",
         "The paper's experiments X1-X3 (PAPER.md:278-433: merged vs two arrays, texture vs global table, "
         "text in shared memory, L1 size) re-asked for this kernel: each row is the product library with one "
         "`PFAC_*` build knob flipped (`scripts/build_ablations.py`), benched by `scripts/ablations.sh` "
         "(fused match+compact kernel, CUDA events, 10 steps after 3 warm-ups). Cells: match+compact ms "
         "(fraction of measured HBM at 4.25 B/base).", "",
         "| variant | what changes | " + " | ".join(cfgs) + " |", "|---|---|" + "---|" * len(cfgs)]
    for v in ["base"] + sorted(x for x in res if x != "base"):
        if v not in res:
            continue
        cells = []
        for c in cfgs:
            if c in res[v]:
                ms, fr = res[v][c]
                rel = f" ×{ms / res['base'][c][0]:.2f}" if v != "base" and c in res.get("base", {}) else ""
                cells.append(f"{ms:.3f} ({fr:.2f}){rel}")
            else:
                cells.append("—")
        L.append(f"| {v} | {WHAT.get(v, '')} | " + " | ".join(cells) + " |")
    L.append("")
    for c in ["cfg2", "cfg5"]:
        L.append(f"### ncu counters of the match kernel, {c} (one launch, `ncu --metrics`, clocks not locked)")
        L.append("")
        L.append("| variant | " + " | ".join(n for _, n in KEYS) + " |")
        L.append("|---|" + "---|" * len(KEYS))
        for v in ["base"] + sorted(x for x in res if x != "base"):
            m = ncu(os.path.join(OUT, f"abl_ncu_{v}_{c}_{tag}.csv"))
            if m:
                L.append(f"| {v} | " + " | ".join(m.get(k, "—") for k, _ in KEYS) + " |")
        L.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r01_ablations.md"), "w") as f:
        f.write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main(*sys.argv[1:])
