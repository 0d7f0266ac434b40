"""Summarise an .ncu-rep: key SOL / memory / stall metrics (run here, no GPU needed)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__warps_eligible.avg.per_cycle_active", "lts__t_sector_hit_rate.pct"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def main(rep):
    recs, units = raw(rep)
    for d in recs:
        print("kernel:", d.get("Kernel Name", "")[:80])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>16s} {units.get(k, '')}")
        st = {k: float(v) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("_not_issued") and v not in ("", "n/a")}
        tot = sum(st.values()) or 1
        print("  stall samples (top):")
        for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]:
            print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {v:10.0f} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    for r in sys.argv[1:]:
        main(r)
