"""Workload for tests/test_gpu_sanitizer.py: every kernel instantiation of libpfac once on small
inputs, checked against the oracle, so that compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) sees each of them: pack (plain and barrier map), the match kernel (unfused, BAR, FUSE,
LIST, TXT with 2048- and 1024-position slices, list-only TXT), the standalone compaction, the
all-occurrence expansion and pfac_scan_host.  Run as a script (not collected by pytest)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pfac_datagen as gen  # noqa: E402
import paper_1811_10498_b200 as P  # noqa: E402
from oracle import Oracle  # noqa: E402

DEV = torch.device("cuda:0")


def check(cond, what):
    if not cond:
        raise SystemExit(f"sanitize_workload: mismatch in {what}")


def run(pats, text, tag):
    n = len(text)
    o = Oracle(pats)
    exp = o.match(text)
    epos, epid = o.match_list(text)
    a = P.Automaton(pats)
    d = torch.from_numpy(text).to(DEV)
    bars = not np.isin(text, np.frombuffer(b"ACGTacgt", np.uint8)).all()
    # pack (+ barrier map), unfused match, standalone compaction
    bad = torch.zeros(1, dtype=torch.int64, device=DEV)
    if bars:
        packed, inv = P.pack_barriers_async(d, first_bad=bad)
        out = P.match_barriers_async(a, packed, inv, n, n)
    else:
        packed = P.pack_async(d, first_bad=bad)
        inv = None
        out = P.match_packed_async(a, packed, n, n)
    torch.cuda.synchronize()
    check((out.cpu().numpy() == exp).all(), f"{tag} match")
    pos, pid, m = P.compact(out, k=len(pats))
    check(m == len(epos) and (pos.cpu().numpy() == epos).all(), f"{tag} compact")
    cap = len(epos) + 16
    pos = torch.empty(cap, dtype=torch.int64, device=DEV)
    pid = torch.empty(cap, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    # fused match + compact (FUSE, BAR when barriers), list only (LIST)
    out2 = torch.empty(n, dtype=torch.int32, device=DEV)
    ws = torch.empty(P.compact_workspace_bytes(n), dtype=torch.uint8, device=DEV)
    P.match_compact_async(a, packed, n, n, out2, pos, pid, cnt, ws, inv=inv)
    torch.cuda.synchronize()
    check(int(cnt.item()) == len(epos) and (out2.cpu().numpy() == exp).all(), f"{tag} fused")
    wsl = torch.empty(P.match_list_workspace_bytes(n), dtype=torch.uint8, device=DEV)
    P.match_list_async(a, packed, n, n, pos, pid, cnt, wsl, inv=inv)
    torch.cuda.synchronize()
    check(int(cnt.item()) == len(epos) and (pos[:len(epos)].cpu().numpy() == epos).all(), f"{tag} list")
    # every text-call path: two kernels, TXT 2048, TXT 1024; dense and list only
    for mode in (0, 1, 2):
        a.set_text_kernel(mode)
        for dense in (True, False):
            wst = torch.empty(P.match_text_workspace_bytes(n, n, not dense), dtype=torch.uint8, device=DEV)
            o3 = torch.empty(n, dtype=torch.int32, device=DEV) if dense else None
            P.match_text_async(a, d, n, n, o3, pos, pid, cnt, wst)
            torch.cuda.synchronize()
            check(int(cnt.item()) == len(epos) and (pos[:len(epos)].cpu().numpy() == epos).all(),
                  f"{tag} text mode {mode} dense {dense}")
            if dense:
                check((o3.cpu().numpy() == exp).all(), f"{tag} text out mode {mode}")
    a.set_text_kernel(-1)
    # all occurrences
    pa, pi, t = P.expand(a, pos[:len(epos)], pid[:len(epos)])
    ap_, ai = o.match_all(text)
    check(t == len(ap_) and (pa.cpu().numpy() == ap_).all() and (pi.cpu().numpy() == ai).all(), f"{tag} expand")
    # host-memory end to end
    hp, hi, hm = P.scan_host(a, torch.from_numpy(text))
    check(hm == len(epos) and (hp.numpy() == epos).all(), f"{tag} scan_host")


def run_log(pats, text, tag):
    """The fused and text kernels on a text long enough (and dense enough: every position whose
    first base is in a set matches) that each warp's staging overflows and its slices go through the
    per-warp match log and, when that is full, the out[] re-read (match.cu, FUSE emission)."""
    n = len(text)
    epos, epid = Oracle(pats).match_list(text)
    a = P.Automaton(pats)
    d = torch.from_numpy(text).to(DEV)
    cap = len(epos) + 16
    pos = torch.empty(cap, dtype=torch.int64, device=DEV)
    pid = torch.empty(cap, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    for mode in (0, 1):
        a.set_text_kernel(mode)
        for dense in (True, False):
            wst = torch.empty(P.match_text_workspace_bytes(n, n, not dense), dtype=torch.uint8, device=DEV)
            o3 = torch.empty(n, dtype=torch.int32, device=DEV) if dense else None
            P.match_text_async(a, d, n, n, o3, pos, pid, cnt, wst)
            torch.cuda.synchronize()
            check(int(cnt.item()) == len(epos) and (pos[:len(epos)].cpu().numpy() == epos).all()
                  and (pid[:len(epos)].cpu().numpy() == epid).all(), f"{tag} text mode {mode} dense {dense}")


def main():
    if os.environ.get("PFAC_SANITIZE_LOG"):
        n = int(os.environ.get("PFAC_SANITIZE_LOG_N", "24000000"))
        for k, first in ((4, "A"), (4, "AC"), (9, "A")):
            pats = [p for p in gen.all_kmers(k) if chr(p[0]) in first]
            run_log(pats, gen.iid_text(300 + k, 0, n), f"log k={k} first={first}")
        print("sanitize_workload ok")
        return
    n = int(os.environ.get("PFAC_SANITIZE_N", "70001"))
    cfg1 = gen.config_patterns(gen.CONFIGS[1])
    big = gen.random_patterns(41, 40_000, 12, 40)  # uint32 image, J2 + chain-head rows
    nested = [b"A" * L for L in range(1, 30)]
    t1 = gen.plant(gen.iid_text(41, 0, n), 0, n, cfg1, 41)
    t2 = gen.plant(gen.iid_text(42, 0, n), 0, n, big, 42)
    t3 = np.frombuffer(b"A" * n, np.uint8).copy()
    t3[::997] = ord("C")
    t4 = gen.add_barriers(t1.copy(), 43, line=60)
    for pats, text, tag in [(cfg1, t1, "cfg1"), (big, t2, "big32"), (nested, t3, "nested"), (cfg1, t4, "fasta"),
                            (cfg1, t1[:4099], "short")]:
        run(pats, text, tag)
    print("sanitize_workload ok")


if __name__ == "__main__":
    main()
