#!/usr/bin/env python
"""PFAC hot-path benchmark (driver contract: one JSON line on rank 0).

A step = one pass of the whole hot path over one batch of synthetic input
resident in HBM: pack (ASCII -> 2-bit) -> match (PFAC walk from every position) -> compact (match
list + count) [-> NCCL gather of counts and lists when N > 1].  Build (row 1) and the device image
upload (row 2) happen once, before timing, and are reported as `build_ms` / `prepare_ms`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--scaling weak|strong]
  python bench.py --impl reference ...   # the oracle (CPU) on the same workload, bounded sample

Default workload: N = 1: BASELINE.json configs[1] (cfg2: 256 Mbp, 1000 patterns of length 20), the
config the metric is quoted on.  N > 1: configs[2] (cfg3: the 3.1 Gbp text, 10000 patterns of length
16-64) split across the N ranks -- strong scaling, the north star's "near-linear 8-GPU scaling on
the 3.1 Gbp config"; `--scaling weak` gives each rank a config-sized shard of a longer text instead.
One process per GPU: under torchrun (WORLD_SIZE set) the ranks are torchrun's; `--gpus N` without
WORLD_SIZE re-launches this script under torch.distributed.run with N ranks (127.0.0.1 rendezvous).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gbases/s per B200 and whole-box at 1/2/4/8 GPUs; % of HBM roofline"
MATCH_BYTES_PER_BASE = 4.25   # 0.25 B packed text read + 4 B int32 out[] written
PACK_BYTES_PER_BASE = 1.25    # 1 B ASCII read + 0.25 B packed written
COMPACT_BYTES_PER_BASE = 4.0  # 4 B out[] read (+12 B per match written)
BARRIER_BYTES_PER_BASE = 0.125  # --barriers: 2 B mask per 16 bases, written by pack, read by match
FALLBACK_HBM_GBS = 6650.0     # /opt/skills/guides/B200_PROFILING.md fallback


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def profiled_traffic(cfg_idx: int, path: str):
    """dram bytes per match launch from the committed ncu --set full capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    key = {"fused": "match_fused", "separate": "match", "list": "match_list", "text": "match_text",
           "text-list": "match_text_list"}[path]
    e = d.get(f"cfg{cfg_idx}", {}).get(key)
    return None if e is None else float(e["dram_bytes_per_launch"])


def secondary_bounds(cfg_idx: int, n: int, kernel_ms: float):
    """The text kernel's other ceilings (cfg4 min(HBM, L2 random gather), cfg5 issue),
    from the per-base counts of the committed ncu capture (profiles/ncu_bounds.json) and the measured
    L2 gather rate (profiles/r01_microbench.json): each floor is the time that resource alone needs at
    its peak; frac = floor / the measured kernel time."""
    pb = os.path.join(ROOT, "profiles", "ncu_bounds.json")
    pm = os.path.join(ROOT, "profiles", "r01_microbench.json")
    if not (os.path.exists(pb) and os.path.exists(pm)):
        return None
    b = json.load(open(pb)).get(f"cfg{cfg_idx}")
    if not b:
        return None
    mb = json.load(open(pm))
    gather = max(x["gsectors_per_s"] for x in mb["l2_gather_32B"]) * 1e9
    attrs = mb["device_attrs"]
    issue = attrs["sms"] * 4 * attrs["sm_clock_khz"] * 1e3  # warp instructions / s (4 schedulers per SM)
    l2_ms = b["l2_sectors_read_per_base"] * n / gather * 1e3
    is_ms = b["warp_inst_per_base"] * n / issue * 1e3
    return {
        "l2_gather": {"sectors_per_base": b["l2_sectors_read_per_base"], "peak_gsectors_s": gather / 1e9,
                      "floor_ms": l2_ms, "frac": l2_ms / kernel_ms},
        "issue": {"warp_inst_per_base": b["warp_inst_per_base"], "peak_ginst_s": issue / 1e9,
                  "floor_ms": is_ms, "frac": is_ms / kernel_ms,
                  "simt_threads_per_inst": b.get("threads_per_warp_inst")},
        "source": f"profiles/ncu_bounds.json ({b.get('report')}), profiles/r01_microbench.json",
    }


class ClockSampler:
    """nvml SM clock + throttle reasons sampled in a thread during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001 - clocks are reported as unavailable
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(s)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(args, world, rank):
    import pfac_datagen as gen
    from paper_1811_10498_b200.parallel import shard

    cfg = gen.CONFIGS[args.config]
    n_total = cfg.n * world if args.scaling == "weak" else cfg.n
    if args.n:
        n_total = args.n * (world if args.scaling == "weak" else 1)
    pats = gen.config_patterns(cfg)
    maxlen = max(len(p) for p in pats)
    sh = shard(n_total, world, rank, maxlen)
    if cfg.repetitive:
        text = gen.config_text(cfg, 0, sh.avail_end, patterns=pats, n=n_total)[sh.start:]
    else:
        text = gen.config_text(cfg, sh.start, sh.avail_end, patterns=pats, n=n_total)
    if args.barriers is not None:  # FASTA-like text: newlines + assembly gaps (reading R5)
        gen.add_barriers(text, cfg.seed, line=args.barriers, a=sh.start, **BARRIER_GAPS)
    return cfg, pats, sh, n_total, text


def verify_gathered(args, gathered, cap, world, n_total, pats, window=200_000):
    """Rank 0, after the warm-up (outside the timed region): the lists gathered from every rank
    (parallel.unpack_lists) are in ascending global position, and for every rank the entries in the
    first `window` owned positions equal the oracle's list of that window (text regenerated
    position-addressably; cfg5's segment text is only regenerated for rank 0).  Returns a summary
    dict; raises AssertionError on a mismatch (the bench then prints no line)."""
    import numpy as np

    import pfac_datagen as gen
    from oracle import Oracle
    from paper_1811_10498_b200.parallel import shard, unpack_lists
    gp, gi, counts = unpack_lists(gathered, cap)
    gp, gi = gp.numpy(), gi.numpy()
    assert (np.diff(gp) > 0).all(), "gathered positions are not strictly ascending"
    cfg = gen.CONFIGS[args.config]
    maxlen = max(len(p) for p in pats)
    o = Oracle(pats)
    checked = 0
    for r in range(world):
        if cfg.repetitive and r > 0:
            break
        sh = shard(n_total, world, r, maxlen)
        w = min(window, sh.n_own)
        hi = min(n_total, sh.start + w + maxlen - 1)
        if cfg.repetitive:
            t = gen.config_text(cfg, 0, hi, patterns=pats, n=n_total)[sh.start:]
        else:
            t = gen.config_text(cfg, sh.start, hi, patterns=pats, n=n_total)
        if args.barriers is not None:
            gen.add_barriers(t, cfg.seed, line=args.barriers, a=sh.start, **BARRIER_GAPS)
        ep, ei = o.match_list(t, 0, w, n=len(t))
        sel = (gp >= sh.start) & (gp < sh.start + w)
        assert (gp[sel] == ep.astype(np.int64) + sh.start).all() and (gi[sel] == ei).all(), f"rank {r} list differs"
        checked += w
    return {"ranks": world, "counts": counts, "total": int(sum(counts)), "ascending": True,
            "oracle_checked_positions": checked}


# assembly gaps for --barriers: in 20% of 1 Mbase blocks a run of up to 100 kbases of N (~1% of bytes)
BARRIER_GAPS = {"block": 1 << 20, "run_max": 100_000, "run_frac": 0.2}


def workload_name(cfg, args) -> str:
    if args.barriers is None:
        return cfg.name
    return f"{cfg.name}; FASTA layout: newline every {args.barriers} bases + N gaps (barriers)"


def oracle_sample(pats, text, n_own, target_s):
    """Time the oracle (as it stands, 1 core) on a prefix of this rank's text sized to ~target_s."""
    from oracle import Oracle
    o = Oracle(pats)
    probe = min(n_own, 2_000_000)
    t0 = time.perf_counter()
    o.match_list(text, 0, probe, n=len(text))
    rate = probe / max(time.perf_counter() - t0, 1e-6)
    m = int(min(n_own, max(probe, rate * target_s)))
    t0 = time.perf_counter()
    pos, _ = o.match_list(text, 0, m, n=len(text))
    dt = time.perf_counter() - t0
    return m, dt, len(pos)


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def oracle_threads(o, text, m, n, p):
    """The oracle (as it stands) over [0, m) split into p disjoint position ranges, one thread each
    (the C oracle runs outside the GIL: ctypes releases it).  Returns (seconds, matches)."""
    from concurrent.futures import ThreadPoolExecutor
    cuts = [m * i // p for i in range(p + 1)]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(p) as ex:
        res = list(ex.map(lambda i: len(o.match_list(text, cuts[i], cuts[i + 1], n=n)[0]), range(p)))
    return time.perf_counter() - t0, sum(res)


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import pfac_datagen as gen
    from oracle import Oracle
    cfg = gen.CONFIGS[args.config]
    n_total = args.n or cfg.n  # the reference arm runs on one host: the whole text is its workload
    pats = gen.config_patterns(cfg)
    maxlen = max(len(p) for p in pats)
    o = Oracle(pats)
    p = host_cores() if args.ref_cores == 0 else args.ref_cores

    def text_prefix(m):  # bases [0, m + maxlen - 1) of the workload's text (position-addressable)
        hi = min(n_total, m + maxlen - 1)
        t = gen.config_text(cfg, 0, hi, patterns=pats, n=n_total)
        if args.barriers is not None:
            gen.add_barriers(t, cfg.seed, line=args.barriers, **BARRIER_GAPS)
        return t

    # size one step's sample so that W + K steps take about args.ref_budget seconds in total
    probe = min(n_total, 2_000_000 * p)
    text = text_prefix(probe)
    dt, _ = oracle_threads(o, text, probe, len(text), p)
    rate = probe / max(dt, 1e-6)
    per_step = args.ref_budget / max(1, args.steps + args.warmup)
    m = int(min(n_total, max(100_000, rate * per_step)))
    if m > probe:
        text = text_prefix(m)
    for _ in range(args.warmup):
        oracle_threads(o, text, m, len(text), p)
    times = []
    for _ in range(args.steps):
        times.append(oracle_threads(o, text, m, len(text), p)[0])
    t = sum(times) / len(times)
    v = m / t / 1e9
    sample = (f"first {m} positions of the {cfg.name} text per step, split into {p} disjoint ranges on {p} "
              f"threads (walks read up to maxlen-1 further)")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "Gbases/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args), "n_bases_per_step": m, "patterns": len(pats)},
        "cpu_baseline": {"value": v, "unit": "Gbases/s", "cores": p, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "Gbases/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_pfac(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1811_10498_b200 as P
    from paper_1811_10498_b200.parallel import gather_lists_async, list_buffer, unpack_lists

    world, rank, local = dist_env()
    ndev = torch.cuda.device_count()
    if ndev == 0:
        raise SystemExit("bench.py: no CUDA device visible (the PFAC path has no CPU fallback)")
    if world > 1:
        if args.backend == "nccl" and world > ndev:
            raise SystemExit(f"bench.py: {world} NCCL ranks need {world} GPUs, {ndev} visible "
                             "(--backend gloo runs the ranks on shared GPUs, for tests only)")
        # --backend gloo + more ranks than GPUs exercises the N>1 control flow on one GPU (tests)
        local = local % ndev
        torch.cuda.set_device(local)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    t_gen = time.perf_counter()
    cfg, pats, sh, n_total, text = workload(args, world, rank)
    t_gen = time.perf_counter() - t_gen

    t0 = time.perf_counter()
    a = P.Automaton(pats)
    build_ms = (time.perf_counter() - t0) * 1e3
    text_plan = None
    if args.text_kernel is not None:
        a.set_text_kernel(args.text_kernel)
    elif hasattr(P.lib(), "pfac_plan_text"):  # (A/B runs may load an older library without it)
        # the library's text plan from a host sample of this rank's text (outside the timed region)
        stride = max(1, len(text) // 200_000)
        mode, deep = a.plan_text(text, stride=stride)
        text_plan = {"api": "pfac_plan_text", "sample_positions": -(-len(text) // stride),
                     "deep_walk_share": deep, "mode": mode}
    t0 = time.perf_counter()
    a.prepare(local)
    prepare_ms = (time.perf_counter() - t0) * 1e3

    n_own, n_avail = sh.n_own, sh.n_avail
    h_text = torch.from_numpy(text).pin_memory()
    d_text = h_text.to(dev)
    packed = torch.empty(P.packed_words(n_avail), dtype=torch.int32, device=dev)
    bars = args.barriers is not None  # barrier path: pack writes the barrier mask, BAR match kernel
    inv = torch.empty(P.inv_words(n_avail), dtype=torch.int16, device=dev) if bars else None
    out = torch.empty(n_own, dtype=torch.int32, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(P.compact_workspace_bytes(n_own), dtype=torch.uint8, device=dev)
    # size the list from a probe pass (the count is exact even when the capacity is exceeded)
    pos = torch.empty(1, dtype=torch.int64, device=dev)
    pid = torch.empty(1, dtype=torch.int32, device=dev)
    def pack(st=None):
        if bars:
            P.pack_barriers_async(d_text, packed, inv, bad, stream=st)
        else:
            P.pack_async(d_text, packed, bad, stream=st)

    pack()
    P.match_compact_async(a, packed, n_own, n_avail, out, pos[:0], pid[:0], count, ws, pos_base=sh.start, inv=inv)
    cap = int(count.item()) + 1024
    if world > 1:  # fixed-size list buffers: the same capacity on every rank
        ct = torch.tensor([cap], dtype=torch.int64, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(ct, op=dist.ReduceOp.MAX)
        cap = int(ct.item())
    # the rank's whole result in one buffer [count | pos[cap] | pid[cap]]: the kernel writes into it and
    # one NCCL gather moves it (no host read of the count inside a step)
    lbuf, count, pos, pid = list_buffer(cap, dev)
    gathered = None
    stream = torch.cuda.current_stream(dev)
    fused = args.path in ("fused", "list", "text", "text-list")
    list_only = args.path in ("list", "text-list")
    text_in = args.path in ("text", "text-list")  # pack fused into the match kernel (pfac_match_text_async)
    if text_in:
        ws = torch.empty(P.match_text_workspace_bytes(n_own, n_avail, list_only), dtype=torch.uint8, device=dev)
    elif list_only:  # the list without the dense out[] (scratch workspace)
        ws = torch.empty(P.match_list_workspace_bytes(n_own), dtype=torch.uint8, device=dev)
    graph_error = None
    # text path: one kernel when the image's plan takes it (pfac_image_info.text_kernel), else pack +
    # first-bad scan + fused kernel inside the call
    text_variant = a.image_info(local)["text_kernel"] if text_in and d_text.data_ptr() % 16 == 0 else 0
    text_one = text_variant in (1, 2, 3)
    kernels_per_step = (1 if text_one else 3 if text_in else 2 if fused else 3) + (1 if args.all_matches else 0)
    if args.all_matches:  # every occurrence: size the output from a probe
        ws_e = torch.empty(P.expand_workspace_bytes(), dtype=torch.uint8, device=dev)
        count_all = torch.zeros(1, dtype=torch.int64, device=dev)
        P.match_compact_async(a, packed, n_own, n_avail, out, pos, pid, count, ws, pos_base=sh.start, inv=inv)
        P.expand_async(a, pos, pid, count, pos[:0], pid[:0], count_all, ws_e)
        cap_all = int(count_all.item()) + 1024
        pos_all = torch.empty(cap_all, dtype=torch.int64, device=dev)
        pid_all = torch.empty(cap_all, dtype=torch.int32, device=dev)

    def step(ev=None, st=None):
        st = stream if st is None else st
        if ev is not None:
            ev[0].record(st)
        if not text_in:
            pack(st)
        if ev is not None:
            ev[1].record(st)
        if text_in:  # one kernel from the ASCII text: pack + match + compact
            P.match_text_async(a, d_text, n_own, n_avail, None if list_only else out, pos, pid, count, ws,
                               pos_base=sh.start, first_bad=bad, stream=st)
            if ev is not None:
                ev[2].record(st)
                ev[3].record(st)
        elif list_only:
            P.match_list_async(a, packed, n_own, n_avail, pos, pid, count, ws, pos_base=sh.start, inv=inv,
                               stream=st)
            if ev is not None:
                ev[2].record(st)
                ev[3].record(st)
        elif fused:  # match + compact in one kernel
            P.match_compact_async(a, packed, n_own, n_avail, out, pos, pid, count, ws, pos_base=sh.start,
                                  stream=st, inv=inv)
            if ev is not None:
                ev[2].record(st)
                ev[3].record(st)
        else:
            if bars:
                P.match_barriers_async(a, packed, inv, n_own, n_avail, out, stream=st)
            else:
                P.match_packed_async(a, packed, n_own, n_avail, out, stream=st)
            if ev is not None:
                ev[2].record(st)
            P.compact_async(out, pos, pid, count, ws, pos_base=sh.start, k=len(pats), stream=st)
            if ev is not None:
                ev[3].record(st)
        if args.all_matches:
            P.expand_async(a, pos, pid, count, pos_all, pid_all, count_all, ws_e, stream=st)
        if ev is not None:
            ev[4].record(st)
        if world > 1:
            return gather_lists_async(lbuf, dst=0)
        return None

    for _ in range(args.warmup):
        gathered = step()
    torch.cuda.synchronize(dev)
    gather_check = None
    if world > 1:  # the gathered lists of the last warm-up step, checked on rank 0 (not timed)
        gather_check = verify_gathered(args, gathered, cap, world, n_total, pats) if rank == 0 else None
    # sanity (not a parity claim; tests/ hold those): bad bytes only with --barriers, count fits,
    # first out[] window
    assert (int(bad.item()) == -1) != bars
    m_final = int(count.item())
    assert m_final <= cap

    # per-kernel times: K steps with events between the C-ABI calls (also the timed pass without graphs)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)

    def timed(run_steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        with clocks:
            start.record(stream)
            run_steps()
            end.record(stream)
            torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        return start.elapsed_time(end)

    def event_steps():
        for i in range(args.steps):
            step(evs[i])

    graph = None
    if args.graph and world == 1:  # the step as one CUDA graph (pack + fused kernel, no launch gaps)
        try:
            cap_stream = torch.cuda.Stream(dev)
            cap_stream.wait_stream(stream)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cap_stream):
                with torch.cuda.graph(graph, stream=cap_stream):
                    step(None, cap_stream)
            stream.wait_stream(cap_stream)
            graph.replay()
            torch.cuda.synchronize(dev)
        except Exception as ex:  # noqa: BLE001 - fall back to plain launches, reported in the JSON
            graph = None
            graph_error = repr(ex)[:200]
    kt_ms = timed(event_steps)
    kt = np.array([[e[j].elapsed_time(e[j + 1]) for j in range(4)] for e in evs])  # pack, match, compact, expand
    step_ms = kt.sum(axis=1)  # per-step times of the pass that gives ms_per_step (the event pass without a graph)
    if graph is not None:
        # the timed pass: K graph replays with an event between consecutive replays, so each step's
        # (= each launch's, for the one-kernel text path) duration comes from the same pass as ms_per_step
        clocks = ClockSampler(local)
        gev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]

        def graph_steps():
            for i in range(args.steps):
                gev[i].record(stream)
                graph.replay()
            gev[args.steps].record(stream)
        t_ms = timed(graph_steps)
        step_ms = np.array([gev[i].elapsed_time(gev[i + 1]) for i in range(args.steps)])
    else:
        t_ms = kt_ms
    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_ms = max_over_ranks(t_ms)
    ms_per_step = t_ms / args.steps
    value = n_total / (ms_per_step * 1e-3) / 1e9

    hbm, hbm_src = peaks()
    pack_ms, match_ms, compact_ms, expand_ms = (float(x) for x in np.median(kt, axis=0))
    dominant_src = "event pass (events between the C-ABI calls), median over K steps"
    if text_one and not args.all_matches and graph is not None:
        # one kernel per step: the dominant kernel's launch times are the timed pass's step times
        match_ms = float(np.median(step_ms))
        dominant_src = "timed graph pass (one kernel per replay), median over K launches"
    kstats = {name: {"median": float(np.median(kt[:, j])), "min": float(kt[:, j].min()),
                     "mean": float(kt[:, j].mean())}
              for j, name in enumerate(["pack", "match", "compact", "expand"]) if kt[:, j].max() > 0.002}
    kstats["step (timed pass)"] = {"median": float(np.median(step_ms)), "min": float(step_ms.min()),
                                   "mean": float(step_ms.mean())}
    if fused:
        compact_ms = 0.0  # inside the fused kernel
    match_bpb = MATCH_BYTES_PER_BASE + (BARRIER_BYTES_PER_BASE if bars else 0.0)
    if list_only:  # packed text read + 12 B per match written (no out[])
        match_bpb = 0.25 + (BARRIER_BYTES_PER_BASE if bars else 0.0) + 12.0 * m_final / max(1, n_own)
    if text_one:  # ASCII text read (1 B/base) + out[] written (4 B/base; list only: 12 B per match)
        match_bpb = 1.0 + (12.0 * m_final / max(1, n_own) if list_only else 4.0)
    elif text_in:  # the call's pack + first-bad + fused kernels: their bytes together
        match_bpb = (PACK_BYTES_PER_BASE + 2 * BARRIER_BYTES_PER_BASE + 0.25 +
                     (12.0 * m_final / max(1, n_own) if list_only else 4.0))
    if fused and not list_only:  # the dense paths also write the list: 12 B per match (8 pos + 4 id)
        match_bpb += 12.0 * m_final / max(1, n_own)
    pack_bpb = PACK_BYTES_PER_BASE + (BARRIER_BYTES_PER_BASE if bars else 0.0)
    match_gbs = match_bpb * n_own / (match_ms * 1e-3) / 1e9
    traffic = profiled_traffic(args.config, args.path) if args.n is None and not bars else None
    other_bounds = secondary_bounds(args.config, n_own, match_ms) if (
        args.n is None and not bars and text_one and not list_only) else None

    # ---- e2e: the same work through the C-ABI's host-memory entry point (pfac_scan_host): the text
    # from pinned HOST memory, chunked H2D overlapped with the kernels, the list copied back to HOST
    e2e = None
    if not args.no_e2e:
        e_steps = max(1, min(args.steps, args.e2e_steps))
        h_pos = torch.empty(cap, dtype=torch.int64).pin_memory()  # cap = measured count + 1024
        h_pid = torch.empty(cap, dtype=torch.int32).pin_memory()

        def e2e_step():
            _, _, mm = P.scan_host(a, h_text, pos=h_pos, pid=h_pid, device=local, n_own=n_own, pos_base=sh.start)
            if world > 1:  # this rank's host list into its list buffer, then the gather
                count.fill_(mm)
                pos[:mm].copy_(h_pos[:mm], non_blocking=True)
                pid[:mm].copy_(h_pid[:mm], non_blocking=True)
                gather_lists_async(lbuf, dst=0)
            return mm

        e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            mm = e2e_step()
        te = max_over_ranks((time.perf_counter() - t0) / e_steps * 1e3)
        e2e = {"value": n_total / (te * 1e-3) / 1e9, "unit": "Gbases/s",
               "h2d_bytes_per_step": int(n_avail), "d2h_bytes_per_step": int(12 * mm + 16),
               "steps": e_steps, "api": "pfac_scan_host (host memory in and out; wall clock, max over ranks)"}

    # ---- quick sanity against the oracle on rank 0 (window of out[]) + CPU baseline
    cpu = cpu_all = None
    if rank == 0:
        from oracle import Oracle
        w = min(n_own, 200_000)
        if list_only:
            ep, ei = Oracle(pats).match_list(text, 0, w, n=n_avail)
            assert (pos[:len(ep)].cpu().numpy() == ep.astype(np.int64) + sh.start).all()
        else:
            assert (out[:w].cpu().numpy() == Oracle(pats).match(text, 0, w, n=n_avail)).all()
        if world == 1 and not args.no_cpu_baseline:
            m, dt, _ = oracle_sample(pats, text, n_own, args.cpu_seconds)
            cpu = {"value": m / dt / 1e9, "unit": "Gbases/s", "cores": 1, "kind": "oracle",
                   "sample": f"first {m} positions of this rank's {cfg.name} text, oracle O2 "
                             f"(plain C, 1 thread), {dt:.1f} s"}
            # the same oracle on every host core (disjoint position ranges, one thread each)
            p = host_cores()
            from oracle import Oracle
            m_all = int(min(n_own, m / dt * p * args.cpu_seconds / 2))
            dt_all, _ = oracle_threads(Oracle(pats), text, m_all, n_avail, p)
            cpu_all = {"value": m_all / dt_all / 1e9, "unit": "Gbases/s", "cores": p, "kind": "oracle",
                       "sample": f"first {m_all} positions, {p} disjoint ranges on {p} threads, {dt_all:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gbases/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded SplitMix64 ACGT text, planted patterns; DESIGN.md §3)",
            "config": {"workload": workload_name(cfg, args), "n_bases_total": n_total, "n_bases_per_rank": n_own,
                       "patterns": len(pats), "states": a.num_states, "max_len": a.max_len,
                       "parallelism": f"text-sharded x{world} (halo maxlen-1)",
                       **({"ranks_per_gpu": -(-world // ndev), "backend": args.backend} if world > 1 else {}),
                       **({"gather_check": gather_check} if gather_check else {}),
                       "l2": "inputs larger than L2 (no flush): ASCII text 1 B/base, out[] 4 B/base",
                       "matches_per_step": m_final, "image": a.image_info(local),
                       **({"text_plan": text_plan} if text_plan else {})},
            "roofline": {"bound": "hbm", "achieved": match_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": match_gbs / hbm, "traffic": traffic,
                         "kernel": ("match_kernel<TXT=1" + ({2: ", 1024-position slices", 3: ", 1024-position slices claimed dynamically"}.get(text_variant, "")) +
                                    "> (pack + match + compact)" if text_one and not list_only else
                                    "match_kernel<TXT=1, list-only> (pack + match + list)" if text_one else
                                    "pack + match_kernel<FUSE=1,BAR=1> (two-kernel text path)" if text_in else
                                    "match_kernel<FUSE=1, list-only>" if list_only else
                                    "match_kernel<FUSE=1> (match + compact)" if fused else "match_kernel")
                         + ("<BAR=1>" if bars else ""),
                         "algorithmic_bytes_per_launch": match_bpb * n_own, "peak_source": hbm_src,
                         "kernel_ms": match_ms, "kernel_ms_source": dominant_src,
                         **({"other_bounds": other_bounds} if other_bounds else {})},
            "path": args.path + (" (one kernel)" if text_one else " (pack + fused kernel)" if text_in else ""),
            "cuda_graph": graph is not None, **({"cuda_graph_error": graph_error} if graph_error else {}),
            "kernels_ms": {"pack": pack_ms, ("match+compact (fused)" if fused else "match"): match_ms,
                           "compact": None if fused else compact_ms,
                           **({"expand": expand_ms, "occurrences": int(count_all.item())} if args.all_matches else {}),
                           "pack_frac": (pack_bpb * n_own / (pack_ms * 1e-3) / 1e9 / hbm if not text_in else None),
                           "compact_frac": (COMPACT_BYTES_PER_BASE * n_own / (compact_ms * 1e-3) / 1e9 / hbm
                                            if compact_ms > 0 else None)},
            "kernels_ms_stats": kstats,
            "match_gbases_per_s_per_gpu": n_own / (match_ms * 1e-3) / 1e9,
            "build_ms": build_ms, "prepare_ms": prepare_ms, "gen_s": t_gen,
            "cpu_baseline": cpu, "cpu_baseline_all_cores": cpu_all, "e2e": e2e,
            "gpu_launches": kernels_per_step * args.steps,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["pfac", "reference"], default="pfac")
    ap.add_argument("--config", type=int, default=None, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (default: 2 at N = 1, 3 at N > 1)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="N > 1: strong (default; the config's text split across the ranks) or weak "
                         "(each rank a config-sized shard of an N-times longer text)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the step's kernels directly instead of replaying one captured CUDA graph")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="process group for N>1 (gloo only to test the multi-rank flow on one GPU)")
    ap.add_argument("--path", choices=["fused", "separate", "list", "text", "text-list"], default="text",
                    help="text (default): pfac_match_text_async, one kernel from the ASCII text where the "
                         "image's plan prefers it (else pack -> match+compact inside the call); fused: pack -> match+compact kernel; separate: pack -> match -> compact; "
                         "list: pack -> list-only match (no dense out[]); text: one kernel from the ASCII "
                         "text (pack + match + compact); text-list: the same without out[]")
    ap.add_argument("--bases-per-rank", dest="n", type=int, default=None, help="override bases per rank (testing)")
    ap.add_argument("--barriers", type=int, default=None, metavar="LINE",
                    help="FASTA-like text: a newline every LINE bases + N gaps; runs the barrier kernels")
    ap.add_argument("--all-matches", action="store_true",
                    help="add the all-occurrence expansion (pfac_expand_async) to the timed step")
    ap.add_argument("--text-kernel", type=int, default=None, choices=[-1, 0, 1, 2, 3],
                    help="pfac_set_text_kernel mode for the text path (default: the library's plan)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-budget", type=float, default=60.0, help="reference arm: total seconds")
    ap.add_argument("--ref-cores", type=int, default=0, help="reference arm threads (0: every host core)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:  # one process per GPU: re-launch under torch.distributed.run
        return relaunch(args.gpus)
    world = max(world, 1)
    if world != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N ranks for --gpus N")
    if args.config is None:
        args.config = 2 if world == 1 else 3
    if args.scaling is None:
        args.scaling = "weak" if world == 1 else "strong"
    return run_reference(args) if args.impl == "reference" else run_pfac(args)


def relaunch(n: int) -> int:
    """`python bench.py --gpus N ...` without WORLD_SIZE: exec torch.distributed.run with N ranks on
    this node (rendezvous on 127.0.0.1, a free port), forwarding every argument."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)
    return 1  # not reached


if __name__ == "__main__":
    sys.exit(main())
