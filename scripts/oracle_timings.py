#!/usr/bin/env python
"""The CPU oracle O2 (as it stands: plain C, -O2) timed on the box's host cores, per config
(SURVEY.md §8(d) "Oracle timing beside it"): 1 thread on cfg1, cfg2 and cfg5; P threads over
disjoint position ranges on cfg3 and cfg4 (P = the cores this process may run on).  Each config runs
a bounded prefix of its text, sized from a probe to about --seconds of CPU work.  The timed region
is the matching loop only (oracle_match_list: walks + the list), not the build or text generation.

  python scripts/oracle_timings.py [--seconds 12] > profiles/r02_oracle_timings.json
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=12.0)
    ap.add_argument("--configs", default="1,2,3,4,5")
    args = ap.parse_args()
    import pfac_datagen as gen
    from oracle import Oracle
    sys.path.insert(0, os.path.join(ROOT))
    from bench import host_cores, oracle_threads

    P = host_cores()
    res = {"cpu": cpu_model(), "host_cores": P, "oracle": "O2 (oracle/pfac_oracle.c, gcc -O2), match_list",
           "configs": {}}
    for c in [int(x) for x in args.configs.split(",")]:
        cfg = gen.CONFIGS[c]
        pats = gen.config_patterns(cfg)
        maxlen = max(len(p) for p in pats)
        t0 = time.perf_counter()
        o = Oracle(pats)
        build_s = time.perf_counter() - t0
        threads = P if c in (3, 4) else 1
        probe = min(cfg.n, 1_000_000 * threads)
        text = gen.config_text(cfg, 0, min(cfg.n, probe + maxlen - 1), patterns=pats, n=cfg.n)
        dt, _ = oracle_threads(o, text, probe, len(text), threads)
        m = int(min(cfg.n, max(probe, probe / max(dt, 1e-6) * args.seconds)))
        text = gen.config_text(cfg, 0, min(cfg.n, m + maxlen - 1), patterns=pats, n=cfg.n)
        dt, matches = oracle_threads(o, text, m, len(text), threads)
        reps = 1
        if dt < args.seconds / 2:  # the whole text is shorter than the budget (cfg1): repeat it
            reps = max(1, int(args.seconds / max(dt, 1e-6)))
            dt = sum(oracle_threads(o, text, m, len(text), threads)[0] for _ in range(reps)) / reps
        res["configs"][f"cfg{c}"] = {
            "workload": cfg.name, "threads": threads, "positions": m, "seconds": dt,
            "gbases_per_s": m / dt / 1e9, "matches": matches, "build_s": build_s, "repetitions": reps,
            "sample": f"first {m} positions of the {cfg.n}-base text" +
                      (f", {threads} disjoint ranges on {threads} threads" if threads > 1 else ", 1 thread"),
        }
        print(f"cfg{c}: {m / dt / 1e9:.4f} Gbases/s on {threads} thread(s), {m} positions, {dt:.1f} s",
              file=sys.stderr, flush=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
