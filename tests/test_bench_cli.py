"""bench.py's launch contract on CPU (no GPU needed): `--gpus N` without WORLD_SIZE re-launches the
script under torch.distributed.run with N ranks (rank 0 alone prints one JSON line), a WORLD_SIZE
that disagrees with --gpus is an error, and N > 1 defaults to the 3.1 Gbp config, strong scaling.
The reference arm (the oracle on the host) is the leg that runs without a GPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=240):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=e, timeout=timeout, cwd=ROOT)


def test_gpus2_relaunches_two_ranks_one_line():
    r = _run(["--gpus", "2", "--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "3",
              "--ref-budget", "1", "--ref-cores", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["workload"].startswith("cfg1")


def test_default_config_at_n_gt_1_is_cfg3_strong():
    r = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "3", "--ref-budget", "1",
              "--ref-cores", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    assert d["config"]["workload"].startswith("cfg3") and d["scaling"] == "strong" and d["n_gpus"] == 2


def test_world_size_mismatch_is_an_error():
    r = _run(["--gpus", "2", "--impl", "reference", "--config", "1"], env={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
