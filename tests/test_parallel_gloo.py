"""N>1 host logic on CPU: sharding with halo + the gather, world_size 2 (and 3) over gloo.

The per-rank match lists here come from the oracle (tests may call it); the product's per-rank
compute is the CUDA path, covered by tests/test_gpu_parity.py::test_match_packed_shard_window.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import pfac_datagen as gen
from oracle import Oracle
from paper_1811_10498_b200.parallel import gather_lists_async, gather_matches, list_buffer, shard, unpack_lists


def test_shard_bounds_cover_and_align():
    for n in [0, 1, 63, 64, 1000, 1_000_003, 3_100_000_000]:
        for G in [1, 2, 3, 4, 8]:
            maxlen = 64
            sh = [shard(n, G, g, maxlen) for g in range(G)]
            assert sh[0].start == 0 and sh[-1].end == n
            for a, b in zip(sh, sh[1:]):
                assert a.end == b.start
            for s in sh:
                assert s.start % 64 == 0
                assert s.start <= s.end <= s.avail_end <= n
                assert s.avail_end == (min(n, s.end + maxlen - 1) if s.end > s.start else s.end)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pats = gen.random_patterns(8, 80, 4, 30)
        sh = shard(n, world, rank, max(len(p) for p in pats))
        # this rank sees only its own text slice (owned + halo), regenerated position-addressably
        text = gen.plant(gen.iid_text(8, sh.start, sh.avail_end), sh.start, n, pats, 8)
        pos, pid = Oracle(pats).match_list(text, 0, sh.n_own, n=sh.n_avail)
        pos_t = torch.from_numpy(pos.astype(np.int64) + sh.start)
        pid_t = torch.from_numpy(pid.astype(np.int32))
        gp, gi, counts = gather_matches(pos_t, pid_t, len(pos), dst=0)
        if rank == 0:
            q.put((gp.numpy(), gi.numpy(), counts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gather_equals_single_run(world):
    n = 300_000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    gp, gi, counts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pats = gen.random_patterns(8, 80, 4, 30)
    text = gen.plant(gen.iid_text(8, 0, n), 0, n, pats, 8)
    epos, epid = Oracle(pats).match_list(text)
    assert sum(counts) == len(epos) > 50
    assert (gp == epos.astype(np.int64)).all() and (gi == epid).all()


def _worker_buf(rank, world, port, n, q):
    """The sync-free form: each rank's result in one list buffer, one gather of the buffers."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pats = gen.random_patterns(9, 120, 4, 25)
        sh = shard(n, world, rank, max(len(p) for p in pats))
        text = gen.plant(gen.iid_text(9, sh.start, sh.avail_end), sh.start, n, pats, 9)
        pos, pid = Oracle(pats).match_list(text, 0, sh.n_own, n=sh.n_avail)
        cap = 20_000  # the same on every rank (fixed-size buffers); each rank's list fits
        buf, count, bpos, bpid = list_buffer(cap, "cpu")
        count[0] = len(pos)  # what the match kernel writes on the GPU
        bpos[:len(pos)] = torch.from_numpy(pos.astype(np.int64) + sh.start)
        bpid[:len(pid)] = torch.from_numpy(pid.astype(np.int32))
        g = gather_lists_async(buf, dst=0)
        if rank == 0:
            gp, gi, counts = unpack_lists(g, cap)
            q.put((gp.numpy(), gi.numpy(), counts))
    finally:
        dist.destroy_process_group()


def test_list_buffer_gather_equals_single_run():
    world, n = 3, 400_000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_buf, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    gp, gi, counts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pats = gen.random_patterns(9, 120, 4, 25)
    text = gen.plant(gen.iid_text(9, 0, n), 0, n, pats, 9)
    epos, epid = Oracle(pats).match_list(text)
    assert sum(counts) == len(epos) > 50 and len(counts) == world
    assert (gp == epos.astype(np.int64)).all() and (gi == epid).all()
