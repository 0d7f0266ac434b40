"""GPU parity (-m gpu) of the N-GPU path with the product kernels.

Two ranks (one process each, torch.multiprocessing spawn).  Each rank regenerates only its shard of
the text -- owned positions [s_g, e_g) plus a (maxlen - 1)-base halo -- runs the CUDA text call
(pfac_match_text_async: pack + match + compact in one kernel) with pos_base = s_g into its list
buffer, and the buffers are gathered to rank 0 (parallel.ShardedMatcher).  Rank 0's concatenation
must equal the oracle's list of the WHOLE text, and each rank's dense out[] the oracle's out[] of
its owned range.  Backend: NCCL when >= 2 GPUs are visible (one per rank), else gloo with both
ranks on cuda:0 (the collective then runs on host copies; the kernels are the same).
"""
import os
import socket

import numpy as np
import pytest

import pfac_datagen as gen
from oracle import Oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pats(kind):
    if kind == "cfg1":
        return gen.config_patterns(gen.CONFIGS[1])
    if kind == "big32":  # uint32 image with the second-level table (the cfg3/cfg4 image kind)
        return gen.random_patterns(31, 40_000, 16, 64)
    raise ValueError(kind)


def _text(kind, a, b, n, pats):
    if kind == "fasta":
        t = gen.plant(gen.iid_text(7, a, b), a, n, pats, 7).copy()
        return gen.add_barriers(t, 7, line=80, a=a)
    return gen.plant(gen.iid_text(7, a, b), a, n, pats, 7)


def _rank(rank, world, port, backend, n, pkind, tkind, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", rank % ndev)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1811_10498_b200 as P
        from paper_1811_10498_b200.parallel import ShardedMatcher, agree_capacity, probe_count, shard, unpack_lists
        pats = _pats(pkind)
        a = P.Automaton(pats)
        sh = shard(n, world, rank, a.max_len)
        text = _text(tkind, sh.start, sh.avail_end, n, pats)
        d_text = torch.from_numpy(text).to(dev)
        cap = agree_capacity(probe_count(a, d_text, sh))
        m = ShardedMatcher(a, d_text, sh, cap)
        for _ in range(2):  # the same step twice: buffers are reused across steps
            g = m.step()
        torch.cuda.synchronize(dev)
        out_ok = bool((m.out.cpu().numpy() == Oracle(pats).match(text, 0, sh.n_own, n=sh.n_avail)).all())
        oks = [None] * world
        dist.all_gather_object(oks, out_ok)
        if rank == 0:
            gp, gi, counts = unpack_lists(g, cap)
            q.put((gp.numpy(), gi.numpy(), counts, oks, cap))
    except Exception as e:  # noqa: BLE001 - reported to the parent
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("pkind,tkind,n", [("cfg1", "iid", 2_000_003), ("big32", "iid", 3_000_000),
                                           ("cfg1", "fasta", 1_500_000)])
def test_two_rank_sharded_text_call_equals_oracle(pkind, tkind, n):
    import torch.multiprocessing as mp
    world = 2
    backend = "nccl" if torch.cuda.device_count() >= world else "gloo"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, backend, n, pkind, tkind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert not isinstance(res, str), res
    for p in procs:
        assert p.exitcode == 0
    gp, gi, counts, oks, cap = res
    assert all(oks), f"a rank's dense out[] differs from the oracle: {oks}"
    pats = _pats(pkind)
    text = _text(tkind, 0, n, n, pats)
    epos, epid = Oracle(pats).match_list(text)
    assert len(counts) == world and sum(counts) == len(epos) > 100 and max(counts) <= cap
    assert (gp == epos.astype(np.int64)).all() and (gi == epid).all()
    assert (np.diff(gp) > 0).all()  # rank order = position order
