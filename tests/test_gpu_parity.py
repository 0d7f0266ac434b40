"""GPU parity (-m gpu): the CUDA path through the C-ABI vs the oracle, element by element.

Bar: bit-exact (integer path).  Sizes span many tiles (8192 positions) and ragged tails; the full
configs compare the complete match lists (equivalent to out[] equality, since out[i] = 0 iff i is
absent) plus sampled out[] windows.
"""
import os

import numpy as np
import pytest

import pfac_datagen as gen
from oracle import Oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # the gpu marker is deselected on CPU runs; be explicit anyway
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1811_10498_b200 as P  # noqa: E402
from paper_1811_10498_b200 import binding as B  # noqa: E402

DEV = torch.device("cuda:0")
TILE = 8192


def to_dev(t: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(t)).to(DEV)


def gpu_match(a, text: np.ndarray) -> np.ndarray:
    out = P.match(a, to_dev(text))
    return out.cpu().numpy()


def np_pack(text: np.ndarray) -> np.ndarray:
    """Test-side packing (definition in include/pfac.h): A0 C1 G2 T3, base j at bits 2(j mod 16)."""
    lut = np.zeros(256, dtype=np.uint32)
    for ch, c in zip(b"ACGTacgt", [0, 1, 2, 3, 0, 1, 2, 3]):
        lut[ch] = c
    n = len(text)
    words = B.packed_words(n)
    codes = np.zeros(words * 16, dtype=np.uint32)
    codes[:n] = lut[text]
    codes = codes.reshape(-1, 16)
    return (codes << (2 * np.arange(16, dtype=np.uint32))).sum(axis=1, dtype=np.uint64).astype(np.uint32)


# --------------------------------------------------------------------------- pack
@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 63, 64, 65, 1000, 4099, 100_003])
@pytest.mark.parametrize("offset", [0, 3])
def test_pack_matches_definition(n, offset):
    rng = np.random.default_rng(n + offset)
    text = np.frombuffer(b"ACGTacgt", np.uint8)[rng.integers(0, 8, n)]
    buf = torch.zeros(n + 16, dtype=torch.uint8, device=DEV)
    buf[offset:offset + n] = to_dev(text) if n else buf[:0]
    dtext = buf[offset:offset + n]
    bad = torch.zeros(1, dtype=torch.int64, device=DEV)
    packed = P.pack_async(dtext, first_bad=bad)
    torch.cuda.synchronize()
    got = packed.cpu().numpy().view(np.uint32)
    assert (got == np_pack(text)).all()
    assert int(bad.item()) == -1  # UINT64_MAX: no bad byte


@pytest.mark.parametrize("where", [[0], [5, 70], [65], [99_999, 12], [4096 * 3 + 7]])
def test_pack_first_bad(where):
    text = gen.iid_text(1, 0, 100_000).copy()
    for w in where:
        text[w] = ord("N")
    bad = torch.zeros(1, dtype=torch.int64, device=DEV)
    P.pack_async(to_dev(text), first_bad=bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == min(where)
    a = P.Automaton([b"ACGT"])  # non-ACGT bytes are barriers (reading R5; tests/test_gpu_barriers.py)
    assert (P.match(a, to_dev(text)).cpu().numpy() == Oracle([b"ACGT"]).match(text)).all()


# --------------------------------------------------------------------------- match
def test_match_config1_full():
    cfg = gen.CONFIGS[1]
    pats = gen.config_patterns(cfg)
    text = gen.config_text(cfg, patterns=pats)
    exp = Oracle(pats).match(text)
    got = gpu_match(P.Automaton(pats), text)
    assert (got == exp).all()
    assert (exp != 0).sum() > 200


def test_hand_outputs_on_gpu(golden):
    for case in golden("hand_outputs.json")["cases"]:
        t = case["text"].encode()
        if not t:
            continue
        got = gpu_match(P.Automaton([p.encode() for p in case["patterns"]]), np.frombuffer(t, np.uint8))
        assert got.tolist() == case["out"], case


EDGE_N = [1, 2, 3, 7, 15, 16, 63, 64, 65, 127, 128, 129, 511, 512, 513, TILE - 1, TILE, TILE + 1,
          2 * TILE + 77, 148 * TILE + 5, 300 * TILE + 4093]


@pytest.mark.parametrize("n", EDGE_N)
def test_edge_sizes(n):
    pats = gen.random_patterns(17, 60, 1, 12) + [b"ACGTACGTACGTACGTACGTAC"]
    text = gen.plant(gen.iid_text(17, 0, n), 0, n, pats, 17)
    got = gpu_match(P.Automaton(pats), text)
    assert (got == Oracle(pats).match(text)).all()


@pytest.mark.parametrize("k", [1, 2, 6, 7, 8, 9])
def test_all_kmers(k):
    """4^k k-mers (k around the jump length K=7): closed form out[i] = 1 + value4(text[i..i+k))."""
    pats = gen.all_kmers(k)
    n = 200_003
    text = gen.iid_text(k, 0, n)
    got = gpu_match(P.Automaton(pats), text)
    codes = np.searchsorted(np.frombuffer(b"ACGT", np.uint8), text).astype(np.int64)
    val = np.zeros(n - k + 1, dtype=np.int64)
    for j in range(k):
        val = val * 4 + codes[j:n - k + 1 + j]
    exp = np.zeros(n, dtype=np.int64)
    exp[:n - k + 1] = 1 + val
    assert (got == exp).all()


def test_long_walks_cross_tiles_and_halo():
    """Patterns up to 1000 bases (> the 64-base halo granularity, < PFAC_MAX_LEN) planted densely."""
    rng = np.random.default_rng(5)
    base = gen.iid_text(23, 0, 1200)
    pats = [base[:L].tobytes() for L in (900, 1000, 999, 8, 9, 150)] + gen.random_patterns(23, 20, 30, 1000)
    pats = list(dict.fromkeys(pats))
    n = 6 * TILE + 333
    text = gen.iid_text(24, 0, n)
    for s in list(range(TILE - 500, n - 1000, 1777)) + [n - 1000, n - 999, n - 950]:
        p = pats[int(rng.integers(0, len(pats)))]
        text[s:s + len(p)] = np.frombuffer(p[: n - s], np.uint8)
    got = gpu_match(P.Automaton(pats), text)
    assert (got == Oracle(pats).match(text)).all()


def test_nested_homopolymer_family():
    pats = [b"A" * L for L in range(1, 101)] + [b"C" * L for L in range(8, 101)]
    text = np.frombuffer((b"A" * 5000 + b"G" + b"C" * 300 + b"T") * 7, np.uint8)
    got = gpu_match(P.Automaton(pats), text)
    assert (got == Oracle(pats).match(text)).all()


def test_no_patterns_and_short_text():
    a = P.Automaton([])
    assert (gpu_match(a, gen.iid_text(1, 0, 10_000)) == 0).all()
    pats = [b"ACGTACGTACGTACGTACGTACG"]
    text = np.frombuffer(b"ACGTACGTACG", np.uint8)  # n < maxlen
    assert (gpu_match(P.Automaton(pats), text) == 0).all()


def test_match_packed_shard_window():
    """out for [0, n_own) with walks bounded by n_avail (the shard + halo form)."""
    pats = gen.random_patterns(31, 200, 5, 40)
    n = 20 * TILE + 123
    text = gen.plant(gen.iid_text(31, 0, n), 0, n, pats, 31)
    a = P.Automaton(pats)
    o = Oracle(pats)
    packed = P.pack_async(to_dev(text))
    for n_own, n_avail in [(n, n), (5 * TILE, 5 * TILE + 39), (5 * TILE + 17, 5 * TILE + 17), (1000, n)]:
        out = P.match_packed_async(a, packed, n_own, n_avail)
        torch.cuda.synchronize()
        assert (out.cpu().numpy() == o.match(text, 0, n_own, n=n_avail)).all(), (n_own, n_avail)


# --------------------------------------------------------------------------- compact
def test_compact_config1_and_hist():
    cfg = gen.CONFIGS[1]
    pats = gen.config_patterns(cfg)
    text = gen.config_text(cfg, patterns=pats)
    a = P.Automaton(pats)
    out = P.match(a, to_dev(text))
    hist = torch.zeros(len(pats) + 1, dtype=torch.int64, device=DEV)
    pos, pid, m = P.compact(out, pos_base=1000, k=len(pats), hist=hist, capacity=10_000)
    epos, epid = Oracle(pats).match_list(text)
    assert m == len(epos)
    assert (pos.cpu().numpy() == epos.astype(np.int64) + 1000).all()
    assert (pid.cpu().numpy() == epid).all()
    eh = np.bincount(epid, minlength=len(pats) + 1)
    assert (hist.cpu().numpy() == eh).all() and eh.sum() == m


def test_compact_dense_and_capacity():
    n = 3 * 4096 * 7 + 5
    rng = np.random.default_rng(9)
    vals = np.where(rng.random(n) < 0.3, rng.integers(1, 50, n), 0).astype(np.int32)
    out = to_dev(vals)
    nz = np.nonzero(vals)[0]
    pos, pid, m = P.compact(out, capacity=len(nz) + 10, k=49)
    assert m == len(nz) and (pos.cpu().numpy() == nz).all() and (pid.cpu().numpy() == vals[nz]).all()
    cap = len(nz) // 3
    with pytest.raises(B.PfacError) as e:
        P.compact(out, capacity=cap, k=49)
    assert e.value.code == B.E_CAPACITY
    # empty and all-zero inputs
    assert P.compact(torch.zeros(0, dtype=torch.int32, device=DEV), capacity=4)[2] == 0
    assert P.compact(torch.zeros(100_000, dtype=torch.int32, device=DEV), capacity=4)[2] == 0


def test_compact_async_workspace_reuse():
    n = 500_000
    rng = np.random.default_rng(3)
    a_vals = np.where(rng.random(n) < 0.01, 7, 0).astype(np.int32)
    ws = torch.empty(P.compact_workspace_bytes(n), dtype=torch.uint8, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    pos = torch.empty(n, dtype=torch.int64, device=DEV)
    pid = torch.empty(n, dtype=torch.int32, device=DEV)
    for rep in range(3):
        vals = np.roll(a_vals, rep * 1000)
        P.compact_async(to_dev(vals), pos, pid, cnt, ws, pos_base=0, k=10)
        torch.cuda.synchronize()
        nz = np.nonzero(vals)[0]
        m = int(cnt.item())
        assert m == len(nz) and (pos[:m].cpu().numpy() == nz).all()


# --------------------------------------------------------------------------- full-size configs
def _oracle_list_parallel(pats, text, procs=None):
    import multiprocessing as mp
    procs = procs or min(32, len(os.sched_getaffinity(0)))
    n = len(text)
    bounds = [n * i // procs for i in range(procs + 1)]
    global _G
    _G = (pats, text)
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        parts = pool.map(_oracle_chunk, list(zip(bounds[:-1], bounds[1:])))
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


_G = None


def _oracle_chunk(ab):
    pats, text = _G
    return Oracle(pats).match_list(text, ab[0], ab[1])


def _full_config(idx):
    cfg = gen.CONFIGS[idx]
    pats = gen.config_patterns(cfg)
    text = gen.config_text(cfg, patterns=pats)
    a = P.Automaton(pats)
    dtext = to_dev(text)
    out = P.match(a, dtext)
    pos, pid, m = P.compact(out, k=len(pats))
    epos, epid = _oracle_list_parallel(pats, text)
    assert m == len(epos)
    assert (pos.cpu().numpy() == epos.astype(np.int64)).all()
    assert (pid.cpu().numpy() == epid).all()
    # the fused match+compact path (the bench default) on the same full input
    n = len(text)
    packed = P.pack_async(dtext)
    out2 = torch.empty(n, dtype=torch.int32, device=DEV)
    cap = len(epos) + 1024
    pos2 = torch.empty(cap, dtype=torch.int64, device=DEV)
    pid2 = torch.empty(cap, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(P.compact_workspace_bytes(n), dtype=torch.uint8, device=DEV)
    P.match_compact_async(a, packed, n, n, out2, pos2, pid2, cnt, ws)
    torch.cuda.synchronize()
    assert int(cnt.item()) == len(epos)
    assert (pos2[:len(epos)].cpu().numpy() == epos.astype(np.int64)).all()
    assert (pid2[:len(epos)].cpu().numpy() == epid).all()
    assert bool((out2 == out).all())
    del out2
    # the list-only path (no dense out[]) on the same full input
    ws = torch.empty(P.match_list_workspace_bytes(n), dtype=torch.uint8, device=DEV)
    pos2.fill_(-1)
    P.match_list_async(a, packed, n, n, pos2, pid2, cnt, ws)
    torch.cuda.synchronize()
    assert int(cnt.item()) == len(epos)
    assert (pos2[:len(epos)].cpu().numpy() == epos.astype(np.int64)).all()
    assert (pid2[:len(epos)].cpu().numpy() == epid).all()
    del packed, ws
    # the text-input call (pack fused into the kernel; the bench default where the plan takes it) in
    # both of its paths, on the same full input: list, count, first_bad and the whole dense out[]
    for mode in (1, 0, 2, 3):
        a.set_text_kernel(mode)
        ws = torch.empty(P.match_text_workspace_bytes(n, n), dtype=torch.uint8, device=DEV)
        out3 = torch.empty(n, dtype=torch.int32, device=DEV)
        bad = torch.zeros(1, dtype=torch.int64, device=DEV)
        pos2.fill_(-1)
        P.match_text_async(a, dtext, n, n, out3, pos2, pid2, cnt, ws, first_bad=bad)
        torch.cuda.synchronize()
        assert int(cnt.item()) == len(epos) and int(bad.item()) == -1
        assert (pos2[:len(epos)].cpu().numpy() == epos.astype(np.int64)).all()
        assert (pid2[:len(epos)].cpu().numpy() == epid).all()
        assert bool((out3 == out).all())
        del out3, ws
    a.set_text_kernel(-1)
    # sampled out[] windows (every element, including the zeros)
    o = Oracle(pats)
    n = len(text)
    for s in [0, n // 3 + 5, n - 70_001]:
        assert (out[s:s + 70_000].cpu().numpy() == o.match(text, s, s + 70_000)).all()
    return m


def test_config2_full():
    m = _full_config(2)
    assert m > 60_000


def test_config5_full():
    _full_config(5)


@pytest.mark.skipif(bool(os.environ.get("PFAC_SKIP_FULL")), reason="PFAC_SKIP_FULL set (3.1 Gbp / 1 Gbp runs)")
@pytest.mark.parametrize("idx", [3, 4])
def test_config3_config4_full(idx):
    _full_config(idx)


# --------------------------------------------------------------------------- fused match + compact
def _fused(a, text, n_own=None, n_avail=None, pos_base=0, cap=None, k=0, hist=None):
    n = len(text)
    n_own = n if n_own is None else n_own
    n_avail = n if n_avail is None else n_avail
    packed = P.pack_async(to_dev(text))
    out = torch.empty(max(n_own, 1), dtype=torch.int32, device=DEV)
    cap = n_own + 16 if cap is None else cap
    pos = torch.empty(max(cap, 1), dtype=torch.int64, device=DEV)
    pid = torch.empty(max(cap, 1), dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(P.compact_workspace_bytes(n_own), dtype=torch.uint8, device=DEV)
    P.binding.match_compact_async(a, packed, n_own, n_avail, out, pos[:cap] if cap else pos[:0], pid[:cap] if cap else pid[:0],
                                  cnt, ws, pos_base=pos_base, hist=hist)
    torch.cuda.synchronize()
    m = int(cnt.item())
    return out[:n_own].cpu().numpy(), pos[:min(m, cap)].cpu().numpy(), pid[:min(m, cap)].cpu().numpy(), m


@pytest.mark.parametrize("case", ["cfg1", "short", "kmers8", "shard", "edge"])
def test_fused_match_compact(case):
    if case == "cfg1":
        cfg = gen.CONFIGS[1]
        pats = gen.config_patterns(cfg)
        text = gen.config_text(cfg, patterns=pats)
        kw = {}
    elif case == "short":  # patterns shorter than K: dead jump-table cells carry answers
        pats = gen.random_patterns(41, 300, 1, 12)
        n = 50 * 1024 + 77
        text = gen.plant(gen.iid_text(41, 0, n), 0, n, pats, 41)
        kw = {}
    elif case == "kmers8":  # every position matches: staging overflows, warps re-read out[]
        pats = gen.all_kmers(4)
        text = gen.iid_text(42, 0, 700_001)
        kw = {}
    elif case == "shard":
        pats = gen.random_patterns(43, 200, 5, 40)
        n = 200_000
        text = gen.plant(gen.iid_text(43, 0, n), 0, n, pats, 43)
        kw = dict(n_own=150_003, n_avail=150_003 + 39, pos_base=10_000_000)
    else:
        pats = gen.random_patterns(44, 60, 1, 12) + [b"ACGTACGTACGTACGTACGTAC"]
        text = gen.plant(gen.iid_text(44, 0, 1000), 0, 1000, pats, 44)
        kw = {}
    a = P.Automaton(pats)
    hist = torch.zeros(len(pats) + 1, dtype=torch.int64, device=DEV)
    out, pos, pid, m = _fused(a, text, hist=hist, **kw)
    o = Oracle(pats)
    n_own, n_avail = kw.get("n_own", len(text)), kw.get("n_avail", len(text))
    exp = o.match(text, 0, n_own, n=n_avail)
    assert (out == exp).all()
    epos, epid = o.match_list(text, 0, n_own, n=n_avail)
    assert m == len(epos)
    assert (pos == epos.astype(np.int64) + kw.get("pos_base", 0)).all() and (pid == epid).all()
    assert (hist.cpu().numpy() == np.bincount(epid, minlength=len(pats) + 1)).all()


def test_fused_capacity_reports_total():
    pats = gen.all_kmers(3)
    text = gen.iid_text(45, 0, 100_000)
    out, pos, pid, m = _fused(P.Automaton(pats), text, cap=1000)
    assert m == 100_000 - 2 and len(pos) == 1000
    assert (pos == np.arange(1000)).all()


# --------------------------------------------------------------------------- large automata (uint32 image + J2)
@pytest.mark.parametrize("lo,hi,k", [(16, 40, 3000), (8, 30, 5000), (1, 14, 40_000)])
def test_large_automaton_second_level_jump(lo, hi, k):
    """uint32 images resolve walks through the L2-resident J2 (K2-mers); short patterns make dead J2
    cells carry answers (patterns shorter than K2)."""
    pats = gen.random_patterns(50 + lo, k, lo, hi)
    n = 300 * 1024 + 555
    text = gen.plant(gen.iid_text(50 + lo, 0, n), 0, n, pats, 50 + lo)
    a = P.Automaton(pats)
    assert a.num_states >= 32768 or k >= 32768  # the uint32 image
    o = Oracle(pats)
    assert (gpu_match(a, text) == o.match(text)).all()
    out, pos, pid, m = _fused(a, text)
    epos, epid = o.match_list(text)
    assert (out == o.match(text)).all() and m == len(epos)
    assert (pos == epos.astype(np.int64)).all() and (pid == epid).all()


# --------------------------------------------------------------------------- end to end over host memory
@pytest.mark.parametrize("n", [1, 1000, (1 << 26) + 12345, (1 << 27) + 3])
def test_scan_host_chunked(n):
    """pfac_scan_host streams the host text in 64 Mbase chunks with a halo; list == oracle's."""
    pats = gen.random_patterns(60, 300, 12, 40)
    text = gen.plant(gen.iid_text(60, 0, n), 0, n, pats, 60)
    # a pattern straddling the chunk boundary
    if n > (1 << 26):
        text[(1 << 26) - 10:(1 << 26) - 10 + len(pats[0])] = np.frombuffer(pats[0], np.uint8)
    pos, pid, m = P.scan_host(P.Automaton(pats), torch.from_numpy(text))
    epos, epid = _oracle_list_parallel(pats, text)
    assert m == len(epos)
    assert (pos.numpy() == epos.astype(np.int64)).all() and (pid.numpy() == epid).all()


def test_scan_host_dense_and_bad_byte():
    pats = gen.all_kmers(2)
    text = gen.iid_text(61, 0, 300_000)
    pos, pid, m = P.scan_host(P.Automaton(pats), torch.from_numpy(text), pos=torch.empty(10, dtype=torch.int64),
                              pid=torch.empty(10, dtype=torch.int32))
    assert m == 300_000 - 1 and (pos.numpy() == np.arange(m)).all()
    text[123_456] = ord("N")  # a barrier: the two 2-mers containing it vanish (reading R5)
    pos, pid, m = P.scan_host(P.Automaton(pats), torch.from_numpy(text))
    exp = np.setdiff1d(np.arange(300_000 - 1), [123_455, 123_456])
    assert m == len(exp) and (pos.numpy() == exp).all()


def test_scan_host_shard_window():
    pats = gen.random_patterns(62, 200, 10, 30)
    n = 400_000
    text = gen.plant(gen.iid_text(62, 0, n), 0, n, pats, 62)
    pos, pid, m = P.scan_host(P.Automaton(pats), torch.from_numpy(text), n_own=250_001, pos_base=7)
    epos, epid = Oracle(pats).match_list(text, 0, 250_001, n=n)
    assert m == len(epos) and (pos.numpy() == epos.astype(np.int64) + 7).all() and (pid.numpy() == epid).all()


def test_config2_fasta_full_text_kernel():
    """The bench's --barriers 80 workload at full size (cfg2 text with a newline every 80 bases and
    N gaps, reading R5) through the text call in both of its paths: the whole list, the first bad
    index, and sampled out[] windows, against the oracle."""
    cfg = gen.CONFIGS[2]
    pats = gen.config_patterns(cfg)
    text = gen.config_text(cfg, patterns=pats)
    gen.add_barriers(text, cfg.seed, line=80, block=1 << 20, run_max=100_000, run_frac=0.2)
    n = len(text)
    a = P.Automaton(pats)
    dtext = to_dev(text)
    epos, epid = _oracle_list_parallel(pats, text)
    bad_idx = int(np.nonzero(~np.isin(text[:1000], np.frombuffer(b"ACGTacgt", np.uint8)))[0][0])
    o = Oracle(pats)
    for mode in (1, 0, 3):
        a.set_text_kernel(mode)
        out = torch.empty(n, dtype=torch.int32, device=DEV)
        cap = len(epos) + 1024
        pos = torch.full((cap,), -1, dtype=torch.int64, device=DEV)
        pid = torch.empty(cap, dtype=torch.int32, device=DEV)
        cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
        bad = torch.zeros(1, dtype=torch.int64, device=DEV)
        ws = torch.empty(P.match_text_workspace_bytes(n, n), dtype=torch.uint8, device=DEV)
        P.match_text_async(a, dtext, n, n, out, pos, pid, cnt, ws, first_bad=bad)
        torch.cuda.synchronize()
        assert int(cnt.item()) == len(epos) and int(bad.item()) == bad_idx
        assert (pos[:len(epos)].cpu().numpy() == epos.astype(np.int64)).all()
        assert (pid[:len(epos)].cpu().numpy() == epid).all()
        for s in [0, n // 2 + 3, n - 90_001]:
            assert (out[s:s + 90_000].cpu().numpy() == o.match(text, s, s + 90_000)).all()
        del out, ws
    a.set_text_kernel(-1)


@pytest.mark.skipif(bool(os.environ.get("PFAC_SKIP_FULL")), reason="PFAC_SKIP_FULL set (4.3 Gbase run)")
def test_text_beyond_2pow32_positions():
    """Maximum-size edge: a text longer than 2^32 bases (64-bit positions, slice indices and byte
    offsets end to end) through the text call in both paths; the whole list against the oracle and
    every out[] element of windows straddling 2^32 and at the end."""
    n = (1 << 32) + 100_003
    pats = gen.random_patterns(300, 1000, 20, 20)
    text = gen.plant(gen.iid_text(300, 0, n), 0, n, pats, 300)
    a = P.Automaton(pats)
    dtext = to_dev(text)
    epos, epid = _oracle_list_parallel(pats, text)
    assert len(epos) > 1_000_000 and int(epos[-1]) > (1 << 32)
    o = Oracle(pats)
    for mode in (1, 0, 3):
        a.set_text_kernel(mode)
        out = torch.empty(n, dtype=torch.int32, device=DEV)
        cap = len(epos) + 1024
        pos = torch.full((cap,), -1, dtype=torch.int64, device=DEV)
        pid = torch.empty(cap, dtype=torch.int32, device=DEV)
        cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
        ws = torch.empty(P.match_text_workspace_bytes(n, n), dtype=torch.uint8, device=DEV)
        P.match_text_async(a, dtext, n, n, out, pos, pid, cnt, ws, pos_base=3)
        torch.cuda.synchronize()
        assert int(cnt.item()) == len(epos)
        assert (pos[:len(epos)].cpu().numpy() == epos.astype(np.int64) + 3).all()
        assert (pid[:len(epos)].cpu().numpy() == epid).all()
        for s in [(1 << 32) - 50_000, n - 60_001]:
            assert (out[s:s + 60_000].cpu().numpy() == o.match(text, s, s + 60_000)).all()
        del out, ws
    a.set_text_kernel(-1)
