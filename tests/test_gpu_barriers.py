"""GPU parity for barrier semantics (-m gpu): text bytes outside ACGTacgt stop every walk.

DESIGN.md reading R5 (SPEC.md:143, :196 with PAPER.md:91): a byte outside ACGTacgt has no
transition, so out[i] = 0 where byte i is such a byte and no reported occurrence contains one.  The
oracle implements this directly (oracle/pfac_oracle.c, `col < 0` ends the walk); the CUDA path packs
a per-word barrier mask and runs the BAR instantiation of the match kernel.  Bar: bit-exact.
"""
import numpy as np
import pytest

import pfac_datagen as gen
from oracle import Oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1811_10498_b200 as P  # noqa: E402
from paper_1811_10498_b200 import binding as B  # noqa: E402

DEV = torch.device("cuda:0")
ACGT8 = np.frombuffer(b"ACGTacgt", np.uint8)


def to_dev(t: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(t)).to(DEV)


def barrier_bits(text: np.ndarray) -> np.ndarray:
    """Test-side definition of the barrier mask (include/pfac.h): bit j of word w = byte 16w+j invalid."""
    n = len(text)
    words = B.inv_words(n)
    bad = np.zeros(words * 16, dtype=np.uint32)
    bad[:n] = ~np.isin(text, ACGT8)
    bad = bad.reshape(-1, 16)
    return (bad << np.arange(16, dtype=np.uint32)).sum(axis=1).astype(np.uint16)


def first_bad(text: np.ndarray) -> int:
    idx = np.nonzero(~np.isin(text, ACGT8))[0]
    return int(idx[0]) if len(idx) else -1


# --------------------------------------------------------------------------- pack
@pytest.mark.parametrize("n", [1, 15, 16, 17, 100, 4099, 100_003])
def test_pack_barriers_definition(n):
    text = gen.add_barriers(gen.iid_text(n, 0, n), n, line=7, block=64, run_max=5, run_frac=0.5)
    packed, inv = P.pack_barriers_async(to_dev(text), first_bad=(bad := torch.zeros(1, dtype=torch.int64,
                                                                                      device=DEV)))
    torch.cuda.synchronize()
    assert (inv.cpu().numpy().view(np.uint16) == barrier_bits(text)).all()
    assert int(bad.item()) == first_bad(text)
    # codes of valid bytes are as pfac_pack_async writes them
    plain = P.pack_async(to_dev(text))
    torch.cuda.synchronize()
    assert (packed.cpu().numpy() == plain.cpu().numpy()).all()


# --------------------------------------------------------------------------- match (sync entry point)
PATTERN_SETS = {
    "short": lambda: gen.random_patterns(70, 80, 1, 9),
    "mixed": lambda: gen.random_patterns(71, 300, 4, 30) + [b"ACGTACGTACGTACGTACGTAC"],
    "long": lambda: gen.random_patterns(72, 500, 20, 100),
    "kmers2": lambda: gen.all_kmers(2),
    "kmers10": lambda: gen.all_kmers(10),
    "large": lambda: gen.random_patterns(73, 20_000, 16, 64),
}


@pytest.mark.parametrize("pset", list(PATTERN_SETS))
@pytest.mark.parametrize("layout", ["fasta", "gaps", "dense"])
def test_match_barriers_vs_oracle(pset, layout):
    pats = PATTERN_SETS[pset]()
    n = 300_017
    text = gen.plant(gen.iid_text(74, 0, n), 0, n, pats, 74)
    if layout == "fasta":
        gen.add_barriers(text, 74, line=60)
    elif layout == "gaps":
        gen.add_barriers(text, 75, line=0, block=2048, run_max=3000, run_frac=0.4)
    else:  # a barrier every few bases: every 10-mer window of the filter sees one
        gen.add_barriers(text, 76, line=5, block=32, run_max=3, run_frac=0.5)
    got = P.match(P.Automaton(pats), to_dev(text)).cpu().numpy()
    exp = Oracle(pats).match(text)
    assert (got == exp).all(), np.nonzero(got != exp)[0][:10]
    assert (got[~np.isin(text, ACGT8)] == 0).all()


@pytest.mark.parametrize("n", [1, 2, 17, 511, 2048, 2049, 8193, 148 * 2048 + 5])
def test_match_barriers_edges(n):
    pats = gen.random_patterns(77, 200, 1, 24)
    text = gen.plant(gen.iid_text(77, 0, n), 0, n, pats, 77)
    for w in (0, n // 2, n - 1):
        text[w] = ord("N")
    got = P.match(P.Automaton(pats), to_dev(text)).cpu().numpy()
    assert (got == Oracle(pats).match(text)).all()


def test_match_all_barriers_and_lowercase():
    pats = gen.random_patterns(78, 50, 3, 12)
    a = P.Automaton(pats)
    text = np.full(10_000, ord("N"), np.uint8)
    assert (P.match(a, to_dev(text)).cpu().numpy() == 0).all()
    # lower case is not a barrier
    text = gen.plant(gen.iid_text(78, 0, 50_000), 0, 50_000, pats, 78)
    low = text.copy()
    low[::3] += 32  # ACGT -> acgt
    low[1000:1100] = ord("n")
    exp = Oracle(pats).match(low)
    assert (P.match(a, to_dev(low)).cpu().numpy() == exp).all()


def test_hand_outputs_with_barriers(golden):
    for case in golden("hand_outputs.json")["cases"]:
        t = case["text"].encode()
        if not t:
            continue
        got = P.match(P.Automaton([p.encode() for p in case["patterns"]]), to_dev(np.frombuffer(t, np.uint8)))
        assert got.cpu().numpy().tolist() == case["out"], case


# --------------------------------------------------------------------------- packed-level + shard windows
@pytest.mark.parametrize("n_own,n_avail", [(100_000, 100_000), (100_000, 100_050), (65_536, 70_000)])
def test_match_barriers_window(n_own, n_avail):
    pats = gen.random_patterns(79, 400, 8, 40)
    text = gen.plant(gen.iid_text(79, 0, n_avail), 0, n_avail, pats, 79)
    gen.add_barriers(text, 79, line=70)
    if n_avail > n_own:
        text[n_own + 3] = ord("N")  # a barrier inside the halo
    packed, inv = P.pack_barriers_async(to_dev(text))
    out = P.match_barriers_async(P.Automaton(pats), packed, inv, n_own, n_avail)
    torch.cuda.synchronize()
    exp = Oracle(pats).match(text)[:n_own]
    assert (out.cpu().numpy() == exp).all()


def test_match_barriers_no_barrier_equals_plain():
    pats = gen.random_patterns(80, 1000, 20, 20)
    n = 1 << 20
    text = gen.plant(gen.iid_text(80, 0, n), 0, n, pats, 80)
    a = P.Automaton(pats)
    packed, inv = P.pack_barriers_async(to_dev(text))
    o1 = P.match_barriers_async(a, packed, inv, n)
    o2 = P.match_packed_async(a, packed, n)
    torch.cuda.synchronize()
    assert (o1 == o2).all()


# --------------------------------------------------------------------------- fused match + compact
@pytest.mark.parametrize("pset", ["mixed", "kmers2", "large"])
def test_fused_barriers_vs_oracle(pset):
    pats = PATTERN_SETS[pset]()
    n = 500_003
    text = gen.plant(gen.iid_text(81, 0, n), 0, n, pats, 81)
    gen.add_barriers(text, 81, line=80)
    a = P.Automaton(pats)
    packed, inv = P.pack_barriers_async(to_dev(text))
    cap = n
    out = torch.empty(n, dtype=torch.int32, device=DEV)
    pos = torch.empty(cap, dtype=torch.int64, device=DEV)
    pid = torch.empty(cap, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(P.compact_workspace_bytes(n), dtype=torch.uint8, device=DEV)
    P.match_compact_async(a, packed, n, n, out, pos, pid, cnt, ws, pos_base=11, inv=inv)
    torch.cuda.synchronize()
    m = int(cnt.item())
    epos, epid = Oracle(pats).match_list(text, 0, n)
    assert m == len(epos)
    assert (pos[:m].cpu().numpy() == epos.astype(np.int64) + 11).all()
    assert (pid[:m].cpu().numpy() == epid).all()
    assert (out.cpu().numpy() == Oracle(pats).match(text)).all()


# --------------------------------------------------------------------------- end to end over host memory
@pytest.mark.parametrize("n", [1000, (1 << 26) + 4321])
def test_scan_host_barriers(n):
    pats = gen.random_patterns(82, 300, 12, 40)
    text = gen.plant(gen.iid_text(82, 0, n), 0, n, pats, 82)
    gen.add_barriers(text, 82, line=0, block=1 << 16, run_max=200, run_frac=0.3)
    text[n // 3] = ord("\n")
    pos, pid, m = P.scan_host(P.Automaton(pats), torch.from_numpy(text))
    o = Oracle(pats)
    if n <= 1 << 20:
        epos, epid = o.match_list(text, 0, n)
    else:
        parts = [o.match_list(text, s, min(n, s + (1 << 22)), n=n) for s in range(0, n, 1 << 22)]
        epos = np.concatenate([p[0] for p in parts])
        epid = np.concatenate([p[1] for p in parts])
    assert m == len(epos)
    assert (pos.numpy() == epos.astype(np.int64)).all() and (pid.numpy() == epid).all()
