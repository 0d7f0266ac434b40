"""GPU parity (-m gpu) for the text-input kernel (pfac_match_text_async): pack fused into the
fused match + compact kernel, reading the ASCII text directly.

Its results must equal the oracle's exactly (PAPER.md:91 longest-only output, reading R5 barriers):
the dense out[] element by element, the ordered (position, id) list, the count, the per-pattern
histogram and the first owned non-ACGT index.  Also covered: list-only mode (no out[]), shard
windows (n_own < n_avail, pos_base), texts whose length is not a multiple of 16 (the kernel's lane
tail reads), an unaligned text pointer and a halo too long for the one-kernel plan (both take the
two-kernel path inside the call), and capacity overflow.
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

DEV = torch.device("cuda:0")
ACGT8 = np.frombuffer(b"ACGTacgt", np.uint8)
U64MAX = (1 << 64) - 1


@pytest.fixture(autouse=True, params=["1", "0", "2", "3"], ids=["one-kernel", "two-kernel", "one-kernel-1k",
                                                              "one-kernel-1k-dyn"])
def text_kernel(request, monkeypatch):
    """Both paths of pfac_match_text_async: the one-kernel TXT instantiation and the pack + fused
    kernel path the call takes for unaligned text or automata the policy keeps off TXT; "2": the text
    kernel with 1024-position slices (both cell widths); "3": that kernel with dynamically claimed slices."""
    monkeypatch.setattr(P.binding, "DEFAULT_TEXT_KERNEL", int(request.param))
    return request.param


def first_bad(text: np.ndarray, n_own: int) -> int:
    idx = np.nonzero(~np.isin(text[:n_own], ACGT8))[0]
    return int(idx[0]) if len(idx) else -1


def run_text(a, text, n_own=None, pos_base=0, cap=None, dense=True, hist=None, offset=0):
    """pfac_match_text_async on `text` (copied to the device at byte `offset` of its buffer)."""
    n = len(text)
    n_own = n if n_own is None else n_own
    buf = torch.zeros(n + offset + 16, dtype=torch.uint8, device=DEV)
    d = buf[offset:offset + n]
    d.copy_(torch.from_numpy(np.ascontiguousarray(text)))
    cap = n_own + 1 if cap is None else cap
    out = torch.full((max(n_own, 1),), -7, dtype=torch.int32, device=DEV) if dense else None
    pos = torch.full((max(cap, 1),), -1, dtype=torch.int64, device=DEV)
    pid = torch.full((max(cap, 1),), -1, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    bad = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.full((P.match_text_workspace_bytes(n_own, n, not dense),), 0x5A, dtype=torch.uint8, device=DEV)
    P.match_text_async(a, d, n_own, n, out[:n_own] if dense else None, pos[:cap], pid[:cap], cnt, ws,
                       pos_base=pos_base, hist=hist, first_bad=bad)
    torch.cuda.synchronize()
    m = int(cnt.item())
    fb = int(bad.item())
    return (out[:n_own].cpu().numpy() if dense else None, pos[:min(m, cap)].cpu().numpy(),
            pid[:min(m, cap)].cpu().numpy(), m, fb)


def check(pats, text, n_own=None, pos_base=0, dense=True, offset=0):
    n = len(text)
    n_own = n if n_own is None else n_own
    a = P.Automaton(pats)
    out, pos, pid, m, fb = run_text(a, text, n_own=n_own, pos_base=pos_base, dense=dense, offset=offset)
    o = Oracle(pats)
    if dense:
        exp = o.match(text, 0, n_own, n=n)
        bad = np.nonzero(out != exp)[0]
        assert len(bad) == 0, f"{len(bad)} mismatches, first at {bad[:5]}: got {out[bad[:5]]} want {exp[bad[:5]]}"
    epos, epid = o.match_list(text, 0, n_own, n=n)
    assert m == len(epos)
    assert (pos == epos.astype(np.int64) + pos_base).all() and (pid == epid.astype(np.int32)).all()
    fbe = first_bad(text, n_own)
    assert fb == (-1 if fbe < 0 else fbe + pos_base)  # int64 view of UINT64_MAX is -1
    return m


SETS = {
    "cfg2like": lambda: gen.random_patterns(200, 1000, 20, 20),
    "short": lambda: gen.random_patterns(201, 100, 1, 9),
    "mixed": lambda: gen.random_patterns(202, 3000, 6, 40),
    "big32": lambda: gen.random_patterns(203, 40000, 12, 40),   # uint32 image
    "kmers2": lambda: gen.all_kmers(2),                          # every position matches
    "kmers6": lambda: gen.all_kmers(6),
    "nested": lambda: gen.repetitive_patterns(5),
}


def make_text(pset, pats, n, seed):
    if pset == "nested":
        return gen.repetitive_text(seed, n)
    return gen.plant(gen.iid_text(seed, 0, n), 0, n, pats, seed)


@pytest.mark.parametrize("pset", list(SETS))
@pytest.mark.parametrize("n", [1, 15, 16, 17, 2047, 2048, 2049, 4097, 300_001, 1_000_003])
def test_text_vs_oracle(pset, n):
    pats = SETS[pset]()
    check(pats, make_text(pset, pats, n, 210 + n % 97), pos_base=5)


@pytest.mark.parametrize("pset", ["cfg2like", "short", "mixed", "big32", "nested"])
@pytest.mark.parametrize("layout", ["fasta", "gaps", "dense"])
def test_text_barriers(pset, layout):
    pats = SETS[pset]()
    n = 600_011
    text = make_text(pset, pats, n, 220)
    if layout == "fasta":
        gen.add_barriers(text, 221, line=80, block=100_000, run_max=5000, run_frac=0.3)
    elif layout == "gaps":
        gen.add_barriers(text, 222, line=0, block=20_000, run_max=3000, run_frac=0.5)
    else:
        gen.add_barriers(text, 223, line=5, block=64, run_max=4, run_frac=0.5)
    check(pats, text)
    check(pats, text, dense=False)


@pytest.mark.parametrize("pset", ["cfg2like", "mixed", "big32"])
def test_text_shard_windows(pset):
    pats = SETS[pset]()
    n = 500_000
    text = make_text(pset, pats, n, 230)
    for n_own in [1, 2048, 131_072, 499_937]:
        check(pats, text[:min(n, n_own + 63)], n_own=n_own, pos_base=1 << 33)
    # a barrier inside the halo only: first_bad must not report it, the walks must stop at it
    t2 = text[:140_000].copy()
    t2[131_080] = ord("N")
    check(pats, t2, n_own=131_072, pos_base=9)


def test_text_lowercase_and_all_n():
    pats = SETS["mixed"]()
    n = 200_003
    text = make_text("mixed", pats, n, 240)
    low = text.copy()
    low[::3] |= 0x20  # ACGT -> acgt (FASTA soft-masking, reading R4)
    check(pats, low)
    check(pats, np.full(70_001, ord("N"), np.uint8))


@pytest.mark.parametrize("offset", [1, 3, 8])
def test_text_unaligned_pointer(offset):
    pats = SETS["cfg2like"]()
    text = make_text("cfg2like", pats, 300_007, 250)
    gen.add_barriers(text, 251, line=61, block=4096, run_max=50, run_frac=0.3)
    check(pats, text, offset=offset)
    check(pats, text, offset=offset, dense=False)


def test_text_long_halo_fallback():
    """max_len 600: the one-kernel plan does not fit; the call runs pack + fused match itself."""
    pats = gen.random_patterns(260, 200, 20, 600)
    n = 400_003
    text = make_text("long", pats, n, 261)
    gen.add_barriers(text, 262, line=0, block=50_000, run_max=10, run_frac=0.5)
    check(pats, text, n_own=300_000)
    check(pats, text, dense=False)


def test_text_hist_capacity():
    pats = SETS["kmers6"]()
    n = 100_000
    text = make_text("kmers6", pats, n, 270)
    a = P.Automaton(pats)
    hist = torch.zeros(len(pats) + 1, dtype=torch.int64, device=DEV)
    out, pos, pid, m, fb = run_text(a, text, hist=hist)
    exp = Oracle(pats).match(text)
    assert (out == exp).all() and m == int((exp != 0).sum()) and fb == -1
    h = hist.cpu().numpy()
    assert (h[1:] == np.bincount(exp[exp != 0], minlength=len(pats) + 1)[1:]).all()
    # capacity overflow: the count is the total, the first `cap` entries are the list's prefix
    cap = 1000
    _, pos2, pid2, m2, _ = run_text(a, text, cap=cap, dense=False)
    epos, epid = Oracle(pats).match_list(text)
    assert m2 == len(epos) and len(pos2) == cap
    assert (pos2 == epos[:cap].astype(np.int64)).all() and (pid2 == epid[:cap].astype(np.int32)).all()


def test_text_policy_info(text_kernel):
    """The image reports which path the call takes (pfac_image_info.text_kernel)."""
    a = P.Automaton(SETS["cfg2like"]())
    info = a.image_info(0)
    assert info["text_kernel"] == {"1": 1, "0": 0, "2": 2, "3": 3}[text_kernel]  # uint16 image
    b = P.Automaton(SETS["big32"]())  # uint32 image
    assert b.image_info(0)["text_kernel"] == {"1": 1, "0": 0, "2": 2, "3": 3}[text_kernel]
    b.set_text_kernel(-1)  # back to the plan: a uint32 image with < 2^20 rows takes 2048-slice text
    assert b.image_info(0)["text_kernel"] in (1, 2)


def test_text_empty():
    a = P.Automaton(SETS["cfg2like"]())
    out, pos, pid, m, fb = run_text(a, np.zeros(0, np.uint8))
    assert m == 0 and fb == -1


def _prefixed_kmers(k: int, first: str) -> list[bytes]:
    """All k-mers whose first base is in `first`: a share len(first)/4 of random-text positions match."""
    return [p for p in gen.all_kmers(k) if chr(p[0]) in first]


@pytest.mark.parametrize("width", ["u16", "u32"])
@pytest.mark.parametrize("first", ["A", "AC"])
@pytest.mark.parametrize("dense", [True, False], ids=["dense", "list"])
def test_text_match_log(width, first, dense):
    """Match densities of 25% / 50% over 24 Mbases: each warp's staging overflows after one slice, so
    the next slices go through the per-warp match log (bitmap + pids, 2-byte pids when every id fits
    in 16 bits, else 4-byte) and, where a slice's record no longer fits the log (50%, and 25% with
    4-byte pids), the out[] re-read.  Lists and out[] must equal the oracle's (the list is in
    position order across staged, logged and spilled slices)."""
    pats = _prefixed_kmers(4 if width == "u16" else 9, first)
    assert (len(pats) < 65536) == (width == "u16")
    n = 24_000_000
    text = gen.iid_text(300 + len(first), 0, n)
    m = check(pats, text, dense=dense)
    assert abs(m / n - 0.25 * len(first)) < 0.01


@pytest.mark.parametrize("cut", range(-2, 8))
def test_text_chain_heads_near_the_end(cut):
    """uint32 images whose J2 entries carry a chain head's first 4 forced bases (the NB form): walks
    that reach depth K2 with 0-3 bases left (the answer is 0 without the head's row), with exactly the
    4 bases (row loaded), with a mismatch inside the first 4 (answer 0) and beyond them, and planted
    complete patterns -- at the very end of the text and in its middle."""
    pats = gen.random_patterns(204, 40_000, 24, 40)
    a = P.Automaton(pats)
    info = a.image_info(0)
    assert info["cell_bytes"] == 4 and info["hr_nb_rows"] > 1000, info
    K2 = info["K2"]
    rng = np.random.default_rng(cut + 10)
    pieces = []
    for j in range(200):
        p = np.frombuffer(pats[j], np.uint8).copy()
        c = min(len(p), K2 + cut)
        q = p[:c].copy()
        if j % 3 == 1 and c > K2:  # a mismatch among the bases after depth K2
            t = K2 + (j // 3) % (c - K2)
            q[t] = b"ACGT"[(b"ACGT".index(q[t]) + 1) % 4]
        pieces.append(gen.iid_text(1000 + j, 0, int(rng.integers(0, 40))))
        pieces.append(q)
    pieces.append(np.frombuffer(pats[7][:K2 + cut] if K2 + cut > 0 else b"", np.uint8))  # at the very end
    text = np.concatenate(pieces)
    check(pats, text)
    check(pats, text, dense=False)
