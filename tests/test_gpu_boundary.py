"""GPU parity (-m gpu) of the SURVEY.md §8(b) boundary calls in their specified, synchronous form:

  pfac_pack(d_text, n, d_packed, first_bad, stream)            -> packed codes + first non-ACGT index
  pfac_match(a, d_text, n, d_out, stream)                      -> out[i]
  pfac_match_packed(a, d_packed, n_own, n_avail, d_out, stream) -> shard form (reading R6)
  pfac_match_checked(...)                                       -> pfac_match + first barrier index

each called through ctypes on device buffers and compared with the oracle (or, for pack, with the
packing definition of include/pfac.h) element by element.  Also: the current device is restored,
and pfac_scan_host's dense-chunk regrow path (a chunk whose list exceeds the slot's capacity) gives
the closed-form list of the all-1-mer automaton.
"""
import ctypes

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
U64MAX = (1 << 64) - 1


def to_dev(t: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(t)).to(DEV)


def np_pack(text: np.ndarray) -> np.ndarray:
    """Packing definition (include/pfac.h): A0 C1 G2 T3, base j at bits 2(j mod 16) of word j/16."""
    lut = np.zeros(256, dtype=np.uint32)
    for ch, c in zip(b"ACGTacgt", [0, 1, 2, 3, 0, 1, 2, 3]):
        lut[ch] = c
    words = B.packed_words(len(text))
    codes = np.zeros(words * 16, dtype=np.uint32)
    codes[:len(text)] = lut[text]
    codes = codes.reshape(-1, 16)
    return (codes << (2 * np.arange(16, dtype=np.uint32))).sum(axis=1, dtype=np.uint64).astype(np.uint32)


def stream_ptr():
    return torch.cuda.current_stream(DEV).cuda_stream


@pytest.mark.parametrize("n", [0, 1, 17, 4099, 300_001])
def test_pfac_pack_sync(n):
    text = np.frombuffer(b"ACGTacgt", np.uint8)[np.random.default_rng(n).integers(0, 8, n)]
    d = to_dev(text) if n else torch.zeros(1, dtype=torch.uint8, device=DEV)
    packed = torch.full((B.packed_words(n),), -1, dtype=torch.int32, device=DEV)
    bad = ctypes.c_uint64(7)
    rc = B.lib().pfac_pack(d.data_ptr(), n, packed.data_ptr(), ctypes.byref(bad), stream_ptr())
    assert rc == B.OK and bad.value == U64MAX
    # returns after completion: no synchronize before reading
    if n:
        assert (packed.cpu().numpy().view(np.uint32) == np_pack(text)).all()


@pytest.mark.parametrize("where", [[0], [70, 5], [299_999]])
def test_pfac_pack_sync_non_acgt(where):
    text = gen.iid_text(3, 0, 300_000).copy()
    for w in where:
        text[w] = ord("N")
    d = to_dev(text)
    packed = torch.empty(B.packed_words(len(text)), dtype=torch.int32, device=DEV)
    bad = ctypes.c_uint64(0)
    rc = B.lib().pfac_pack(d.data_ptr(), len(text), packed.data_ptr(), ctypes.byref(bad), stream_ptr())
    assert rc == B.E_NON_ACGT and bad.value == min(where)
    assert b"not ACGT" in B.lib().pfac_last_error()
    # every other word is exact
    got, exp = packed.cpu().numpy().view(np.uint32), np_pack(text)
    bad_words = {w // 16 for w in where}
    keep = np.array([i not in bad_words for i in range(len(exp))])
    assert (got[keep] == exp[keep]).all()
    p2, fb = P.pack(d)
    assert fb == min(where)


SETS = {
    "cfg1": lambda: gen.config_patterns(gen.CONFIGS[1]),
    "cfg2like": lambda: gen.random_patterns(11, 1000, 20, 20),
    "big32": lambda: gen.random_patterns(12, 40_000, 12, 40),  # uint32 image with J2
    "kmers3": lambda: gen.all_kmers(3),
}


@pytest.mark.parametrize("name", list(SETS))
@pytest.mark.parametrize("n", [1, 2048 * 3 + 5, 1_000_003])
def test_pfac_match_sync(name, n):
    pats = SETS[name]()
    text = gen.plant(gen.iid_text(n % 97, 0, n), 0, n, pats, n % 97)
    a = P.Automaton(pats)
    d = to_dev(text)
    out = torch.full((n,), -7, dtype=torch.int32, device=DEV)
    rc = B.lib().pfac_match(a.handle, d.data_ptr(), n, out.data_ptr(), stream_ptr())
    assert rc == B.OK
    assert (out.cpu().numpy() == Oracle(pats).match(text)).all()


def test_pfac_match_checked_barriers():
    pats = SETS["cfg1"]()
    n = 500_000
    text = gen.plant(gen.iid_text(5, 0, n), 0, n, pats, 5).copy()
    gen.add_barriers(text, 5, line=80)
    a = P.Automaton(pats)
    out, fb = P.match_checked(a, to_dev(text))
    assert fb == int(np.nonzero(~np.isin(text, np.frombuffer(b"ACGTacgt", np.uint8)))[0][0])
    assert (out.cpu().numpy() == Oracle(pats).match(text)).all()
    out2 = P.match(a, to_dev(text))
    assert bool((out2 == out).all())


@pytest.mark.parametrize("name", ["cfg1", "big32"])
@pytest.mark.parametrize("n_own,n_avail", [(100_000, 100_000), (100_000, 100_039), (65_536 + 7, 90_000),
                                           (1, 64)])
def test_pfac_match_packed_sync(name, n_own, n_avail):
    pats = SETS[name]()
    text = gen.plant(gen.iid_text(9, 0, n_avail), 0, n_avail, pats, 9)
    a = P.Automaton(pats)
    packed, fb = P.pack(to_dev(text))
    assert fb == -1
    out = torch.full((n_own,), -7, dtype=torch.int32, device=DEV)
    rc = B.lib().pfac_match_packed(a.handle, packed.data_ptr(), n_own, n_avail, out.data_ptr(), stream_ptr())
    assert rc == B.OK
    assert (out.cpu().numpy() == Oracle(pats).match(text, 0, n_own, n=n_avail)).all()
    out2 = P.match_packed(a, packed, n_own, n_avail)
    assert bool((out2 == out).all())


def test_current_device_restored():
    """Every call leaves the calling thread's current device as it found it (pfac.h conventions):
    with buffers on device d and another device current, torch's cudaGetDevice is unchanged after
    the call (the static runtime in libpfac switches through the driver's per-thread context).
    Meaningful with >= 2 GPUs; with one it checks the call on the only device."""
    ndev = torch.cuda.device_count()
    pats = SETS["cfg1"]()
    a = P.Automaton(pats)
    text = gen.iid_text(1, 0, 10_000)
    exp = Oracle(pats).match(text)
    for dev in range(ndev):
        d = torch.from_numpy(text).to(f"cuda:{dev}")
        torch.cuda.set_device(ndev - 1 - dev)
        before = torch.cuda.current_device()
        out = P.match(a, d)
        assert torch.cuda.current_device() == before
        assert out.device.index == dev and (out.cpu().numpy() == exp).all()
    torch.cuda.set_device(0)


def test_scan_host_dense_chunk_regrow():
    """pfac_scan_host with a chunk whose list exceeds the slot's preallocated capacity (chunk/8 + 65536
    entries): the all-1-mer automaton matches every position, so the first 64-Mbase chunk's 2^26
    matches force the regrow-and-rerun path.  Closed form (all 4^k k-mers in lexicographic id
    order, k = 1): out[i] = 1 + code(text[i]), list = every position."""
    n = (1 << 26) + 3_000_001
    text = gen.iid_text(21, 0, n)
    a = P.Automaton([b"A", b"C", b"G", b"T"])
    pos, pid, m = P.scan_host(a, torch.from_numpy(text), pos_base=11)
    assert m == n
    assert (pos.numpy() == np.arange(n, dtype=np.int64) + 11).all()
    lut = np.zeros(256, np.int32)
    for ch, c in zip(b"ACGT", range(1, 5)):
        lut[ch] = c
    assert (pid.numpy() == lut[text]).all()
