"""GPU parity (-m gpu) for the all-occurrence expansion (pfac_expand).

The CUDA path (fused match + compact, then expand, all through the C-ABI) against the oracle's
Oracle.match_all, which emits every final state each walk passes (pinned in test_oracle_pins.py to
the classic failure-link machine and to brute force).  Bar: bit-exact lists, same order.
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


def to_dev(t: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(t)).to(DEV)


def gpu_list(a, text: np.ndarray, inv=False):
    """pack -> fused match+compact on the device; returns device (pos, pid, count tensor)."""
    n = len(text)
    d = to_dev(text)
    if inv:
        packed, iv = P.pack_barriers_async(d)
    else:
        packed, iv = P.pack_async(d), None
    out = torch.empty(n, dtype=torch.int32, device=DEV)
    pos = torch.empty(n + 1, dtype=torch.int64, device=DEV)
    pid = torch.empty(n + 1, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(P.compact_workspace_bytes(n), dtype=torch.uint8, device=DEV)
    P.match_compact_async(a, packed, n, n, out, pos, pid, cnt, ws, inv=iv)
    return pos, pid, cnt


def gpu_all(a, pos, pid, cnt, cap):
    pa = torch.empty(max(cap, 1), dtype=torch.int64, device=DEV)
    pi = torch.empty(max(cap, 1), dtype=torch.int32, device=DEV)
    ca = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(P.expand_workspace_bytes(), dtype=torch.uint8, device=DEV)
    P.expand_async(a, pos, pid, cnt, pa[:cap], pi[:cap], ca, ws)
    torch.cuda.synchronize()
    t = int(ca.item())
    return pa[:min(t, cap)].cpu().numpy(), pi[:min(t, cap)].cpu().numpy(), t


PATTERN_SETS = {
    "kmers1to4": lambda: gen.all_kmers(1) + gen.all_kmers(2) + gen.all_kmers(3) + gen.all_kmers(4),
    "nested": lambda: gen.repetitive_patterns(5),
    "random": lambda: gen.random_patterns(90, 500, 4, 30),
    "mixed": lambda: gen.random_patterns(91, 200, 8, 12) + [b"ACGT" * k for k in range(1, 8)],
}


@pytest.mark.parametrize("pset", list(PATTERN_SETS))
@pytest.mark.parametrize("n", [1, 777, 100_003])
def test_expand_vs_oracle(pset, n):
    pats = PATTERN_SETS[pset]()
    if pset == "nested":
        text = gen.repetitive_text(5, n)
    else:
        text = gen.plant(gen.iid_text(92, 0, n), 0, n, pats, 92)
    a = P.Automaton(pats)
    pos, pid, cnt = gpu_list(a, text)
    epos, epid = Oracle(pats).match_all(text)
    gp, gi, t = gpu_all(a, pos, pid, cnt, len(epos) + 64)
    assert t == len(epos)
    assert (gp == epos.astype(np.int64)).all() and (gi == epid.astype(np.int32)).all()


def test_expand_with_barriers():
    pats = PATTERN_SETS["mixed"]()
    n = 200_000
    text = gen.plant(gen.iid_text(93, 0, n), 0, n, pats, 93)
    gen.add_barriers(text, 93, line=61)
    a = P.Automaton(pats)
    pos, pid, cnt = gpu_list(a, text, inv=True)
    epos, epid = Oracle(pats).match_all(text)
    gp, gi, t = gpu_all(a, pos, pid, cnt, len(epos) + 1)
    assert t == len(epos) and (gp == epos.astype(np.int64)).all() and (gi == epid.astype(np.int32)).all()


def test_expand_capacity_and_truncated_input():
    pats = PATTERN_SETS["kmers1to4"]()
    n = 50_000
    text = gen.iid_text(94, 0, n)
    a = P.Automaton(pats)
    pos, pid, cnt = gpu_list(a, text)
    epos, epid = Oracle(pats).match_all(text)
    # capacity below the total: exact total, the first `cap` entries
    gp, gi, t = gpu_all(a, pos, pid, cnt, 1000)
    assert t == len(epos) and (gp == epos[:1000].astype(np.int64)).all() and (gi == epid[:1000]).all()
    # input capacity below the input count: only the first in_capacity entries are expanded
    m_in = 5000
    gp, gi, t = gpu_all(a, pos[:m_in], pid[:m_in], cnt, len(epos))
    lpos, _ = Oracle(pats).match_list(text)
    last = int(lpos[m_in - 1])
    keep = epos <= last
    assert t == int(keep.sum()) and (gp == epos[keep].astype(np.int64)).all()


def test_expand_empty_and_sync_api():
    pats = PATTERN_SETS["random"]()
    a = P.Automaton(pats)
    e = torch.zeros(0, dtype=torch.int64, device=DEV)
    ei = torch.zeros(0, dtype=torch.int32, device=DEV)
    pa, pi, t = P.expand(a, e, ei)
    assert t == 0 and pa.numel() == 0
    n = 300_000
    text = gen.plant(gen.iid_text(95, 0, n), 0, n, pats, 95)
    lpos, lpid, m = P.compact(P.match(a, to_dev(text)))
    pa, pi, t = P.expand(a, lpos, lpid, capacity=None)
    epos, epid = Oracle(pats).match_all(text)
    assert t == len(epos) and (pa.cpu().numpy() == epos.astype(np.int64)).all()
    assert (pi.cpu().numpy() == epid.astype(np.int32)).all()
    with pytest.raises(B.PfacError) as ex:
        P.expand(a, lpos, lpid, capacity=3)
    assert ex.value.code == B.E_CAPACITY


def test_expand_cfg5_prefix():
    """cfg5's nested families on a 4 Mbase prefix of its repetitive text: long prefix chains."""
    cfg = gen.CONFIGS[5]
    pats = gen.config_patterns(cfg)
    n = 4_000_000
    text = gen.config_text(cfg, 0, n, patterns=pats, n=n)
    a = P.Automaton(pats)
    pos, pid, cnt = gpu_list(a, text)
    epos, epid = Oracle(pats).match_all(text)
    gp, gi, t = gpu_all(a, pos, pid, cnt, len(epos))
    assert t == len(epos) and (gp == epos.astype(np.int64)).all() and (gi == epid.astype(np.int32)).all()
    assert t > 10 * int(cnt.item())  # chains are long on this workload
