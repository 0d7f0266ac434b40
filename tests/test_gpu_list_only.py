"""GPU parity (-m gpu) for the list-only match (pfac_match_list_async) and
for the fused kernel's spilled-bitmap fallback (dense outputs).

The list-only call never writes the dense out[]; its list must equal the oracle's match list
(Oracle.match_list) exactly, including the per-pattern histogram and the capacity semantics.
Full-size configs are compared in test_gpu_parity.py::_full_config.
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


def to_dev(t: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(t)).to(DEV)


def run_list(a, text, n_own=None, pos_base=0, cap=None, hist=None, barriers=False):
    n = len(text)
    n_own = n if n_own is None else n_own
    d = to_dev(text)
    if barriers:
        packed, inv = P.pack_barriers_async(d)
    else:
        packed, inv = P.pack_async(d), None
    cap = n_own + 1 if cap is None else cap
    pos = torch.full((max(cap, 1),), -1, dtype=torch.int64, device=DEV)
    pid = torch.full((max(cap, 1),), -1, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.full((P.match_list_workspace_bytes(n_own),), 0x5A, dtype=torch.uint8, device=DEV)  # dirty
    P.match_list_async(a, packed, n_own, n, pos[:cap], pid[:cap], cnt, ws, pos_base=pos_base, hist=hist, inv=inv)
    torch.cuda.synchronize()
    m = int(cnt.item())
    return pos[:min(m, cap)].cpu().numpy(), pid[:min(m, cap)].cpu().numpy(), m


SETS = {
    "cfg2like": lambda: gen.random_patterns(100, 1000, 20, 20),
    "short": lambda: gen.random_patterns(101, 100, 1, 9),
    "mixed": lambda: gen.random_patterns(102, 3000, 6, 40),
    "kmers2": lambda: gen.all_kmers(2),        # every position matches: staging spills
    "kmers6": lambda: gen.all_kmers(6),
    "nested": lambda: gen.repetitive_patterns(5),
}


@pytest.mark.parametrize("pset", list(SETS))
@pytest.mark.parametrize("n", [1, 4097, 1_000_003])
def test_list_only_vs_oracle(pset, n):
    pats = SETS[pset]()
    text = gen.repetitive_text(5, n) if pset == "nested" else gen.plant(gen.iid_text(103, 0, n), 0, n, pats, 103)
    a = P.Automaton(pats)
    pos, pid, m = run_list(a, text, pos_base=17)
    epos, epid = Oracle(pats).match_list(text)
    assert m == len(epos)
    assert (pos == epos.astype(np.int64) + 17).all() and (pid == epid.astype(np.int32)).all()


def test_list_only_window_barriers_hist_capacity():
    pats = SETS["mixed"]()
    n = 700_001
    text = gen.plant(gen.iid_text(104, 0, n), 0, n, pats, 104)
    gen.add_barriers(text, 104, line=70)
    a = P.Automaton(pats)
    n_own = 650_000
    hist = torch.zeros(len(pats) + 1, dtype=torch.int64, device=DEV)
    pos, pid, m = run_list(a, text, n_own=n_own, hist=hist, barriers=True)
    epos, epid = Oracle(pats).match_list(text, 0, n_own, n=n)
    assert m == len(epos) and (pos == epos.astype(np.int64)).all() and (pid == epid.astype(np.int32)).all()
    assert (hist.cpu().numpy() == np.bincount(epid, minlength=len(pats) + 1)).all()
    pos, pid, m = run_list(a, text, n_own=n_own, cap=100, barriers=True)
    assert m == len(epos) and (pos == epos[:100].astype(np.int64)).all()


def test_fused_spill_dense_cfg5_prefix():
    """Dense matches (cfg5's nested families on its repetitive text): the fused kernel's staging spills
    to slice bitmaps; its list and out[] must still equal the oracle's."""
    cfg = gen.CONFIGS[5]
    pats = gen.config_patterns(cfg)
    n = 32_000_000
    text = gen.config_text(cfg, 0, n, patterns=pats, n=n)
    a = P.Automaton(pats)
    packed = P.pack_async(to_dev(text))
    out = torch.empty(n, dtype=torch.int32, device=DEV)
    epos, epid = Oracle(pats).match_list(text)
    cap = len(epos) + 16
    pos = torch.empty(cap, dtype=torch.int64, device=DEV)
    pid = torch.empty(cap, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(P.compact_workspace_bytes(n), dtype=torch.uint8, device=DEV)
    P.match_compact_async(a, packed, n, n, out, pos, pid, cnt, ws)
    torch.cuda.synchronize()
    assert int(cnt.item()) == len(epos) > 3_000_000  # well past the 2.8 M staging entries
    assert (pos[:len(epos)].cpu().numpy() == epos.astype(np.int64)).all()
    assert (pid[:len(epos)].cpu().numpy() == epid.astype(np.int32)).all()
    pos2, pid2, m = run_list(a, text, cap=cap)
    assert m == len(epos) and (pos2 == epos.astype(np.int64)).all() and (pid2 == epid.astype(np.int32)).all()
