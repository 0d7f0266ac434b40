"""Host builder through the C-ABI (no GPU needed): canonical export, invariants, parity with the
oracle's trie, error codes, and that libpfac exports every symbol include/pfac.h declares."""
import ctypes
import os
import random
import re

import numpy as np
import pytest

import pfac_datagen as gen
from oracle import Oracle
from paper_1811_10498_b200 import Automaton, PfacError, lib
from paper_1811_10498_b200 import binding as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def pats(*xs):
    return [x.encode() for x in xs]


def test_abi_exports_every_declared_symbol():
    src = open(os.path.join(ROOT, "include", "pfac.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(pfac_[a-z_]+)\s*\(", src))
    assert len(names) >= 14
    L = lib()
    for nm in sorted(names):
        assert hasattr(L, nm), nm
    assert set(B._SIGS) == names


def test_canonical_tables_hand_derived(golden):
    for case in golden("canonical_tables.json")["cases"]:
        a = Automaton(pats(*case["patterns"]))
        assert a.num_states == len(case["table"])
        assert a.table().tolist() == case["table"]
        assert a.num_patterns == len(case["patterns"])
        assert a.max_len == max(len(p) for p in case["patterns"])


def _paths(table):
    """state -> path string, by walking the exported table from the root."""
    paths = {0: ""}
    stack = [0]
    parents = {}
    while stack:
        u = stack.pop()
        for c in range(4):
            v = int(table[u][c])
            if v:
                assert v not in paths, "state with two parents"
                paths[v] = paths[u] + "ACGT"[c]
                parents[v] = u
                stack.append(v)
    return paths


def _oracle_paths(o: Oracle):
    t = o.table()
    paths, finals = {0: ""}, {}
    stack = [0]
    while stack:
        u = stack.pop()
        for c in range(4):
            nxt, pid = int(t[u, c, 0]), int(t[u, c, 1])
            if nxt:
                paths[nxt] = paths[u] + "ATCG"[c]
                if pid:
                    finals[pid] = paths[nxt]
                stack.append(nxt)
    return paths, finals


@pytest.mark.parametrize("seed", range(6))
def test_invariants_and_oracle_parity(seed):
    rng = random.Random(seed)
    P = list({("".join(rng.choice("ACGT") for _ in range(rng.randint(1, 12)))).encode()
              for _ in range(rng.randint(1, 200))})
    a = Automaton(P)
    T = a.table()
    S, k = a.num_states, len(P)
    paths = _paths(T)
    assert len(paths) == S  # every state reachable, exactly one parent each
    # ids 1..k are the finals, state p spells pattern p
    for p in range(1, k + 1):
        assert paths[p] == P[p - 1].decode()
    # non-finals k+1.. in BFS order: depth non-decreasing, lexicographic (A<C<G<T) within a depth
    rest = [paths[s] for s in range(k + 1, S)]
    keys = [(len(x), x) for x in rest]
    assert keys == sorted(keys)
    # same automaton as the oracle's insertion-order trie (numbering-independent)
    o = Oracle(P)
    opaths, ofinals = _oracle_paths(o)
    assert sorted(opaths.values()) == sorted(paths.values())
    assert {pid: s for pid, s in ofinals.items()} == {p: P[p - 1].decode() for p in range(1, k + 1)}
    assert S == o.num_states


def test_mixed_case_patterns():
    a = Automaton([b"acg", b"CT"])
    assert a.table().tolist()[0] == [3, 4, 0, 0]


def test_kmer_set_state_count():
    for k in (1, 2, 3, 4):
        a = Automaton(gen.all_kmers(k))
        assert a.num_states == (4 ** (k + 1) - 1) // 3


def test_build_errors():
    with pytest.raises(PfacError) as e:
        Automaton(pats("AC", ""))
    assert e.value.code == B.E_EMPTY and "id 2" in str(e.value)
    with pytest.raises(PfacError) as e:
        Automaton(pats("AC", "ANC"))
    assert e.value.code == B.E_NON_ACGT and "id 2" in str(e.value)
    with pytest.raises(PfacError) as e:
        Automaton(pats("ACG", "TT", "acg"))
    assert e.value.code == B.E_DUP and "id 3" in str(e.value) and "id 1" in str(e.value)
    with pytest.raises(PfacError) as e:
        Automaton([b"A" * (B.MAX_LEN + 1)])
    assert e.value.code == B.E_TOO_LONG
    Automaton([b"A" * B.MAX_LEN])  # the limit itself is fine


def test_empty_pattern_set():
    a = Automaton([])
    assert a.num_states == 1 and a.num_patterns == 0
    assert a.table().tolist() == [[0, 0, 0, 0]]


def test_null_arguments():
    L = lib()
    assert L.pfac_build(None, None, 3, ctypes.byref(ctypes.c_void_p())) == B.E_ARG
    assert L.pfac_build(None, None, 0, None) == B.E_ARG
    assert L.pfac_num_states(None) == 0
    assert L.pfac_prepare(None, 0) == B.E_ARG
    assert L.pfac_match_packed_async(None, None, 1, 1, None, None) == B.E_ARG
    assert L.pfac_compact(None, 5, 0, None, None, 0, None, 0, None, None) == B.E_ARG
    assert B.packed_words(0) == 0 and B.packed_words(1) == 4 and B.packed_words(64) == 4
    assert B.packed_words(65) == 8
    assert b"null" in L.pfac_last_error()


def test_large_config_builds():
    P = gen.config_patterns(gen.CONFIGS[2])
    a = Automaton(P)
    assert a.num_patterns == 1000 and a.max_len == 20
    assert 15000 < a.num_states < 17000  # SURVEY Appendix A estimate 15 818


def test_prefix_chain_definition():
    """pfac_prefix_chain: [p] = longest pattern that is a proper prefix of p, length = patterns that are
    prefixes of p (p included) -- by direct string comparison."""
    import random
    rng = random.Random(5)
    for trial in range(50):
        k = rng.randint(1, 60)
        pats = list({"".join(rng.choice("AC") for _ in range(rng.randint(1, 9))).encode() for _ in range(k)})
        ch = Automaton(pats).prefix_chain()
        assert ch[0].tolist() == [0, 0]
        for i, p in enumerate(pats, start=1):
            pre = [j for j, q in enumerate(pats, start=1) if len(q) < len(p) and p.startswith(q)]
            parent = max(pre, key=lambda j: len(pats[j - 1])) if pre else 0
            assert ch[i].tolist() == [parent, len(pre) + 1], (p, pats)


def test_text_walk_stats_closed_forms():
    """pfac_text_walk_stats (host code): transition counts of the PFAC walk from
    sampled positions, against closed forms.  All 4^3 3-mers: every walk makes min(3, n - i)
    transitions.  Nested family A^1..A^10 over A^25 C A^5 N A^4: min(10, run left) inside A runs,
    0 at C and at the N barrier (reading R5)."""
    rng = np.random.default_rng(5)
    a = Automaton(gen.all_kmers(3))
    n = 1000
    text = rng.choice(np.frombuffer(b"ACGT", np.uint8), n)
    steps = [min(3, n - i) for i in range(n)]
    for stride in (1, 7):
        s = steps[::stride]
        df, ms = a.text_walk_stats(text, stride=stride, deep=3)
        assert df == pytest.approx(sum(x >= 3 for x in s) / len(s)) and ms == pytest.approx(sum(s) / len(s))
    b = Automaton([b"A" * m for m in range(1, 11)])
    t = b"A" * 25 + b"C" + b"A" * 5 + b"N" + b"aaaa"  # lowercase: the same bases (reading R4)
    run_left = []
    for i, ch in enumerate(t):
        j = i
        while j < len(t) and t[j] in b"Aa":
            j += 1
        run_left.append(min(10, j - i))
    for deep in (1, 5, 10):
        df, ms = b.text_walk_stats(t, deep=deep)
        assert df == pytest.approx(sum(x >= deep for x in run_left) / len(t))
        assert ms == pytest.approx(sum(run_left) / len(t))
    assert b.text_walk_stats(b"", deep=4) == (0.0, 0.0)
    with pytest.raises(PfacError):
        b.text_walk_stats(t, stride=0)


def test_plan_text_policy():
    """pfac_plan_text: walk-heavy text (repetitive text against cfg5's nested families: ~20% of walks
    make >= 16 transitions) gets the 1024-position-slice text kernel with dynamically claimed slices
    (mode 3); random text keeps the plan."""
    cfg = gen.CONFIGS[5]
    p5 = gen.config_patterns(cfg)
    a = Automaton(p5)
    rep = gen.config_text(cfg, 0, 400_000, patterns=p5, n=cfg.n)
    mode, deep = a.plan_text(rep, stride=3)
    assert mode == 3 and deep > 0.05
    rnd = gen.iid_text(9, 0, 400_000)
    mode, deep = a.plan_text(rnd, stride=3)
    assert mode == -1 and deep < 0.01
    assert a.plan_text(b"")[0] == -1
