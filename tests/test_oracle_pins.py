"""Pins for the oracle (-m "not gpu"): each test fixes the oracle against something other than itself.

* Fig. 1 goto graph / Table 1 rows 0-5 (paper's printed values)            -> trie construction
* hand-worked outputs (tests/golden/hand_outputs.json)                       -> per-position walk
* exhaustive brute force over all short texts (O1, the plain definition)     -> the walk, exactly
* classic failure-link Aho-Corasick all-occurrence sets (O3, §III) -> longest-only semantics
* closed forms (all k-mers, nested homopolymer family)                       -> large n without a 2nd run
"""
import itertools
import random

import numpy as np
import pytest

import pfac_datagen as gen
from oracle import Oracle, OracleError
from oracle.bruteforce import all_occurrences, longest_at
from oracle.classic_ac import ClassicAC, expand


def pats(*xs):
    return [x.encode() for x in xs]


# --------------------------------------------------------------------------- paper pins
def test_fig1_goto_graph(golden):
    g = golden("fig1_goto_graph.json")
    o = Oracle(pats(*g["patterns"]))
    assert o.num_states == g["num_states"]
    for letter, s in g["root_edges"].items():
        assert o.cell(0, letter)[0] == s
    assert o.cell(0, "G") == (0, 0)
    # the state each pattern is matched in = the target of the edge carrying its id
    for pid, p in enumerate(g["patterns"], start=1):
        s = 0
        for ch in p:
            nxt, got = o.cell(s, ch)
            s = nxt
        assert s == g["final_state"][p]
        assert got == pid


def test_table1_rows_0_to_5(golden):
    g = golden("table1_rows0_5.json")
    o = Oracle(pats(*g["patterns"]))
    for s, letter, nxt, pid in g["cells"]:
        assert o.cell(s, letter) == (nxt, pid), (s, letter)
    assert o.num_states == g["num_states_fresh_allocation"]


def test_fig2_failure_function(golden):
    g = golden("fig2_failure.json")
    ac = ClassicAC(pats(*g["patterns"]))
    assert len(ac.goto) == 10
    for s, f in g["failure"].items():
        assert ac.fail[int(s)] == f, s
    for s in range(10):
        assert ac.output[s] == set(g["outputs"].get(str(s), [])), s


def test_hand_outputs(golden):
    for case in golden("hand_outputs.json")["cases"]:
        o = Oracle(pats(*case["patterns"]))
        got = o.match(case["text"].encode()).tolist()
        assert got == case["out"], case
        assert longest_at(pats(*case["patterns"]), case["text"].encode()) == case["out"], case


def test_build_errors():
    with pytest.raises(OracleError) as e:
        Oracle(pats("AC", ""))
    assert e.value.code == -2 and e.value.bad_id == 2
    with pytest.raises(OracleError) as e:
        Oracle(pats("AC", "ANC"))
    assert e.value.code == -3 and e.value.bad_id == 2
    with pytest.raises(OracleError) as e:
        Oracle(pats("ACG", "TT", "acg"))
    assert e.value.code == -4 and (e.value.bad_id, e.value.other_id) == (3, 1)


# --------------------------------------------------------------------------- brute force (O1)
def _random_set(rng, k, lo, hi, alphabet="ACGT"):
    seen, out = set(), []
    while len(out) < k:
        p = "".join(rng.choice(alphabet) for _ in range(rng.randint(lo, hi)))
        if p.upper() not in seen:
            seen.add(p.upper())
            out.append(p.encode())
    return out


def test_exhaustive_short_texts_vs_bruteforce():
    """All texts over {A,C,G,T} of length <= 6 for 12 random small pattern sets (exact)."""
    rng = random.Random(1811)
    texts = [b""] + [bytes(t) for L in range(1, 7) for t in itertools.product(b"ACGT", repeat=L)]
    for trial in range(12):
        P = _random_set(rng, rng.randint(1, 6), 1, 4)
        o = Oracle(P)
        for t in texts:
            assert o.match(t).tolist() == longest_at(P, t), (P, t)


def test_random_vs_bruteforce_with_barriers_and_case():
    """SPEC.md:186/:508 style: 1-50 patterns of length 1-20, texts over {A,C,G,T,N,a,c,g,t}."""
    rng = random.Random(7)
    for trial in range(150):
        P = _random_set(rng, rng.randint(1, 50), 1, rng.choice([3, 6, 20]), alphabet="ACGTacgt")
        L = rng.randint(0, 400)
        alpha = rng.choice(["ACGT", "ACGTN", "AC", "AAAAC", "ACGTacgtN\n"])
        t = "".join(rng.choice(alpha) for _ in range(L)).encode()
        # plant a few patterns so long matches happen
        t = bytearray(t)
        for _ in range(rng.randint(0, 5)):
            if not t:
                break
            p = rng.choice(P)
            i = rng.randrange(len(t))
            t[i:i + len(p)] = p
        t = bytes(t)
        assert Oracle(P).match(t).tolist() == longest_at(P, t), (P, t)


# --------------------------------------------------------------------------- classic AC (O3)
def test_classic_ac_matches_bruteforce_occurrences():
    rng = random.Random(3)
    for trial in range(100):
        P = _random_set(rng, rng.randint(1, 30), 1, 8)
        t = "".join(rng.choice("ACGTN") for _ in range(rng.randint(0, 300))).encode()
        assert ClassicAC(P).occurrences(t) == all_occurrences(P, t)


def test_expand_longest_equals_classic_ac():
    """expand(PFAC longest-only out) == all occurrences of the failure-link machine (§III vs §IV)."""
    rng = random.Random(11)
    for trial in range(300):
        P = _random_set(rng, rng.randint(1, 40), 1, rng.choice([4, 10, 20]))
        t = bytearray("".join(rng.choice("ACGTN") for _ in range(rng.randint(0, 2000))).encode())
        for _ in range(rng.randint(0, 20)):
            if t:
                p = rng.choice(P)
                i = rng.randrange(len(t))
                t[i:i + len(p)] = p
        t = bytes(t)
        out = Oracle(P).match(t)
        assert expand(out, P) == ClassicAC(P).occurrences(t)


def test_match_all_equals_classic_ac_and_bruteforce():
    """Oracle.match_all (every final the walk passes) == classic AC occurrences == brute force, as a list
    ordered by position then length."""
    rng = random.Random(13)
    for trial in range(300):
        P = _random_set(rng, rng.randint(1, 40), 1, rng.choice([3, 8, 20]))
        t = bytearray("".join(rng.choice("ACGTN") for _ in range(rng.randint(0, 1500))).encode())
        for _ in range(rng.randint(0, 20)):
            if t:
                p = rng.choice(P)
                i = rng.randrange(len(t))
                t[i:i + len(p)] = p
        t = bytes(t)
        pos, pid = Oracle(P).match_all(t)
        got = list(zip(pos.tolist(), pid.tolist()))
        exp = sorted(all_occurrences(P, t), key=lambda x: (x[0], len(P[x[1] - 1])))
        assert got == exp
        assert set(got) == ClassicAC(P).occurrences(t)


def test_match_all_nested_closed_form():
    """Nested family A^1..A^m over a poly-A run of length R then a non-A: position i has the
    min(m, R-i) occurrences A^1..A^min(m, R-i), in that order."""
    m, R = 7, 30
    P = [b"A" * L for L in range(1, m + 1)]
    pos, pid = Oracle(P).match_all(b"A" * R + b"C")
    exp = [(i, L) for i in range(R) for L in range(1, min(m, R - i) + 1)]
    assert list(zip(pos.tolist(), pid.tolist())) == exp


# --------------------------------------------------------------------------- closed forms
@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_all_kmers_closed_form(k):
    """Patterns = all 4^k k-mers, ids lexicographic -> out[i] = 1 + value4(text[i..i+k)) for i <= n-k."""
    P = gen.all_kmers(k)
    t = gen.iid_text(99, 0, 5000)
    out = Oracle(P).match(t)
    codes = np.searchsorted(np.frombuffer(b"ACGT", np.uint8), t).astype(np.int64)
    n = len(t)
    val = np.zeros(n, dtype=np.int64)
    for j in range(k):
        val[: n - k + 1] = val[: n - k + 1] * 4 + codes[j: n - k + 1 + j]
    exp = np.zeros(n, dtype=np.int64)
    exp[: n - k + 1] = 1 + val[: n - k + 1]
    assert (out == exp).all()
    assert Oracle(P).num_states == (4 ** (k + 1) - 1) // 3


def test_nested_homopolymer_closed_form():
    """Family A^1..A^m over a poly-A run of length R then a non-A: out[i] = min(m, R - i)."""
    for m, R in [(5, 3), (8, 100), (100, 250), (100, 100)]:
        P = [b"A" * L for L in range(1, m + 1)]
        t = b"A" * R + b"C" + b"A" * 7
        out = Oracle(P).match(t)
        assert out[:R].tolist() == [min(m, R - i) for i in range(R)]
        assert out[R] == 0
        assert out[R + 1:].tolist() == [min(m, 7 - i) for i in range(7)]


def test_range_and_walk_bound():
    """match over [a,b) with walks bounded by n equals the full run's slice (shard invariance)."""
    P = gen.random_patterns(5, 50, 3, 12)
    t = gen.plant(gen.iid_text(5, 0, 20000), 0, 20000, P, 5)
    o = Oracle(P)
    full = o.match(t)
    for a, b in [(0, 1), (17, 4099), (19990, 20000), (5000, 5000)]:
        assert (o.match(t, a, b) == full[a:b]).all()
    # a walk bound n < len(text) cuts walks exactly like a shorter text
    assert (o.match(t, 0, 9000, n=9000) == o.match(t[:9000])).all()
    pos, pid = o.match_list(t)
    nz = np.nonzero(full)[0]
    assert (pos == nz).all() and (pid == full[nz]).all()


def test_chance_rate_sanity():
    """chance matches ~ sum_p (n-|p|+1) 4^-|p| on iid text (no planting)."""
    P = gen.random_patterns(21, 200, 5, 7)
    n = 400_000
    t = gen.iid_text(21, 0, n)
    exp = gen.expected_chance_matches(n, P)
    got = len(expand(Oracle(P).match(t), P))
    assert abs(got - exp) < 6 * exp ** 0.5 + 5
