"""The seeded generator: deterministic, position-addressable, planted as DESIGN.md §3 states."""
import numpy as np

import pfac_datagen as gen
from oracle import Oracle


def test_splitmix64_reference_values():
    # SplitMix64 with state 0: first outputs are the published reference sequence
    v = gen.u64(0, 0, 4)
    assert [hex(int(x)) for x in v] == ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4", "0x6c45d188009454f", "0xf88bb8a8724c81ec"]


def test_text_slices_are_position_addressable():
    full = gen.iid_text(3, 0, 10_000)
    assert set(np.unique(full).tobytes()) <= set(b"ACGT")
    for a, b in [(0, 1), (31, 33), (64, 4096), (9999, 10_000)]:
        assert (gen.iid_text(3, a, b) == full[a:b]).all()
    counts = np.bincount(np.searchsorted(np.frombuffer(b"ACGT", np.uint8), full), minlength=4)
    assert counts.min() > 2300 and counts.max() < 2700


def test_planting_slices_and_presence():
    cfg = gen.CONFIGS[1]
    P = gen.config_patterns(cfg)
    assert len(P) == 100 and len(set(P)) == 100
    assert all(8 <= len(p) <= 20 for p in P)
    n = 200_000
    full = gen.config_text(cfg, n=n, patterns=P)
    for a, b in [(0, 5000), (4090, 12_300), (199_000, 200_000)]:
        assert (gen.config_text(cfg, a, b, patterns=P, n=n) == full[a:b]).all()
    # every block holds its planted pattern somewhere -> at least ~n/4096 matches
    pos, pid = Oracle(P).match_list(full)
    assert len(pos) >= n // 4096 - 1


def test_config_shapes():
    assert [len(gen.config_patterns(gen.CONFIGS[i])) for i in (1, 2)] == [100, 1000]
    p5 = gen.config_patterns(gen.CONFIGS[5])
    assert len(p5) == len(set(p5)) == 12 * 93 + 1000
    t5 = gen.config_text(gen.CONFIGS[5], n=300_000)
    # low complexity: a large fraction of positions sit inside runs
    same = (t5[1:] == t5[:-1]).mean()
    assert same > 0.3


def test_exhausted_length_classes_terminate():
    """Only 4 patterns of length 1 exist: redraw the length instead of looping forever."""
    P = gen.random_patterns(41, 300, 1, 12)
    assert len(P) == len(set(P)) == 300 and all(1 <= len(p) <= 12 for p in P)
    import pytest
    with pytest.raises(ValueError):
        gen.random_patterns(1, 30, 1, 2)  # only 4 + 16 = 20 distinct patterns exist


def bad_at(t):
    return ~np.isin(t, np.frombuffer(b"ACGT", np.uint8))


def test_add_barriers_windows_and_layout():
    """Barrier placement depends on global positions only (shards see the same bytes as the whole)."""
    n = 300_000
    full = gen.add_barriers(gen.iid_text(1, 0, n), 1, line=60, block=2048, run_max=3000, run_frac=0.4)
    for a, b in [(0, 1000), (12_345, 200_000), (150_000, n), (n - 1, n)]:
        part = gen.add_barriers(gen.iid_text(1, a, b), 1, line=60, block=2048, run_max=3000, run_frac=0.4, a=a)
        assert (part == full[a:b]).all()
    assert bad_at(full)[60::61].all() and (full[60::61] == ord("\n")).mean() > 0.5  # runs may cover a newline
    bad = bad_at(full)
    assert set(np.unique(full[bad]).tolist()) <= set(gen.BARRIER_BYTES.tolist()) | {ord("\n")}
    assert 0.05 < (full == ord("N")).mean() < 0.5
