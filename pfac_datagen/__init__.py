"""Seeded synthetic inputs for the PFAC hot path (shared by the oracle side and the CUDA side).

This module holds NO matching arithmetic: it only draws pattern sets and ASCII DNA texts.
Both `oracle/` and `paper_1811_10498_b200/` consume what it returns; neither imports the other.

Recipe (stated again in DESIGN.md §3):

* PRNG: counter-based SplitMix64.  ``u64(key, i)`` is the SplitMix64 output after ``i+1``
  increments of a state initialised to ``key``; every substream has its own key,
  ``key = mix(seed * GOLDEN ^ fnv1a64(name))``.  Being counter-based, any slice of a text can be
  regenerated independently (needed to hand each GPU rank its own shard).
* Text (configs 1-4): iid uniform ACGT, 32 bases per 64-bit word, base t of word w is
  ``(u64(key_text, w) >> 2t) & 3`` mapped through ``b"ACGT"``.
* Planting: for every block of 4096 bases one pattern ``j = r % k`` is copied at offset
  ``(r >> 32) % (4096 - |p| + 1)`` inside the block (``r = u64(key_plant, block)``); a pattern
  that would run past the end of the text is not planted.  Chance matches of 20-100 bp patterns
  on random text are ~0, so planting is what gives configs 2-4 a non-empty match list.
* Patterns: lengths ``lo + u64(key_len, j) % (hi - lo + 1)``; bases from one counter stream
  consumed in order; a duplicate is redrawn from the next bases of the stream.
* Config 5 (divergence stress, BASELINE.json configs[4]): nested-prefix families (all prefixes of
  length 8..100 of 4 homopolymers and 8 primitive tandem units of length 2-6 repeated to 100 bp,
  one rotation per unit) plus 1000 random 20-mers; text made of segments, P(random)=1/2 (mean 512),
  P(homopolymer)=1/4 (mean 256), P(tandem)=1/4 (mean 512), geometric lengths.

Cited workload shapes: patterns of ~100 bp in sets of 1000-5000 (Table 2),
texts of 76-380 MB of DNA lines (Table 3); sizes per BASELINE.json `configs`.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
ACGT = np.frombuffer(b"ACGT", dtype=np.uint8)
PLANT_BLOCK = 4096


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    z ^= z >> np.uint64(30)
    z *= _M1
    z ^= z >> np.uint64(27)
    z *= _M2
    z ^= z >> np.uint64(31)
    return z


def _fnv1a64(name: str) -> int:
    h = 0xCBF29CE484222325
    for ch in name.encode():
        h ^= ch
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def substream_key(seed: int, name: str) -> int:
    """Key of the named substream of ``seed``."""
    x = ((seed * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF) ^ _fnv1a64(name)
    return int(_mix(np.array([x], dtype=np.uint64))[0])


def u64(key: int, start: int, count: int) -> np.ndarray:
    """Counter-based SplitMix64: outputs ``start .. start+count-1`` of the stream keyed ``key``."""
    with np.errstate(over="ignore"):
        idx = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        state = np.uint64(key) + idx * GOLDEN
        return _mix(state)


# --------------------------------------------------------------------------- iid text
def iid_codes(seed: int, a: int, b: int, name: str = "text") -> np.ndarray:
    """2-bit codes (0..3 = A,C,G,T) of bases [a, b) of the iid text of ``seed``."""
    if b <= a:
        return np.zeros(0, dtype=np.uint8)
    key = substream_key(seed, name)
    w0, w1 = a // 32, (b - 1) // 32 + 1
    out = np.empty(b - a, dtype=np.uint8)
    chunk_words = 1 << 22  # 128 Mbases per chunk keeps temporaries bounded
    for cw in range(w0, w1, chunk_words):
        ce = min(w1, cw + chunk_words)
        words = u64(key, cw, ce - cw)
        # (words[:,None] >> 2t) & 3 for t in 0..31, done bytewise to stay light on memory
        by = words.view(np.uint8).reshape(-1, 8)  # little-endian: byte m holds bases 4m..4m+3
        codes = np.empty((ce - cw, 32), dtype=np.uint8)
        for t in range(4):
            codes[:, t::4] = (by >> np.uint8(2 * t)) & np.uint8(3)
        flat = codes.reshape(-1)
        lo = max(a, cw * 32)
        hi = min(b, ce * 32)
        out[lo - a:hi - a] = flat[lo - cw * 32:hi - cw * 32]
    return out


def iid_text(seed: int, a: int, b: int) -> np.ndarray:
    """ASCII bytes of bases [a, b) of the iid uniform ACGT text of ``seed``."""
    return ACGT[iid_codes(seed, a, b)]


# --------------------------------------------------------------------------- patterns
def random_patterns(seed: int, k: int, lo: int, hi: int, avoid=None, name: str = "patterns") -> list[bytes]:
    """k distinct iid ACGT patterns with lengths uniform in [lo, hi] (redrawn on duplicate)."""
    if k == 0:
        return []
    lens = lo + (u64(substream_key(seed, name + ":len"), 0, k) % np.uint64(hi - lo + 1)).astype(np.int64)
    seen = set(avoid or ())
    pats: list[bytes] = []
    need = int(lens.sum()) + 64 * hi
    key = name + ":bases"
    cursor = 0
    buf = iid_text_named(seed, key, 0, need)
    len_key = substream_key(seed, name + ":relen")
    redraws = 0
    for j in range(k):
        L = int(lens[j])
        tries = 0
        while True:
            if cursor + L > len(buf):
                buf = np.concatenate([buf, iid_text_named(seed, key, len(buf), len(buf) + need)])
            p = buf[cursor:cursor + L].tobytes()
            cursor += L
            if p not in seen:
                break
            tries += 1
            if tries >= 64:  # this length class may be exhausted (e.g. only 4 patterns of length 1)
                L = lo + int(u64(len_key, redraws, 1)[0] % np.uint64(hi - lo + 1))
                redraws += 1
                tries = 0
                if redraws > 64 * k + 1024:
                    raise ValueError(f"cannot draw {k} distinct patterns with lengths in [{lo}, {hi}]")
        seen.add(p)
        pats.append(p)
    return pats


def iid_text_named(seed: int, name: str, a: int, b: int) -> np.ndarray:
    return ACGT[iid_codes(seed, a, b, name=name)]


def all_kmers(k: int) -> list[bytes]:
    """All 4^k k-mers in lexicographic (A<C<G<T) order: the closed-form workload of SURVEY §8(c)."""
    if k == 0:
        return []
    idx = np.arange(4 ** k, dtype=np.int64)
    codes = np.stack([(idx >> (2 * (k - 1 - t))) & 3 for t in range(k)], axis=1).astype(np.uint8)
    return [bytes(r) for r in ACGT[codes]]


# --------------------------------------------------------------------------- planting
def plant(text: np.ndarray, a: int, n_total: int, patterns: list[bytes], seed: int) -> np.ndarray:
    """Overwrite the planted patterns that overlap ``text`` = bases [a, a+len(text)) in place."""
    if not patterns or len(text) == 0:
        return text
    b = a + len(text)
    key = substream_key(seed, "plant")
    blk0, blk1 = a // PLANT_BLOCK, (b - 1) // PLANT_BLOCK + 1
    r = u64(key, blk0, blk1 - blk0)
    k = len(patterns)
    lens = np.fromiter((len(p) for p in patterns), dtype=np.int64, count=k)
    j = (r % np.uint64(k)).astype(np.int64)
    L = lens[j]
    span = np.maximum(PLANT_BLOCK - L + 1, 1).astype(np.uint64)
    off = ((r >> np.uint64(32)) % span).astype(np.int64)
    starts = (np.arange(blk0, blk1, dtype=np.int64) * PLANT_BLOCK) + off
    for s, jj, ll in zip(starts.tolist(), j.tolist(), L.tolist()):
        if ll > PLANT_BLOCK or s + ll > n_total:
            continue
        lo, hi = max(s, a), min(s + ll, b)
        if lo >= hi:
            continue
        p = patterns[jj]
        text[lo - a:hi - a] = np.frombuffer(p[lo - s:hi - s], dtype=np.uint8)
    return text


# --------------------------------------------------------------------------- barriers (reading R5)
BARRIER_BYTES = np.frombuffer(b"NNNNNNRYKMn-", dtype=np.uint8)


def add_barriers(text: np.ndarray, seed: int, line: int = 80, block: int = 4096, run_max: int = 300,
                 run_frac: float = 0.25, a: int = 0) -> np.ndarray:
    """FASTA-like barriers over ``text`` = bases [a, a+len(text)) in place: a newline after every
    ``line`` bases (global positions g with g mod (line+1) == line; line = 0: none) and, in a
    ``run_frac`` share of the ``block``-base blocks, one run of 1..run_max bytes drawn from
    BARRIER_BYTES (mostly 'N', the assembly-gap code) at a random offset.  Holds none of the method's
    arithmetic; both the oracle and the CUDA path read the result."""
    n = len(text)
    if n == 0:
        return text
    b = a + n
    if line > 0:
        first = a + (line - a % (line + 1)) % (line + 1)
        text[first - a::line + 1] = ord("\n")
    blk0 = max(0, (a - run_max - block) // block)
    blk1 = (b - 1) // block + 1
    nb = blk1 - blk0
    key = substream_key(seed, "barriers")
    r, r2 = u64(key, blk0, nb), u64(key, (1 << 40) + blk0, nb)
    pick = (r >> np.uint64(11)).astype(np.float64) / float(1 << 53) < run_frac
    ln = (r % np.uint64(run_max)).astype(np.int64) + 1
    off = ((r2 >> np.uint64(32)) % np.uint64(block)).astype(np.int64)
    code = (r2 % np.uint64(len(BARRIER_BYTES))).astype(np.int64)
    for j in np.nonzero(pick)[0].tolist():
        s = (blk0 + j) * block + int(off[j])
        lo, hi = max(s, a), min(b, s + int(ln[j]))
        if lo < hi:
            text[lo - a:hi - a] = BARRIER_BYTES[int(code[j])]
    return text


# --------------------------------------------------------------------------- config 5 (repetitive)
def _primitive(u: bytes) -> bool:
    n = len(u)
    return not any(n % d == 0 and u[:d] * (n // d) == u for d in range(1, n))


def repeat_family_seeds(seed: int) -> tuple[list[bytes], list[bytes]]:
    """(seeds of length 100, tandem units): 4 homopolymers, then 8 primitive tandem units."""
    seeds = [bytes([c]) * 100 for c in b"ACGT"]
    units: list[bytes] = []
    key = substream_key(seed, "units")
    i = 0
    while len(units) < 8:
        r = int(u64(key, i, 1)[0])
        i += 1
        L = 2 + r % 5
        u = bytes(ACGT[[(r >> (8 + 2 * t)) & 3 for t in range(L)]])
        rots = {u[s:] + u[:s] for s in range(L)}
        if not _primitive(u) or any(x in rots for x in units) or any(
                (x * 100)[:100] == (u * 100)[:100] for x in units):
            continue
        units.append(u)
    seeds += [(u * (100 // len(u) + 1))[:100] for u in units]
    return seeds, units


def repetitive_patterns(seed: int) -> list[bytes]:
    seeds, _ = repeat_family_seeds(seed)
    pats: list[bytes] = []
    seen = set()
    for s in seeds:
        for L in range(8, 101):
            p = s[:L]
            if p not in seen:
                seen.add(p)
                pats.append(p)
    pats += random_patterns(seed, 1000, 20, 20, avoid=seen)
    return pats


def repetitive_text(seed: int, n: int) -> np.ndarray:
    """Low-entropy text: random / homopolymer / tandem segments (config 5)."""
    _, units = repeat_family_seeds(seed)
    codes = iid_codes(seed, 0, n)
    key = substream_key(seed, "segments")
    unit_codes = [np.frombuffer(u, dtype=np.uint8) for u in units]
    lut = np.zeros(256, dtype=np.uint8)
    lut[ord("A")], lut[ord("C")], lut[ord("G")], lut[ord("T")] = 0, 1, 2, 3
    unit_codes = [lut[u] for u in unit_codes]
    pos = 0
    seg = 0
    chunk = 1 << 16
    while pos < n:
        r = u64(key, seg, chunk)
        seg += chunk
        kind = (r & np.uint64(3)).astype(np.int64)            # 0,1 random; 2 homopolymer; 3 tandem
        uf = ((r >> np.uint64(11)).astype(np.float64) + 0.5) / float(1 << 53)
        mean = np.where(kind == 2, 256.0, 512.0)
        lens = np.maximum(1, np.ceil(-mean * np.log(uf))).astype(np.int64)
        starts = pos + np.concatenate([[0], np.cumsum(lens)[:-1]])
        keep = starts < n
        kind, lens, starts, r = kind[keep], lens[keep], starts[keep], r[keep]
        lens = np.minimum(lens, n - starts)
        for t, L, s, rr in zip(kind.tolist(), lens.tolist(), starts.tolist(), r.tolist()):
            if t == 2:
                codes[s:s + L] = (rr >> 8) & 3
            elif t == 3:
                u = unit_codes[(rr >> 8) % len(unit_codes)]
                reps = L // len(u) + 1
                codes[s:s + L] = np.tile(u, reps)[:L]
        pos = int(starts[-1] + lens[-1]) if len(starts) else n
    return ACGT[codes]


# --------------------------------------------------------------------------- configs
@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json workload (``configs[idx-1]``)."""
    idx: int
    n: int
    k: int
    lo: int
    hi: int
    repetitive: bool = False
    name: str = ""

    @property
    def seed(self) -> int:
        return self.idx


CONFIGS = {
    1: Config(1, 1_000_000, 100, 8, 20, name="cfg1: 1 Mbp random ACGT, 100 patterns of length 8-20"),
    2: Config(2, 256_000_000, 1000, 20, 20, name="cfg2: 256 Mbp random ACGT, 1000 patterns of length 20"),
    3: Config(3, 3_100_000_000, 10_000, 16, 64, name="cfg3: 3.1 Gbp random ACGT, 10000 patterns of length 16-64"),
    4: Config(4, 1_000_000_000, 100_000, 24, 100, name="cfg4: 1 Gbp random ACGT, 100000 patterns of length 24-100"),
    5: Config(5, 512_000_000, 2116, 8, 100, repetitive=True,
              name="cfg5: 512 Mbp repetitive text, nested-prefix families + 1000 random 20-mers"),
}


def config_patterns(cfg: Config) -> list[bytes]:
    if cfg.repetitive:
        return repetitive_patterns(cfg.seed)
    return random_patterns(cfg.seed, cfg.k, cfg.lo, cfg.hi)


def config_text(cfg: Config, a: int = 0, b: int | None = None, patterns: list[bytes] | None = None,
                n: int | None = None) -> np.ndarray:
    """ASCII text of bases [a, b) of config ``cfg`` (planted). ``n`` overrides the total length."""
    n_total = cfg.n if n is None else n
    b = n_total if b is None else min(b, n_total)
    if patterns is None:
        patterns = config_patterns(cfg)
    if cfg.repetitive:
        t = repetitive_text(cfg.seed, b)[a:b].copy()
    else:
        t = iid_text(cfg.seed, a, b)
    return plant(t, a, n_total, patterns, cfg.seed)


def flatten(patterns: list[bytes]) -> tuple[np.ndarray, np.ndarray]:
    """(bytes, offsets) with pattern j = bytes[offsets[j]:offsets[j+1]] (the C-ABI's pattern form)."""
    offs = np.zeros(len(patterns) + 1, dtype=np.uint64)
    if patterns:
        offs[1:] = np.cumsum([len(p) for p in patterns])
    data = np.frombuffer(b"".join(patterns), dtype=np.uint8).copy() if patterns else np.zeros(0, np.uint8)
    return data, offs


def expected_chance_matches(n: int, patterns: list[bytes]) -> float:
    """SPEC.md:366 hit-rate sanity: sum_p (n - |p| + 1) * 4^-|p| for iid uniform text."""
    return sum(max(0, n - len(p) + 1) * math.pow(4.0, -len(p)) for p in patterns)
