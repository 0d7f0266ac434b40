"""O1 — brute force by direct substring comparison.  TEST INFRASTRUCTURE ONLY.

The plain definition that the PFAC walk reaches exactly: out[i] is the id of the
*longest* pattern p with text[i .. i+|p|) = p, or 0 — "PFAC can detect only the longest patterns and
it does not detect sub-patterns" (§IV).  Letters compare case-insensitively (DESIGN.md
reading R4); any other byte equals no pattern letter (reading R5).  Pure Python, tiny inputs only.
"""
from __future__ import annotations


def _norm(b: bytes) -> bytes:
    return bytes(c - 32 if 97 <= c <= 122 else c for c in b)


def all_occurrences(patterns: list[bytes], text: bytes) -> set[tuple[int, int]]:
    """Every (start, id) with text[start:start+|p|] == p (scan_naive)."""
    t = _norm(bytes(text))
    ps = [_norm(p) for p in patterns]
    occ = set()
    for i in range(len(t)):
        for j, p in enumerate(ps):
            if t[i:i + len(p)] == p:
                occ.add((i, j + 1))
    return occ


def longest_at(patterns: list[bytes], text: bytes) -> list[int]:
    """out[i] = id of the longest pattern occurring at i, else 0."""
    t = _norm(bytes(text))
    ps = [_norm(p) for p in patterns]
    out = []
    for i in range(len(t)):
        best, best_len = 0, 0
        for j, p in enumerate(ps):
            if len(p) > best_len and t[i:i + len(p)] == p:
                best, best_len = j + 1, len(p)
        out.append(best)
    return out
