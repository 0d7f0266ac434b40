"""O3 — the classic serial Aho-Corasick machine.  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §III (lines 62-87): build the goto function (the goto graph of Fig. 1, states
numbered in insertion order), then the failure function "calculated for all the states of the goto
graph" (breadth-first, as in the original Aho-Corasick construction), then the output
function (the red output nodes of Fig. 2).  The processing phase reads the text
once: on a goto miss it follows failure links; whenever it is in an output state it reports the
patterns of that state.  A byte outside ACGTacgt resets the machine to the start state (DESIGN.md
reading R5, the barrier).

Used only to cross-check O2: every pattern occurring at i is a prefix of the longest one occurring at
i, so the all-occurrence set of this machine must equal ``expand(out)`` (SURVEY.md §8(c) pin O3).
"""
from __future__ import annotations

from collections import deque

LETTERS = {ord(c): c.upper() for c in "ACGTacgt"}


class ClassicAC:
    def __init__(self, patterns: list[bytes]):
        self.patterns = [bytes(p).upper() for p in patterns]
        # goto function: goto[s][letter] -> state; states numbered as created (Fig. 1)
        self.goto: list[dict[str, int]] = [{}]
        self.own: list[int] = [0]  # pattern id whose last letter enters state s (0 = none)
        for pid, p in enumerate(self.patterns, start=1):
            s = 0
            for ch in p.decode():
                if ch not in self.goto[s]:
                    self.goto.append({})
                    self.own.append(0)
                    self.goto[s][ch] = len(self.goto) - 1
                s = self.goto[s][ch]
            self.own[s] = pid
        # failure function, breadth-first from the start state
        n = len(self.goto)
        self.fail = [0] * n
        self.depth = [0] * n
        q = deque()
        for ch, s in self.goto[0].items():
            self.fail[s] = 0
            self.depth[s] = 1
            q.append(s)
        order = []
        while q:
            r = q.popleft()
            order.append(r)
            for ch, s in self.goto[r].items():
                q.append(s)
                self.depth[s] = self.depth[r] + 1
                f = self.fail[r]
                while f != 0 and ch not in self.goto[f]:
                    f = self.fail[f]
                self.fail[s] = self.goto[f].get(ch, 0)
        # output function: own pattern plus the outputs of the failure state (BFS order => ready)
        self.output: list[set[int]] = [set() for _ in range(n)]
        for s in order:
            self.output[s] = ({self.own[s]} if self.own[s] else set()) | self.output[self.fail[s]]

    def occurrences(self, text: bytes) -> set[tuple[int, int]]:
        """All (start, id) pairs found by the serial processing phase."""
        s = 0
        occ = set()
        for j, b in enumerate(bytes(text)):
            ch = LETTERS.get(b)
            if ch is None:          # no transition from any state: back to the start state
                s = 0
                continue
            while s != 0 and ch not in self.goto[s]:
                s = self.fail[s]    # goto failed: consult the failure function
            s = self.goto[s].get(ch, 0)
            for pid in self.output[s]:
                occ.add((j - len(self.patterns[pid - 1]) + 1, pid))
        return occ


def expand(out, patterns: list[bytes]) -> set[tuple[int, int]]:
    """{(i, q) : out[i] != 0 and pattern q is a prefix of pattern out[i]}."""
    ps = [bytes(p).upper() for p in patterns]
    prefixes: dict[int, list[int]] = {}
    by_str = {p: i + 1 for i, p in enumerate(ps)}
    occ = set()
    for i, v in enumerate(out):
        v = int(v)
        if v == 0:
            continue
        if v not in prefixes:
            p = ps[v - 1]
            prefixes[v] = [by_str[p[:L]] for L in range(1, len(p) + 1) if p[:L] in by_str]
        for q in prefixes[v]:
            occ.add((i, q))
    return occ
