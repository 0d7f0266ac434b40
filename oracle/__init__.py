"""PFAC oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` and
``--impl reference`` legs) may import this package.  It shares no code with the product package
``paper_1811_10498_b200`` and the product never imports it.

Contents (each function cites the passage it follows):

* ``Oracle`` — O2, the bit-exactness reference: the paper's insertion-order 4 x N transition
  table (Table 1) walked failure-lessly from every text position
  (PAPER.md:91-93, :204).  Implemented in plain C (``pfac_oracle.c``), loaded with ctypes.
  ``Oracle.match_all`` emits every pattern the walk completes (all occurrences, ascending length).
* ``bruteforce.longest_at`` — O1, the plain definition by direct substring comparison.
* ``classic_ac`` — O3, the serial Aho-Corasick machine with goto/failure/output
  (PAPER.md:62-87), whose all-occurrence set must equal ``expand(out)``.

Pins (tests/test_oracle_pins.py): Fig. 1, Table 1 rows 0-5,
hand-worked outputs (tests/golden/), exhaustive brute force on tiny inputs, classic AC agreement
and closed forms.  No part of the oracle is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pfac_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ERRORS = {-2: "empty pattern", -3: "non-ACGT pattern byte", -4: "duplicate pattern", -9: "out of memory"}


def build_lib(force: bool = False) -> str:
    """Compile the C oracle with gcc (plain -O2, no vectorisation tricks)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build_lib())
        vp, u8p, u64p, u32p, i32p = (ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint8),
                                     ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32),
                                     ctypes.POINTER(ctypes.c_int32))
        L.oracle_build.argtypes = [u8p, u64p, ctypes.c_uint32, ctypes.POINTER(vp), u32p, u32p]
        L.oracle_build.restype = ctypes.c_int
        L.oracle_free.argtypes = [vp]
        L.oracle_num_states.argtypes = [vp]
        L.oracle_num_states.restype = ctypes.c_uint32
        L.oracle_max_len.argtypes = [vp]
        L.oracle_max_len.restype = ctypes.c_uint32
        L.oracle_cell.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32, u32p, u32p]
        L.oracle_match.argtypes = [vp, u8p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, i32p]
        L.oracle_match_list.argtypes = [vp, u8p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                        u64p, u32p, ctypes.c_uint64]
        L.oracle_match_list.restype = ctypes.c_uint64
        L.oracle_match_all.argtypes = L.oracle_match_list.argtypes
        L.oracle_match_all.restype = ctypes.c_uint64
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class OracleError(ValueError):
    def __init__(self, code: int, bad_id: int, other_id: int):
        self.code, self.bad_id, self.other_id = code, bad_id, other_id
        super().__init__(f"{ERRORS.get(code, code)} (pattern id {bad_id}"
                         + (f", repeats id {other_id})" if other_id else ")"))


COLUMNS = "ATCG"  # the paper's column order


class Oracle:
    """O2: the paper's transition table + failure-less per-position walk (see pfac_oracle.c)."""

    def __init__(self, patterns: list[bytes]):
        data = np.frombuffer(b"".join(patterns), dtype=np.uint8).copy() if patterns else np.zeros(1, np.uint8)
        offs = np.zeros(len(patterns) + 1, dtype=np.uint64)
        if patterns:
            offs[1:] = np.cumsum([len(p) for p in patterns])
        h = ctypes.c_void_p()
        bad, other = ctypes.c_uint32(0), ctypes.c_uint32(0)
        rc = lib().oracle_build(_ptr(data, ctypes.c_uint8), _ptr(offs, ctypes.c_uint64), len(patterns),
                                ctypes.byref(h), ctypes.byref(bad), ctypes.byref(other))
        if rc != 0:
            raise OracleError(rc, bad.value, other.value)
        self._h = h
        self.k = len(patterns)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.oracle_free(h)
            self._h = None

    @property
    def num_states(self) -> int:
        return int(lib().oracle_num_states(self._h))

    @property
    def max_len(self) -> int:
        return int(lib().oracle_max_len(self._h))

    def cell(self, s: int, letter: str) -> tuple[int, int]:
        """(next state, matched pattern id) of Table-1 cell (s, letter)."""
        nx, pid = ctypes.c_uint32(), ctypes.c_uint32()
        lib().oracle_cell(self._h, s, COLUMNS.index(letter), ctypes.byref(nx), ctypes.byref(pid))
        return nx.value, pid.value

    def table(self) -> np.ndarray:
        """The whole 4 x N table as an (N, 4, 2) array, columns A,T,C,G."""
        S = self.num_states
        t = np.zeros((S, 4, 2), dtype=np.uint32)
        for s in range(S):
            for c in range(4):
                t[s, c] = self.cell(s, COLUMNS[c])
        return t

    def match(self, text, a: int = 0, b: int | None = None, n: int | None = None) -> np.ndarray:
        """out[i - a] for i in [a, b); walks read text up to n (default len(text))."""
        t = _as_u8(text)
        n = len(t) if n is None else n
        b = n if b is None else b
        out = np.zeros(max(0, b - a), dtype=np.int32)
        if b > a:
            lib().oracle_match(self._h, _ptr(t, ctypes.c_uint8) if len(t) else None, n, a, b,
                               _ptr(out, ctypes.c_int32))
        return out

    def match_list(self, text, a: int = 0, b: int | None = None, n: int | None = None,
                   cap: int | None = None) -> tuple[np.ndarray, np.ndarray]:
        """(pos uint64, pid uint32) of out[i] != 0 for i in [a, b), ascending."""
        t = _as_u8(text)
        n = len(t) if n is None else n
        b = n if b is None else b
        cap = max(1, (b - a) // 64 + 1024) if cap is None else cap
        while True:
            pos = np.zeros(cap, dtype=np.uint64)
            pid = np.zeros(cap, dtype=np.uint32)
            m = 0
            if b > a:
                m = int(lib().oracle_match_list(self._h, _ptr(t, ctypes.c_uint8), n, a, b,
                                                _ptr(pos, ctypes.c_uint64), _ptr(pid, ctypes.c_uint32), cap))
            if m <= cap:
                return pos[:m], pid[:m]
            cap = m


    def match_all(self, text, a: int = 0, b: int | None = None, n: int | None = None,
                  cap: int | None = None) -> tuple[np.ndarray, np.ndarray]:
        """Every occurrence (pos uint64, pid uint32) starting in [a, b): ascending position, then
        ascending pattern length (pfac_oracle.c oracle_match_all)."""
        t = _as_u8(text)
        n = len(t) if n is None else n
        b = n if b is None else b
        cap = max(1, (b - a) // 32 + 1024) if cap is None else cap
        while True:
            pos = np.zeros(cap, dtype=np.uint64)
            pid = np.zeros(cap, dtype=np.uint32)
            m = 0
            if b > a:
                m = int(lib().oracle_match_all(self._h, _ptr(t, ctypes.c_uint8), n, a, b,
                                               _ptr(pos, ctypes.c_uint64), _ptr(pid, ctypes.c_uint32), cap))
            if m <= cap:
                return pos[:m], pid[:m]
            cap = m


def _as_u8(text) -> np.ndarray:
    if isinstance(text, (bytes, bytearray)):
        return np.frombuffer(bytes(text), dtype=np.uint8)
    t = np.asarray(text)
    assert t.dtype == np.uint8
    return np.ascontiguousarray(t)
