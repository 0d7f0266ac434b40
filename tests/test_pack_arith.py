"""CPU check (-m "not gpu") of the byte arithmetic the pack and text-input kernels share
(paper_1811_10498_b200/csrc/pack_common.cuh, compiled here for the host with g++).

pack16 must give, for every 16-byte group, the 2-bit codes A0 C1 G2 T3 of include/pfac.h (base j
at bits 2j) for every ACGTacgt byte, and flag the group iff one of its bytes is outside ACGTacgt
(reading R5).  Checked exhaustively: every byte value at every one of the 16 positions (the other
15 random valid bases), plus random groups mixing valid and invalid bytes.
"""
import ctypes
import os
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_1811_10498_b200", "csrc", "pack_common.cuh")

SRC = r'''
#include <cstddef>
#include "%s"
extern "C" void bad_masks(const uint8_t *b, size_t groups, uint32_t *masks) {
    for (size_t g = 0; g < groups; ++g) {
        uint32_t r[4];
        for (int k = 0; k < 4; ++k) {
            const uint32_t x = b[16 * g + 4 * k] | (b[16 * g + 4 * k + 1] << 8) | (b[16 * g + 4 * k + 2] << 16) |
                               ((uint32_t)b[16 * g + 4 * k + 3] << 24);
            pfac::pack4r(x, r[k]);
        }
        masks[g] = pfac::badmask16(r[0], r[1], r[2], r[3]);
    }
}
extern "C" void pack_groups(const uint8_t *b, size_t groups, uint32_t *words, uint8_t *bad) {
    for (size_t g = 0; g < groups; ++g) {
        uint32_t v[4];
        for (int k = 0; k < 4; ++k)
            v[k] = b[16 * g + 4 * k] | (b[16 * g + 4 * k + 1] << 8) | (b[16 * g + 4 * k + 2] << 16) |
                   ((uint32_t)b[16 * g + 4 * k + 3] << 24);
        uint32_t acc = 0;
        words[g] = pfac::pack16(v[0], v[1], v[2], v[3], acc);
        bad[g] = (acc & pfac::kBadMask) != 0;
    }
}
'''


@pytest.fixture(scope="module")
def lib():
    d = tempfile.mkdtemp()
    src = os.path.join(d, "p.cpp")
    so = os.path.join(d, "p.so")
    with open(src, "w") as f:
        f.write(SRC % HDR)
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-x", "c++", "-shared", "-fPIC", "-o", so, src])
    L = ctypes.CDLL(so)
    L.pack_groups.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]
    L.bad_masks.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    return L


CODE = {ord(c): i for i, c in enumerate("ACGT")} | {ord(c): i for i, c in enumerate("acgt")}


def run(L, groups: np.ndarray):
    g = np.ascontiguousarray(groups, dtype=np.uint8)
    n = len(g)
    words = np.zeros(n, np.uint32)
    bad = np.zeros(n, np.uint8)
    L.pack_groups(g.ctypes.data, n, words.ctypes.data, bad.ctypes.data)
    return words, bad.astype(bool)


def expected(groups: np.ndarray):
    valid = np.isin(groups, np.frombuffer(b"ACGTacgt", np.uint8))
    codes = np.vectorize(lambda b: CODE.get(int(b), 0))(groups).astype(np.uint64)
    words = (codes << (2 * np.arange(16, dtype=np.uint64))).sum(axis=1)
    return words.astype(np.uint32), ~valid.all(axis=1), valid


def test_every_byte_at_every_position(lib):
    rng = np.random.default_rng(0)
    acgt = np.frombuffer(b"ACGTacgt", np.uint8)
    groups = acgt[rng.integers(0, 8, (256 * 16, 16))]
    for p in range(16):
        groups[p * 256:(p + 1) * 256, p] = np.arange(256)
    words, bad = run(lib, groups)
    ew, ebad, valid = expected(groups)
    assert (bad == ebad).all()
    ok = valid.all(axis=1)  # codes are defined only for ACGTacgt bytes
    assert (words[ok] == ew[ok]).all()


def test_random_groups(lib):
    rng = np.random.default_rng(1)
    alphabet = np.frombuffer(b"ACGTacgtNnRYKMSWBDHVU-\n\r >eEuU", np.uint8)
    groups = alphabet[rng.integers(0, len(alphabet), (200_000, 16))]
    groups[::2] = np.frombuffer(b"ACGTacgt", np.uint8)[rng.integers(0, 8, (100_000, 16))]
    words, bad = run(lib, groups)
    ew, ebad, valid = expected(groups)
    assert (bad == ebad).all()
    assert (words[~ebad] == ew[~ebad]).all()


def test_exact_barrier_bits_from_residues(lib):
    """badmask16: bit j set iff byte j of the group is outside ACGTacgt (the text kernel's barrier
    bits, reading R5), for every byte value at every position and for random mixed groups."""
    rng = np.random.default_rng(2)
    acgt = np.frombuffer(b"ACGTacgt", np.uint8)
    groups = acgt[rng.integers(0, 8, (256 * 16, 16))]
    for p in range(16):
        groups[p * 256:(p + 1) * 256, p] = np.arange(256)
    alphabet = np.frombuffer(b"ACGTacgtNnRYKM-\n>", np.uint8)
    groups = np.concatenate([groups, alphabet[rng.integers(0, len(alphabet), (100_000, 16))]])
    g = np.ascontiguousarray(groups)
    masks = np.zeros(len(g), np.uint32)
    lib.bad_masks(g.ctypes.data, len(g), masks.ctypes.data)
    invalid = ~np.isin(g, acgt)
    expect = (invalid.astype(np.uint32) << np.arange(16, dtype=np.uint32)).sum(axis=1)
    assert (masks == expect).all()
