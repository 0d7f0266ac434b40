"""Builds libpfac.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build() and the binding."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "libpfac.so")
SOURCES = ["api.cu", "match.cu", "pack.cu", "compact.cu", "expand.cu", "builder.cpp"]
HEADERS = ["pfac_internal.h", "ptx.cuh", "pack_common.cuh", "compact_common.cuh", os.path.join("..", "..", "include", "pfac.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC,-O2", "-shared", "--cudart", "static",
]


def _inputs():
    return [os.path.join(CSRC, s) for s in SOURCES + HEADERS]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _inputs())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile libpfac.so; `out`/`defines` build an alternative library for A/B experiments."""
    target = out or LIB
    if out is None and not force and not stale():
        return LIB
    os.makedirs(os.path.dirname(target), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = target + f".tmp{os.getpid()}"
    cmd = [nvcc, *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines],
           "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target
