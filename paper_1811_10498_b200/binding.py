"""Thin ctypes binding of libpfac (include/pfac.h): argument marshalling only.

Every step of the path (pack, match, compact) runs in the CUDA kernels of libpfac.so; there is no
CPU fallback.  If the library cannot be loaded the import of the op fails loudly.  torch supplies
device memory (tensors) and streams; nothing here computes on tensors.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

_lib = None

OK, E_ARG, E_EMPTY, E_NON_ACGT, E_DUP, E_TOO_LONG, E_TOO_MANY, E_CAPACITY, E_CUDA, E_OOM = (
    0, -1, -2, -3, -4, -5, -6, -7, -8, -9)
MAX_LEN = 1024

_SIGS = {
    "pfac_build": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]),
    "pfac_free": (None, [ctypes.c_void_p]),
    "pfac_num_states": (ctypes.c_uint32, [ctypes.c_void_p]),
    "pfac_num_patterns": (ctypes.c_uint32, [ctypes.c_void_p]),
    "pfac_max_len": (ctypes.c_uint32, [ctypes.c_void_p]),
    "pfac_table": (ctypes.c_void_p, [ctypes.c_void_p]),
    "pfac_prepare": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "pfac_packed_words": (ctypes.c_uint64, [ctypes.c_uint64]),
    "pfac_pack_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p]),
    "pfac_match_packed_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                               ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_match": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                  ctypes.c_void_p]),
    "pfac_match_checked": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_pack": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p]),
    "pfac_match_packed": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_set_text_kernel": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "pfac_plan_text": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]),
    "pfac_text_walk_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_uint32, ctypes.POINTER(ctypes.c_double),
                                            ctypes.POINTER(ctypes.c_double)]),
    "pfac_compact_workspace_bytes": (ctypes.c_uint64, [ctypes.c_uint64]),
    "pfac_compact_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint32,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_compact": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint32,
                                    ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_match_compact_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                                ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p]),
    "pfac_inv_words": (ctypes.c_uint64, [ctypes.c_uint64]),
    "pfac_pack_barriers_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_match_barriers_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                                 ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_match_compact_barriers_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                         ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                                                         ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                                         ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                                         ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_match_text_workspace_bytes": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]),
    "pfac_match_text_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_prefix_chain": (ctypes.c_void_p, [ctypes.c_void_p]),
    "pfac_expand_workspace_bytes": (ctypes.c_uint64, []),
    "pfac_expand_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_expand": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                   ctypes.c_void_p]),
    "pfac_match_list_workspace_bytes": (ctypes.c_uint64, [ctypes.c_uint64]),
    "pfac_match_list_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                             ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p]),
    "pfac_image_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "pfac_scan_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                      ctypes.c_void_p, ctypes.c_void_p]),
    "pfac_last_error": (ctypes.c_char_p, []),
}


def lib() -> ctypes.CDLL:
    """The loaded libpfac.so (built in-tree on first use if absent)."""
    global _lib
    if _lib is None:
        path = os.environ.get("PFAC_LIB") or _build.LIB  # PFAC_LIB: A/B experiments with another build
        if not os.path.exists(path):
            _build.build()
        L = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            try:
                f = getattr(L, name)
            except AttributeError:
                if os.environ.get("PFAC_LIB"):  # A/B runs may load an older build lacking newer entry points
                    continue
                raise
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class ImageInfo(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("cell_bytes", ctypes.c_uint32), ("K", ctypes.c_uint32),
                ("K2", ctypes.c_uint32), ("states", ctypes.c_uint32), ("window_rows", ctypes.c_uint32),
                ("all_smem", ctypes.c_uint32), ("short_pat", ctypes.c_uint32), ("smem_bytes", ctypes.c_uint64),
                ("l2_persist_bytes", ctypes.c_uint64), ("image_bytes", ctypes.c_uint64),
                ("text_kernel", ctypes.c_uint32), ("text_window_rows", ctypes.c_uint32),
                ("hr_rows", ctypes.c_uint32), ("hr_nb_rows", ctypes.c_uint32)]


class PfacError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"libpfac error {code}: {msg}")


def _check(rc: int) -> None:
    if rc != OK:
        raise PfacError(rc, lib().pfac_last_error().decode(errors="replace"))


def _ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream, device) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream


def _flatten(patterns) -> tuple[np.ndarray, np.ndarray]:
    pats = [p.encode() if isinstance(p, str) else bytes(p) for p in patterns]
    offs = np.zeros(len(pats) + 1, dtype=np.uint64)
    if pats:
        offs[1:] = np.cumsum([len(p) for p in pats])
    data = np.frombuffer(b"".join(pats), dtype=np.uint8).copy() if pats else np.zeros(1, np.uint8)
    return data, offs


def _host_bytes(text) -> np.ndarray:
    if isinstance(text, (bytes, bytearray)):
        return np.frombuffer(bytes(text), np.uint8)
    if hasattr(text, "numpy"):  # a CPU torch tensor
        return text.numpy().view(np.uint8).reshape(-1)
    return np.asarray(text, dtype=np.uint8).reshape(-1)


# pfac_set_text_kernel mode applied to every new Automaton when its text_kernel argument is None
# (None: the library's default, the plan's choice).  Tests switch it to cover every text path.
DEFAULT_TEXT_KERNEL = None


class Automaton:
    """pfac_build(patterns): the BFS-ordered automaton, finals numbered as pattern ids.
    text_kernel: pfac_set_text_kernel mode (-1 plan, 0 two kernels, 1 one kernel, 2 one kernel with
    1024-position slices, 3 the same with dynamically claimed slices); None = DEFAULT_TEXT_KERNEL."""

    def __init__(self, patterns, text_kernel=None):
        data, offs = _flatten(patterns)
        h = ctypes.c_void_p()
        _check(lib().pfac_build(data.ctypes.data, offs.ctypes.data, len(offs) - 1, ctypes.byref(h)))
        self._h = h
        mode = DEFAULT_TEXT_KERNEL if text_kernel is None else text_kernel
        if mode is not None:
            self.set_text_kernel(mode)

    def set_text_kernel(self, mode: int) -> None:
        """pfac_set_text_kernel: the path policy of match_text_async for this automaton."""
        _check(lib().pfac_set_text_kernel(self._h, int(mode)))

    def text_walk_stats(self, text, stride: int = 1, deep: int = 16) -> tuple[float, float]:
        """pfac_text_walk_stats on a host text (numpy uint8 / bytes / CPU tensor): (deep_frac,
        mean_steps) of the walks from every stride-th position."""
        t = np.ascontiguousarray(_host_bytes(text))
        df, ms = ctypes.c_double(), ctypes.c_double()
        _check(lib().pfac_text_walk_stats(self._h, t.ctypes.data if len(t) else None, len(t), int(stride), int(deep),
                                          ctypes.byref(df), ctypes.byref(ms)))
        return df.value, ms.value

    def plan_text(self, sample, stride: int = 1) -> tuple[int, float]:
        """pfac_plan_text: set the text-call path from a host text sample; returns (mode, deep_frac)."""
        t = np.ascontiguousarray(_host_bytes(sample))
        m, df = ctypes.c_int(), ctypes.c_double()
        _check(lib().pfac_plan_text(self._h, t.ctypes.data if len(t) else None, len(t), int(stride),
                                    ctypes.byref(m), ctypes.byref(df)))
        return m.value, df.value

    def close(self) -> None:
        if getattr(self, "_h", None) and _lib is not None:
            _lib.pfac_free(self._h)
            self._h = None

    __del__ = close

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    @property
    def num_states(self) -> int:
        return int(lib().pfac_num_states(self._h))

    @property
    def num_patterns(self) -> int:
        return int(lib().pfac_num_patterns(self._h))

    @property
    def max_len(self) -> int:
        return int(lib().pfac_max_len(self._h))

    def table(self) -> np.ndarray:
        """Canonical S x 4 table (columns A,C,G,T), copied out of the library."""
        S = self.num_states
        p = lib().pfac_table(self._h)
        return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint32)), shape=(S, 4)).copy()

    def prepare(self, device: int = 0) -> None:
        _check(lib().pfac_prepare(self._h, device))

    def prefix_chain(self) -> np.ndarray:
        """pfac_prefix_chain: (k+1) x 2 uint32 [longest proper-prefix pattern id, chain length]."""
        k = self.num_patterns
        p = lib().pfac_prefix_chain(self._h)
        return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint32)), shape=(k + 1, 2)).copy()

    def image_info(self, device: int = 0) -> dict:
        """pfac_image_info: the device image's layout facts (builds the image if needed)."""
        info = ImageInfo()
        _check(lib().pfac_image_info(self._h, device, ctypes.byref(info)))
        return {name: getattr(info, name) for name, _ in ImageInfo._fields_}


def packed_words(n: int) -> int:
    return int(lib().pfac_packed_words(n))


def compact_workspace_bytes(n: int) -> int:
    return int(lib().pfac_compact_workspace_bytes(n))


def pack_async(text, packed=None, first_bad=None, stream=None):
    """pfac_pack_async: uint8 CUDA tensor of n ASCII bases -> packed uint32 tensor."""
    import torch
    n = text.numel()
    if packed is None:
        packed = torch.empty(packed_words(n), dtype=torch.int32, device=text.device)
    _check(lib().pfac_pack_async(_ptr(text), n, _ptr(packed), _ptr(first_bad), _stream(stream, text.device)))
    return packed


def inv_words(n: int) -> int:
    return int(lib().pfac_inv_words(n))


def pack_barriers_async(text, packed=None, inv=None, first_bad=None, stream=None):
    """pfac_pack_barriers_async: packed uint32 words + per-word uint16 barrier masks (non-ACGT bytes)."""
    import torch
    n = text.numel()
    if packed is None:
        packed = torch.empty(packed_words(n), dtype=torch.int32, device=text.device)
    if inv is None:
        inv = torch.empty(inv_words(n), dtype=torch.int16, device=text.device)
    _check(lib().pfac_pack_barriers_async(_ptr(text), n, _ptr(packed), _ptr(inv), _ptr(first_bad),
                                          _stream(stream, text.device)))
    return packed, inv


def match_barriers_async(a: Automaton, packed, inv, n_own: int, n_avail: int | None = None, out=None, stream=None):
    """pfac_match_barriers_async: as match_packed_async, walks stop at barrier bytes."""
    import torch
    n_avail = n_own if n_avail is None else n_avail
    if out is None:
        out = torch.empty(n_own, dtype=torch.int32, device=packed.device)
    _check(lib().pfac_match_barriers_async(a.handle, _ptr(packed), _ptr(inv), n_own, n_avail, _ptr(out),
                                           _stream(stream, packed.device)))
    return out


def match_packed_async(a: Automaton, packed, n_own: int, n_avail: int | None = None, out=None, stream=None):
    """pfac_match_packed_async: out[i] for i < n_own, walks bounded by n_avail."""
    import torch
    n_avail = n_own if n_avail is None else n_avail
    if out is None:
        out = torch.empty(n_own, dtype=torch.int32, device=packed.device)
    _check(lib().pfac_match_packed_async(a.handle, _ptr(packed), n_own, n_avail, _ptr(out),
                                         _stream(stream, packed.device)))
    return out


def match(a: Automaton, text, out=None, stream=None):
    """pfac_match: ASCII CUDA tensor -> int32 out (returns after completion; non-ACGT bytes are barriers)."""
    import torch
    n = text.numel()
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=text.device)
    _check(lib().pfac_match(a.handle, _ptr(text), n, _ptr(out), _stream(stream, text.device)))
    return out


def match_checked(a: Automaton, text, out=None, stream=None):
    """pfac_match_checked: as match(), also returning the first non-ACGT index (-1 if none)."""
    import torch
    n = text.numel()
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=text.device)
    bad = ctypes.c_uint64(0)
    _check(lib().pfac_match_checked(a.handle, _ptr(text), n, _ptr(out), ctypes.byref(bad),
                                    _stream(stream, text.device)))
    return out, (-1 if bad.value == (1 << 64) - 1 else int(bad.value))


def pack(text, packed=None, stream=None):
    """pfac_pack (returns after completion): (packed, first_bad) with first_bad -1 if every byte is
    ACGTacgt.  A non-ACGT byte is not an error here: the library's PFAC_E_NON_ACGT is returned as
    first_bad >= 0 (the packed codes of such bytes are unspecified)."""
    import torch
    n = text.numel()
    if packed is None:
        packed = torch.empty(packed_words(n), dtype=torch.int32, device=text.device)
    bad = ctypes.c_uint64(0)
    rc = lib().pfac_pack(_ptr(text), n, _ptr(packed), ctypes.byref(bad), _stream(stream, text.device))
    if rc != E_NON_ACGT:
        _check(rc)
    return packed, (-1 if bad.value == (1 << 64) - 1 else int(bad.value))


def match_packed(a: Automaton, packed, n_own: int, n_avail: int | None = None, out=None, stream=None):
    """pfac_match_packed: as match_packed_async, returning after completion."""
    import torch
    n_avail = n_own if n_avail is None else n_avail
    if out is None:
        out = torch.empty(n_own, dtype=torch.int32, device=packed.device)
    _check(lib().pfac_match_packed(a.handle, _ptr(packed), n_own, n_avail, _ptr(out),
                                   _stream(stream, packed.device)))
    return out


def compact_async(out, pos, pid, count, workspace, pos_base: int = 0, k: int = 0, hist=None, stream=None):
    """pfac_compact_async into caller buffers (count: 1-element int64 CUDA tensor)."""
    _check(lib().pfac_compact_async(_ptr(out), out.numel(), pos_base, _ptr(pos), _ptr(pid), pos.numel(),
                                    _ptr(count), k, _ptr(hist), _ptr(workspace), _stream(stream, out.device)))


def match_compact_async(a: Automaton, packed, n_own: int, n_avail: int, out, pos, pid, count, workspace,
                        pos_base: int = 0, hist=None, stream=None, inv=None):
    """pfac_match_compact_async: fused match + ordered match list (count: 1-element int64 CUDA tensor).
    inv: barrier masks from pack_barriers_async (pfac_match_compact_barriers_async)."""
    if inv is not None:
        _check(lib().pfac_match_compact_barriers_async(a.handle, _ptr(packed), _ptr(inv), n_own, n_avail, _ptr(out),
                                                       pos_base, _ptr(pos), _ptr(pid), pos.numel(), _ptr(count),
                                                       _ptr(hist), _ptr(workspace), _stream(stream, out.device)))
        return
    _check(lib().pfac_match_compact_async(a.handle, _ptr(packed), n_own, n_avail, _ptr(out), pos_base, _ptr(pos),
                                          _ptr(pid), pos.numel(), _ptr(count), _ptr(hist), _ptr(workspace),
                                          _stream(stream, out.device)))


def scan_host(a: Automaton, text, pos=None, pid=None, device: int = 0, n_own: int | None = None,
              pos_base: int = 0):
    """pfac_scan_host: the match list of a HOST text (CPU uint8 tensor or numpy array), end to end.

    Positions [0, n_own) are matched (default: all), walks read the whole text (a shard + halo).
    pos/pid: optional preallocated CPU int64/int32 tensors (pinned for fast copies); the call retries
    once with exact-size buffers if they are too small.  Returns (pos, pid, count)."""
    import torch
    t = torch.as_tensor(text) if not isinstance(text, torch.Tensor) else text
    assert t.device.type == "cpu" and t.dtype == torch.uint8 and t.is_contiguous()
    n_avail = t.numel()
    n = n_avail if n_own is None else n_own
    if pos is None:
        cap = n // 64 + 1024
        pos = torch.empty(cap, dtype=torch.int64)
        pid = torch.empty(cap, dtype=torch.int32)
    c = ctypes.c_uint64(0)
    bad = ctypes.c_uint64(0)
    rc = lib().pfac_scan_host(a.handle, device, t.data_ptr(), n, n_avail, pos_base, pos.data_ptr(), pid.data_ptr(),
                              pos.numel(), ctypes.byref(c), ctypes.byref(bad))
    if rc == E_CAPACITY:
        pos = torch.empty(int(c.value), dtype=torch.int64)
        pid = torch.empty(int(c.value), dtype=torch.int32)
        rc = lib().pfac_scan_host(a.handle, device, t.data_ptr(), n, n_avail, pos_base, pos.data_ptr(),
                                  pid.data_ptr(), pos.numel(), ctypes.byref(c), ctypes.byref(bad))
    _check(rc)
    m = int(c.value)
    return pos[:m], pid[:m], m


def compact(out, pos_base: int = 0, capacity: int | None = None, k: int = 0, hist=None, stream=None):
    """pfac_compact: returns (pos int64, pid int32, count) trimmed to count (synchronous)."""
    import torch
    n = out.numel()
    cap = max(1024, n // 256) if capacity is None else capacity
    while True:
        pos = torch.empty(max(cap, 1), dtype=torch.int64, device=out.device)
        pid = torch.empty(max(cap, 1), dtype=torch.int32, device=out.device)
        c = ctypes.c_uint64(0)
        rc = lib().pfac_compact(_ptr(out), n, pos_base, _ptr(pos), _ptr(pid), cap, ctypes.byref(c), k,
                                _ptr(hist), _stream(stream, out.device))
        if rc == E_CAPACITY and capacity is None:
            cap = int(c.value)
            if hist is not None:
                raise PfacError(rc, "capacity too small with an accumulating histogram; pass capacity")
            continue
        _check(rc)
        m = int(c.value)
        return pos[:m], pid[:m], m


def expand_workspace_bytes() -> int:
    return int(lib().pfac_expand_workspace_bytes())


def expand_async(a: Automaton, pos, pid, count, pos_all, pid_all, count_all, workspace, stream=None):
    """pfac_expand_async: every occurrence from the longest-only list (count/count_all: 1-element int64
    CUDA tensors; the input is the first min(count, pos.numel()) entries)."""
    _check(lib().pfac_expand_async(a.handle, _ptr(pos), _ptr(pid), _ptr(count), pos.numel(), _ptr(pos_all),
                                   _ptr(pid_all), pos_all.numel(), _ptr(count_all), _ptr(workspace),
                                   _stream(stream, count_all.device)))


def expand(a: Automaton, pos, pid, capacity: int | None = None, stream=None):
    """pfac_expand: (pos_all int64, pid_all int32, total) trimmed to total (synchronous)."""
    import torch
    m = pos.numel()
    cap = max(1024, 2 * m) if capacity is None else capacity
    while True:
        pa = torch.empty(max(cap, 1), dtype=torch.int64, device=pos.device)
        pi = torch.empty(max(cap, 1), dtype=torch.int32, device=pos.device)
        c = ctypes.c_uint64(0)
        rc = lib().pfac_expand(a.handle, _ptr(pos), _ptr(pid), m, _ptr(pa), _ptr(pi), cap, ctypes.byref(c),
                               _stream(stream, pos.device))
        if rc == E_CAPACITY and capacity is None:
            cap = int(c.value)
            continue
        _check(rc)
        t = int(c.value)
        return pa[:t], pi[:t], t


def match_list_workspace_bytes(n_own: int) -> int:
    return int(lib().pfac_match_list_workspace_bytes(n_own))


def match_list_async(a: Automaton, packed, n_own: int, n_avail: int, pos, pid, count, workspace, pos_base: int = 0,
                     hist=None, inv=None, stream=None):
    """pfac_match_list_async: the ordered match list without the dense out[] (count: 1-element int64 CUDA
    tensor; workspace: match_list_workspace_bytes(n_own) bytes)."""
    _check(lib().pfac_match_list_async(a.handle, _ptr(packed), _ptr(inv), n_own, n_avail, pos_base, _ptr(pos),
                                       _ptr(pid), pos.numel(), _ptr(count), _ptr(hist), _ptr(workspace),
                                       _stream(stream, count.device)))


def match_text_workspace_bytes(n_own: int, n_avail: int | None = None, list_only: bool = False) -> int:
    return int(lib().pfac_match_text_workspace_bytes(n_own, n_own if n_avail is None else n_avail, int(list_only)))


def match_text_async(a: Automaton, text, n_own: int, n_avail: int, out, pos, pid, count, workspace,
                     pos_base: int = 0, hist=None, first_bad=None, stream=None):
    """pfac_match_text_async: pack + match + ordered match list from the ASCII text in one kernel.
    out=None: list only.  count / first_bad: 1-element int64 CUDA tensors; workspace:
    match_text_workspace_bytes(n_own, n_avail, out is None) bytes."""
    _check(lib().pfac_match_text_async(a.handle, _ptr(text), n_own, n_avail, _ptr(out), pos_base, _ptr(pos),
                                       _ptr(pid), pos.numel(), _ptr(count), _ptr(hist), _ptr(first_bad),
                                       _ptr(workspace), _stream(stream, count.device)))
