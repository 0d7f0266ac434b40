"""B200-native (sm_100a) hot path of Parallel Failure-less Aho-Corasick for DNA (arxiv 1811.10498).

Public Python surface = the C-ABI of include/pfac.h with the same names (see binding.py):
``Automaton`` (pfac_build), ``pack_async``, ``match_packed_async``, ``match``, ``compact_async``,
``compact``, ``match_compact_async`` (fused), ``scan_host`` (end to end over host memory); ``parallel`` holds the multi-GPU text sharding + NCCL gather.
"""
from .binding import (Automaton, PfacError, compact, compact_async, compact_workspace_bytes, lib, match,
                      match_compact_async, match_packed_async, pack_async, packed_words, scan_host)

__all__ = ["Automaton", "PfacError", "compact", "compact_async", "compact_workspace_bytes", "lib", "match",
           "match_compact_async", "match_packed_async", "pack_async", "packed_words", "scan_host"]
