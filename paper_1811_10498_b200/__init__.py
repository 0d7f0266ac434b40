"""B200-native (sm_100a) hot path of Parallel Failure-less Aho-Corasick for DNA (arxiv 1811.10498).

Public Python surface = the C-ABI of include/pfac.h with the same names (see binding.py):
``Automaton`` (pfac_build), ``pack`` / ``pack_async``, ``match_packed`` / ``match_packed_async``,
``match`` / ``match_checked``, ``compact_async``,
``compact``, ``match_compact_async`` (fused), ``scan_host`` (end to end over host memory), and the
barrier variants ``pack_barriers_async`` / ``match_barriers_async`` (bytes outside ACGT stop walks,
DESIGN.md reading R5), ``expand`` / ``expand_async`` (every occurrence from the longest-only list) and ``match_list_async``
(the list without the dense out[]), ``match_text_async`` (pack + match + list from the ASCII text in one
kernel); ``parallel`` holds the multi-GPU text sharding + NCCL gather.
"""
from .binding import (Automaton, PfacError, compact, compact_async, compact_workspace_bytes, expand, expand_async,
                      expand_workspace_bytes, inv_words, lib, match, match_checked, match_list_async, match_list_workspace_bytes,
                      match_barriers_async, match_compact_async, match_packed, match_packed_async, match_text_async,
                      match_text_workspace_bytes, pack, pack_async, pack_barriers_async, packed_words, scan_host)

__all__ = ["Automaton", "PfacError", "compact", "compact_async", "compact_workspace_bytes", "expand", "expand_async",
           "expand_workspace_bytes", "inv_words", "lib", "match_list_async", "match_list_workspace_bytes",
           "match", "match_checked", "match_barriers_async", "match_compact_async", "match_packed",
           "match_packed_async", "match_text_async", "match_text_workspace_bytes", "pack", "pack_async",
           "pack_barriers_async", "packed_words", "scan_host"]
