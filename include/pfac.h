/*
 * pfac.h -- C-ABI of libpfac, the B200 (sm_100a) hot path of Parallel Failure-less Aho-Corasick
 * (PFAC) for DNA (Thambawita, Ragel, Elkaduwe, arxiv 1811.10498; cited as PAPER.md:<line>).
 *
 * The method (PAPER.md:91-93, Sec. IV; :204, Sec. V-B): every text position i starts its own walk
 * of the failure-less goto automaton of the patterns over {A,C,G,T}; the walk stops at the first
 * missing transition; out[i] is the id of the last pattern completed on the way, i.e. the id of
 * the LONGEST pattern p with text[i .. i+|p|) = p ("PFAC can detect only the longest patterns"),
 * or 0 if no pattern starts at i.  Pattern ids are 1-based in input order (Table 1 cell "6,1",
 * PAPER.md:135).
 *
 * Conventions for every entry point:
 *  - No call throws across the ABI or aborts; each returns PFAC_OK or a negative PFAC_E_* code
 *    and pfac_last_error() then returns a thread-local message.
 *  - "d_" pointers are CUDA device pointers owned by the caller (e.g. torch tensors).  The device
 *    a call runs on is the one that owns its device buffers (found with cudaPointerGetAttributes),
 *    independent of any runtime's "current device"; every call restores the calling thread's
 *    current device before it returns.
 *  - `stream` is a cudaStream_t (CUstream) of that device, passed as void* so that this header
 *    needs no CUDA include (the same pointer-sized handle; reading R18).  "_async" calls
 *    only enqueue work on `stream`; the other compute calls return after completion (they
 *    synchronise `stream`).
 *  - L2 side effect: the first use of an automaton with a second-level jump table on a device
 *    raises that device's cudaLimitPersistingL2CacheSize to the table's size (J2 + chain-head rows,
 *    <= ~24 MiB; never lowered), and match launches mark that window persisting.  Co-resident
 *    kernels of the same process see that much less normal L2; cudaCtxResetPersistingL2Cache
 *    releases the lines.
 *  - Bases are the bytes A,C,G,T,a,c,g,t (case-insensitive; reading R4).
 */
#ifndef PFAC_H
#define PFAC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pfac_automaton pfac_automaton; /* opaque; immutable after pfac_build */

enum {
    PFAC_OK = 0,
    PFAC_E_ARG = -1,             /* bad argument (null, misaligned, n_avail < n_own, ...) */
    PFAC_E_EMPTY_PATTERN = -2,   /* a pattern of length 0 (reading R3) */
    PFAC_E_NON_ACGT = -3,        /* a pattern or text byte outside ACGTacgt (reading R5) */
    PFAC_E_DUPLICATE = -4,       /* two equal patterns (reading R2) */
    PFAC_E_TOO_LONG = -5,        /* a pattern longer than PFAC_MAX_LEN (reading R13) */
    PFAC_E_TOO_MANY_STATES = -6, /* automaton would need >= 2^31 states */
    PFAC_E_CAPACITY = -7,        /* compaction output larger than the caller's capacity */
    PFAC_E_CUDA = -8,            /* a CUDA runtime error (message in pfac_last_error) */
    PFAC_E_OOM = -9              /* host or device allocation failed */
};

#define PFAC_MAX_LEN 1024u

/* ------------------------------------------------------------------------------------------
 * Build (host only).  PAPER.md:120 (4 x N table over A,T,C,G), :147-149 (patterns loaded one
 * by one, a new state per new character), Table 1.
 *
 * Pattern j (id j+1) is bytes[offsets[j] .. offsets[j+1]), j < k; `offsets` has k+1 entries.
 * On success *out owns a new automaton (free with pfac_free).  Errors, checked before any work
 * that could allocate device memory: PFAC_E_EMPTY_PATTERN, PFAC_E_NON_ACGT, PFAC_E_TOO_LONG,
 * PFAC_E_DUPLICATE (message names both ids), PFAC_E_TOO_MANY_STATES, PFAC_E_ARG (null pointers
 * with k > 0).  k = 0 is allowed (every out[i] is 0).
 *
 * Canonical numbering (the exported table): state 0 is the root; the state completing pattern p
 * has number p (1..k); all other states get k+1, k+2, ... in breadth-first order with children
 * visited in column order A, C, G, T.  (The paper's column order is A,T,C,G; the
 * export uses A,C,G,T -- DESIGN.md reading R9.)
 */
int pfac_build(const uint8_t *bytes, const uint64_t *offsets, uint32_t k, pfac_automaton **out);

/* Frees the host tables and every device image of `a` (null is a no-op). */
void pfac_free(pfac_automaton *a);

/* Inspection (host memory owned by `a`, valid until pfac_free). */
uint32_t pfac_num_states(const pfac_automaton *a);   /* S: states including the root */
uint32_t pfac_num_patterns(const pfac_automaton *a); /* k */
uint32_t pfac_max_len(const pfac_automaton *a);      /* longest pattern; walks read <= this */
/* Canonical transition table, S*4 uint32 row-major, columns A,C,G,T; cell = next state, 0 = no
 * transition (the root is nobody's child, so 0 is unambiguous -- the paper's "0,0" cells). */
const uint32_t *pfac_table(const pfac_automaton *a);

/* Build and upload the device image of `a` for CUDA device `device` now (otherwise it is built
 * lazily by the first match on that device).  Returns PFAC_E_CUDA / PFAC_E_OOM on failure. */
int pfac_prepare(const pfac_automaton *a, int device);

/* ------------------------------------------------------------------------------------------
 * Pack (step 3 of SURVEY.md Sec. 8(a)): ASCII bases -> 2-bit codes A=0,C=1,G=2,T=3, 16 bases per
 * uint32, base j in bits 2*(j mod 16) of word j/16.  d_packed must hold pfac_packed_words(n)
 * uint32 (a multiple of 4 words; padding words are written as 0) and be 16-byte aligned.
 * d_first_bad (device, nullable) receives the smallest index of a byte outside ACGTacgt, or
 * UINT64_MAX if there is none; codes of such bytes are unspecified.  Asynchronous.
 */
uint64_t pfac_packed_words(uint64_t n);
/* pfac_pack: the same, returning after completion.  first_bad (HOST, nullable)
 * receives the first non-ACGTacgt index or UINT64_MAX; such a byte makes the call return
 * PFAC_E_NON_ACGT (d_packed is still fully written; the codes of those bytes are unspecified). */
int pfac_pack(const uint8_t *d_text, uint64_t n, uint32_t *d_packed, uint64_t *first_bad, void *stream);
int pfac_pack_async(const uint8_t *d_text, uint64_t n, uint32_t *d_packed, uint64_t *d_first_bad,
                    void *stream);

/* Pack + barrier map (reading R5): as pfac_pack_async, and
 * d_inv[w] bit j (j < 16) is set iff text byte 16*w + j is outside ACGTacgt -- a barrier: no walk
 * crosses it and no pattern occurrence contains it (PAPER.md:91 with SPEC.md:143's reading).
 * d_inv holds pfac_inv_words(n) uint16 (a multiple of 8, 16-byte aligned; padding words are 0).
 * Asynchronous. */
uint64_t pfac_inv_words(uint64_t n);
int pfac_pack_barriers_async(const uint8_t *d_text, uint64_t n, uint32_t *d_packed,
                             uint16_t *d_inv, uint64_t *d_first_bad, void *stream);

/* ------------------------------------------------------------------------------------------
 * Match (step 4): for every i in [0, n_own): out[i] = id of the longest pattern starting at i
 * whose bases all lie in [0, n_avail) of the packed text, else 0.  n_avail >= n_own
 * lets a shard see a halo of (max_len - 1) bases past its owned range (reading R6).
 * d_packed: as written by pfac_pack_async for n_avail bases (16-byte aligned, padded);
 * d_out: n_own int32, 16-byte aligned.  Asynchronous.
 */
int pfac_match_packed_async(const pfac_automaton *a, const uint32_t *d_packed, uint64_t n_own,
                            uint64_t n_avail, int32_t *d_out, void *stream);
/* The same, returning after completion (SURVEY.md Sec. 8(b) shard form). */
int pfac_match_packed(const pfac_automaton *a, const uint32_t *d_packed, uint64_t n_own,
                      uint64_t n_avail, int32_t *d_out, void *stream);

/* Match with barriers: as pfac_match_packed_async, and walks stop at every byte whose d_inv bit is
 * set (d_inv as written by pfac_pack_barriers_async for n_avail bases), so out[i] = 0 where text
 * byte i is a barrier and no reported occurrence contains one.  The barrier kernel is an
 * instantiation of the filter path; an image without the filter (built with PFAC_FB16=0) returns
 * PFAC_E_CUDA ("operation not supported").  Asynchronous. */
int pfac_match_barriers_async(const pfac_automaton *a, const uint32_t *d_packed,
                              const uint16_t *d_inv, uint64_t n_own, uint64_t n_avail,
                              int32_t *d_out, void *stream);

/* pfac_match (one walk per character into an integer array):
 * pack + match over one ASCII text of n bytes on the device (d_text: n bytes, any alignment; d_out:
 * n int32, 16-byte aligned).  Bytes outside ACGTacgt are barriers (reading R5): the call packs with
 * the barrier map, and only when the text holds such a byte runs the barrier kernel.  Returns after
 * completion.  PFAC_E_NON_ACGT only if the text has a barrier and the image has no filter
 * (PFAC_FB16=0 ablation builds). */
int pfac_match(const pfac_automaton *a, const uint8_t *d_text, uint64_t n, int32_t *d_out,
               void *stream);
/* pfac_match that also reports the first barrier: *first_bad (HOST, nullable) receives the index
 * of the first byte outside ACGTacgt, or UINT64_MAX.  Returns after completion. */
int pfac_match_checked(const pfac_automaton *a, const uint8_t *d_text, uint64_t n, int32_t *d_out,
                       uint64_t *first_bad, void *stream);

/* ------------------------------------------------------------------------------------------
 * Compact (step 5): the match list {(pos_base + i, out[i]) : out[i] != 0} in ascending i.
 * d_pos (uint64) / d_pid (uint32) receive the first min(count, capacity) entries; *count is the
 * total.  d_hist (device, nullable): k+1 uint64 per-pattern counters, ACCUMULATED (+=) so shards
 * and ranks can be summed; values out[i] > k are counted nowhere.
 * pfac_compact_async: d_count is a device uint64; d_workspace holds
 * pfac_compact_workspace_bytes(n) bytes (any content; reset by the call).  Asynchronous.
 * pfac_compact: *count is host memory; returns PFAC_E_CAPACITY if count > capacity (the first
 * `capacity` entries are still written).  Synchronous.
 */
uint64_t pfac_compact_workspace_bytes(uint64_t n);
int pfac_compact_async(const int32_t *d_out, uint64_t n, uint64_t pos_base, uint64_t *d_pos,
                       uint32_t *d_pid, uint64_t capacity, uint64_t *d_count, uint32_t k,
                       uint64_t *d_hist, void *d_workspace, void *stream);
int pfac_compact(const int32_t *d_out, uint64_t n, uint64_t pos_base, uint64_t *d_pos,
                 uint32_t *d_pid, uint64_t capacity, uint64_t *count, uint32_t k, uint64_t *d_hist,
                 void *stream);

/* ------------------------------------------------------------------------------------------
 * Fused match + compact: one pass that writes out[0..n_own) exactly as
 * pfac_match_packed_async and the match list exactly as pfac_compact_async(d_out, n_own, pos_base,
 * ...) would, without re-reading out[].  Same buffer rules as those two calls; d_workspace holds
 * pfac_compact_workspace_bytes(n_own) bytes; the histogram uses k = pfac_num_patterns(a).
 * Asynchronous (a cooperative launch: every CTA of the grid is resident at once).
 */
int pfac_match_compact_async(const pfac_automaton *a, const uint32_t *d_packed, uint64_t n_own,
                             uint64_t n_avail, int32_t *d_out, uint64_t pos_base, uint64_t *d_pos,
                             uint32_t *d_pid, uint64_t capacity, uint64_t *d_count, uint64_t *d_hist,
                             void *d_workspace, void *stream);
/* The same with barriers (d_inv as for pfac_match_barriers_async; null = no barriers). */
int pfac_match_compact_barriers_async(const pfac_automaton *a, const uint32_t *d_packed,
                                      const uint16_t *d_inv, uint64_t n_own, uint64_t n_avail,
                                      int32_t *d_out, uint64_t pos_base, uint64_t *d_pos,
                                      uint32_t *d_pid, uint64_t capacity, uint64_t *d_count,
                                      uint64_t *d_hist, void *d_workspace, void *stream);

/* ------------------------------------------------------------------------------------------
 * List-only match (second half): the match list of
 * pfac_match_compact_async without the dense out[] array -- the paper's output is the dense array
 * (PAPER.md:207); when only the occurrences are wanted, skipping it cuts the kernel's HBM traffic
 * from 4.25 to ~0.25 B/base (+12 B per match).  d_inv: barrier masks as for
 * pfac_match_barriers_async, or null.  d_workspace holds pfac_match_list_workspace_bytes(n_own)
 * bytes, 16-byte aligned (any content; it includes an n_own-int32 scratch written only at match
 * positions).  Images without the filter (PFAC_FB16=0 builds) return PFAC_E_CUDA.  Asynchronous
 * (a cooperative launch).
 */
uint64_t pfac_match_list_workspace_bytes(uint64_t n_own);
int pfac_match_list_async(const pfac_automaton *a, const uint32_t *d_packed, const uint16_t *d_inv,
                          uint64_t n_own, uint64_t n_avail, uint64_t pos_base, uint64_t *d_pos,
                          uint32_t *d_pid, uint64_t capacity, uint64_t *d_count, uint64_t *d_hist,
                          void *d_workspace, void *stream);

/* ------------------------------------------------------------------------------------------
 * Match from the ASCII text in one kernel (pack fused into the match + compact kernel): the same
 * results as pfac_pack_barriers_async -> pfac_match_compact_barriers_async (or, d_out == NULL, ->
 * pfac_match_list_async) on d_text[0..n_avail), positions [0, n_own), without the packed and
 * barrier-mask arrays in HBM.  Definition: out[i] = id of the longest pattern starting at i
 * (PAPER.md:91, :204-207); bytes outside ACGTacgt are barriers (reading R5).
 *   d_text     device, n_avail bytes (16-byte aligned for the one-kernel path; otherwise, when
 *              the automaton's halo is too long for its shared-memory plan (max_len > ~112), or
 *              when the plan prefers it (pfac_image_info().text_kernel; pfac_set_text_kernel
 *              overrides the plan), the call runs pack -> fused kernel through buffers in
 *              d_workspace -- same results)
 *   d_out      device int32[n_own], 16-byte aligned, or NULL: list only (no dense out[])
 *   d_pos/d_pid/capacity/d_count/d_hist/pos_base: as pfac_match_compact_async
 *   d_first_bad (nullable, device uint64): pos_base + the first owned index (< n_own) whose byte
 *              is not ACGTacgt, or UINT64_MAX
 *   d_workspace: pfac_match_text_workspace_bytes(n_own, n_avail, d_out == NULL) bytes, 16-byte
 *              aligned, any content.
 * Errors: PFAC_E_ARG (null / misaligned / n_avail < n_own), PFAC_E_CUDA (launch; images built
 * without the filter, PFAC_FB16=0).  Asynchronous (a cooperative launch); a list longer than
 * capacity is reported through *d_count > capacity (read it after a sync).
 */
uint64_t pfac_match_text_workspace_bytes(uint64_t n_own, uint64_t n_avail, int list_only);
/* Path policy of pfac_match_text_async for automaton `a` (all devices): mode -1 = the plan's
 * measured choice (default), 0 = always pack -> fused kernel, 1 = the one-kernel path whenever it
 * fits (2048-position slices first), 2 = its 1024-position-slice form whenever it fits, 3 = that
 * form with the slices claimed dynamically by the warps (a global counter) instead of a fixed run
 * per warp, the matches placed after a scan of per-slice counts at the end (load balance for text
 * whose per-slice walk work varies widely).  Results are identical in every mode; only the kernels
 * differ.  PFAC_E_ARG for other modes or a null a.
 * The one mutable property of an automaton (an atomic; safe to change between calls). */
int pfac_set_text_kernel(pfac_automaton *a, int mode);
/* A cheap statistic of a text for that policy (host memory, host code, no device work): the PFAC
 * walk (goto function only; a byte outside ACGTacgt has no transition, reading R5)
 * from positions 0, stride, 2*stride, ... < n of h_text, counting transitions.  *deep_frac = share
 * of the sampled walks with >= deep transitions, *mean_steps = mean transitions per sampled walk.
 * Repetitive text against nested patterns (long walks) shows a large deep_frac; random text a tiny
 * one.  PFAC_E_ARG for null pointers (h_text may be null when n = 0) or stride = 0. */
int pfac_text_walk_stats(const pfac_automaton *a, const uint8_t *h_text, uint64_t n, uint64_t stride,
                         uint32_t deep, double *deep_frac, double *mean_steps);
/* The text-call path from a text sample (host memory; host code, no device work): the walk statistic
 * above (deep = 16, every stride-th position) decides -- walk-heavy text (>= 1% of the sampled walks
 * make 16 or more transitions: repetitive text against nested patterns) takes the 1024-position-slice
 * text kernel with dynamically claimed slices (mode 3): its smaller per-warp staging leaves shared
 * memory for a row window and L1 room for rows, and claiming balances the widely varying per-slice
 * walk work (measured on cfg5: 3.10 ms vs 3.54 ms with a fixed run per warp (mode 2), 3.96 ms with
 * 2048-position slices); other text keeps the automaton's plan (mode -1: on such text mode 3's
 * interleaved out[] write streams cost cfg2 +40%, cfg4 +26%).  Applies the mode with
 * pfac_set_text_kernel and returns it in *mode (nullable), the statistic in *deep_frac (nullable).
 * Errors as pfac_text_walk_stats. */
int pfac_plan_text(pfac_automaton *a, const uint8_t *h_sample, uint64_t n, uint64_t stride, int *mode,
                   double *deep_frac);
int pfac_match_text_async(const pfac_automaton *a, const uint8_t *d_text, uint64_t n_own, uint64_t n_avail,
                          int32_t *d_out, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                          uint64_t capacity, uint64_t *d_count, uint64_t *d_hist, uint64_t *d_first_bad,
                          void *d_workspace, void *stream);

/* ------------------------------------------------------------------------------------------
 * End to end over HOST memory (the call a user with a text in RAM makes): the match list
 * {(pos_base + i, out[i]) : out[i] != 0, i < n_own} of the ASCII text h_text[0..n_avail) (walks
 * read up to n_avail >= n_own: a shard and its halo) on CUDA device `device`.  The text is streamed
 * in chunks with a (max_len - 1)-base halo: the host-to-device copy of chunk c+1 runs on one stream
 * while chunk c goes through the text call (pfac_match_text_async: pack + match + compact in one
 * kernel where the plan takes it) on another, and each chunk's list is copied back into h_pos/h_pid
 * at its offset.  Pinned h_text gives copy/compute overlap; pageable memory works too.  Bytes
 * outside ACGTacgt are barriers (reading R5).  *first_bad (nullable) receives the index (relative to
 * h_text) of the first such byte at a position < n_own, or UINT64_MAX.  Returns PFAC_E_CAPACITY if
 * count > capacity (the first `capacity` entries are written and *count is the total); PFAC_E_CUDA
 * for images without the filter (PFAC_FB16=0 ablation builds).  Synchronous.
 */
int pfac_scan_host(const pfac_automaton *a, int device, const uint8_t *h_text, uint64_t n_own,
                   uint64_t n_avail, uint64_t pos_base, uint64_t *h_pos, uint32_t *h_pid,
                   uint64_t capacity, uint64_t *count, uint64_t *first_bad);

/* ------------------------------------------------------------------------------------------
 * All occurrences: the set the serial Aho-Corasick machine reports
 * (PAPER.md:77, :87), from PFAC's longest-only list.  Every pattern occurring at i is a prefix of
 * the longest one there, so the set is {(i, q) : (i, p) in the list, q on the prefix chain of p}.
 * pfac_prefix_chain(a): host array of 2*(k+1) uint32 owned by `a`: [2p] = id of the longest pattern
 * that is a proper prefix of pattern p (0 = none), [2p+1] = length of p's chain (p included);
 * entries for p = 0 are 0.
 * pfac_expand_async: reads m = min(*d_count, in_capacity) entries (d_pos uint64 / d_pid uint32,
 * e.g. pfac_compact_async's output with its d_count) and writes the occurrences in ascending
 * position and, at one position, ascending pattern length: the first min(total, capacity) into
 * d_pos_all / d_pid_all, the total into *d_count_all (device).  pid values 0 or > k contribute
 * nothing.  d_workspace holds pfac_expand_workspace_bytes() bytes (reset by the call).
 * Asynchronous (a cooperative launch).
 * pfac_expand: `count` input entries (host value), *count_all on the host; PFAC_E_CAPACITY if the
 * total exceeds capacity (the first `capacity` entries are written).  Synchronous.
 */
const uint32_t *pfac_prefix_chain(const pfac_automaton *a);
uint64_t pfac_expand_workspace_bytes(void);
int pfac_expand_async(const pfac_automaton *a, const uint64_t *d_pos, const uint32_t *d_pid,
                      const uint64_t *d_count, uint64_t in_capacity, uint64_t *d_pos_all,
                      uint32_t *d_pid_all, uint64_t capacity, uint64_t *d_count_all,
                      void *d_workspace, void *stream);
int pfac_expand(const pfac_automaton *a, const uint64_t *d_pos, const uint32_t *d_pid,
                uint64_t count, uint64_t *d_pos_all, uint32_t *d_pid_all, uint64_t capacity,
                uint64_t *count_all, void *stream);

/* Device image facts for reports and tests; builds the image if needed. */
typedef struct {
    int32_t device;
    uint32_t cell_bytes;      /* 2 (uint16 image) or 4 */
    uint32_t K;               /* jump-table length (J has 4^K cells, in shared memory) */
    uint32_t K2;              /* second-level jump length (0 = none; J2 in L2-persisting memory) */
    uint32_t states;          /* S */
    uint32_t window_rows;     /* device states whose row is staged in shared memory */
    uint32_t all_smem;        /* 1 if every row fits */
    uint32_t short_pat;       /* a pattern shorter than the jump length exists */
    uint64_t smem_bytes;      /* dynamic shared memory per CTA of the match kernel */
    uint64_t l2_persist_bytes;/* access-policy window over J2 + the chain-head rows HR */
    uint64_t image_bytes;     /* device memory of the image (all tables, HR and prefix chains) */
    uint32_t text_kernel;     /* pfac_match_text_async on aligned text: 0 = pack + fused kernel,
                                 1 = one kernel, 2 = one kernel with 1024-position slices,
                                 3 = that kernel with dynamically claimed slices */
    uint32_t text_window_rows;/* rows staged in shared memory by that kernel */
    uint32_t hr_rows;         /* chain-head row copies next to J2 (uint32 images; 0 = none) */
    uint32_t hr_nb_rows;      /* of which NOFIN chains whose J2 entry carries their first 4 bases
                                 (a walk that differs there answers 0 without loading the row) */
} pfac_image_info_t;
int pfac_image_info(const pfac_automaton *a, int device, pfac_image_info_t *out);

/* Thread-local message for the last non-OK return on this thread ("" if none). */
const char *pfac_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PFAC_H */
