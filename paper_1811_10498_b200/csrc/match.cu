// Match kernel: out[i] = id of the longest pattern starting at i.
// The walk itself is PAPER.md:91-93 / :204: follow the goto function from the start state, stop at
// the first missing transition; the answer is the deepest final state passed (F).
//
// Layout and schedule (every constant below was chosen by an A/B measurement, the
// PFAC_* macros are the knobs):
//  * One persistent CTA of 896 threads per SM.  Shared memory holds the first-level table -- the
//    4^10-bit filter FB (default) or the jump table J (4^K cells) -- the first W rows of the device
//    transition table T and of F (all of them when they fit), and per warp a double-buffered text
//    slice (2048 bases + a halo of >= maxlen bases) that the warp's lane 0 fetches with a TMA bulk
//    copy (cp.async.bulk + mbarrier).
//  * Each warp owns a contiguous run of slices.  Lane l handles 8 consecutive positions of each
//    256-position sub-slice: one 64-bit text window gives the eight 10-mers, one filter bit each.
//    Unflagged positions answer 0; the zeros are stored right away with two coalesced 16-byte stores
//    per lane.  (J variant: one J lookup per position answers every walk that dies within K bases.)
//  * Flagged positions go into a warp-private queue (one ballot per round gives each lane its slot)
//    and are resolved 32 at a time, one per lane: one L2 load of J2 (the K2-mer jump table, in an
//    L2-persisting access-policy window) answers the first K2 = 10-11 bases; the few walks still alive
//    continue over T rows.  Unary runs of the trie are "chain rows" that advance over up to 16 forced
//    bases with one XOR.  Results patch out[] after a __syncwarp.
//  * FUSE (pfac_match_compact_async): nonzero results also set bits in a per-slice match bitmap; at
//    the end of each slice the warp stages its matches in position order, and a grid-wide count
//    prefix (cooperative launch) places every warp's list.
//  * TXT (pfac_match_text_async): the same fused kernel reading the ASCII text itself -- the pack step
//     moves into the kernel.  Each warp's lane 0 fetches the slice's ASCII
//    bytes (+ halo) by TMA into a shared staging buffer; the warp packs them into its 2-bit slice
//    buffer and the barrier bits (reading R5) in shared memory, then lane 0 prefetches the next
//    slice's bytes while the warp matches this one.  Slices with a non-ACGT byte take the barrier
//    path.  HBM traffic per base: 1 B of ASCII read + 4 B of out[] written (vs 1.25 + 4.25 split).
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "compact_common.cuh"
#include "pack_common.cuh"
#include "pfac_internal.h"
#include "ptx.cuh"

namespace pfac {

#ifndef PFAC_MT
#define PFAC_MT 896
#endif
// Ablation knobs (report-only builds, scripts/ablations.sh):
//   PFAC_TEXT_DIRECT=1: the walk reads the packed text straight from global memory (L1/L2) instead
//     of the per-warp TMA-staged shared-memory slices (the paper's "text in shared memory" question,
//     PAPER.md:327-330).  Reads may touch up to 16 bytes past the packed buffer (the bench's caching
//     allocator rounds allocations up), so it is not a product setting.
//   PFAC_WINDOW_MAX=W: at most W transition-table rows staged in shared memory (0: every row through
//     L2 with ld.global.nc -- the paper's table-in-texture/global question).
#ifndef PFAC_TEXT_DIRECT
#define PFAC_TEXT_DIRECT 0
#endif
#ifndef PFAC_PH1_UNROLL
#define PFAC_PH1_UNROLL 1
#endif
#ifndef PFAC_MT_1K
#define PFAC_MT_1K 1024  // the 1024-position text kernels: 32 warps (cfg4 -3.5%, cfg5 -4.4% vs 28; profiles/r02_cta_ab.jsonl)
#endif
constexpr int kMT = PFAC_MT;                // threads per CTA (A/B knob)
constexpr int kPh1Unroll = PFAC_PH1_UNROLL; // sub-slices unrolled in the lookup phase (A/B knob)
constexpr int kMWarps = kMT / 32;
// threads per CTA of the 1024-position-slice text kernels (A/B knob: their smaller per-warp buffers leave
// the shared memory for more warps)
static __host__ __device__ constexpr int mt_for(uint32_t slice) { return slice == 1024 ? PFAC_MT_1K : kMT; }
static_assert(PFAC_MT_1K % 32 == 0 && PFAC_MT_1K <= 1024, "whole warps, <= 32 per CTA (grid_prefix)");
constexpr uint32_t kP = 8;                  // consecutive positions per lane per sub-slice
constexpr uint32_t kSubN = 32 * kP;         // 256 positions per sub-slice
#ifndef PFAC_SLICE
#define PFAC_SLICE 2048
#endif
constexpr uint32_t kSlice = PFAC_SLICE;     // positions per warp slice (A/B knob; multiple of 1024)
constexpr uint32_t kBmWords = kSlice / 32;  // words of the fused kernel's per-slice match bitmap
static_assert(kSlice % 1024 == 0 && kSlice <= 65536, "slice = whole 1024-position groups, u16 positions");

struct MatchArgs {
    const uint32_t *packed;
    int32_t *out;
    uint64_t n_own, n_avail, nslices, avail_words;
    const void *J, *T, *F;
    uint32_t window;       // device ids [0, window) have T row / F entry in smem
    uint32_t root;         // device id of the start state
    uint32_t slice_words;  // kSlice/16 + halo words copied per slice (buffers hold +4 words of slack)
    uint32_t short_pat;    // some pattern is shorter than K (K2): dead J (J2) entries may hold answers
    const uint32_t *J2;    // second-level jump table (uint32 images), L2-persisting
    const uint32_t *FB;    // uint32 images: the K1-mer filter bitmap (staged in smem instead of J)
    uint32_t K2, mask2;
    const uint16_t *inv;   // BAR: bit j of inv[w] = base 16w+j is not ACGT (a barrier), pfac_inv_words
    uint32_t bar_dead;     // BAR: (1 << min(minlen, K1)) - 1: a barrier this close ends every match
    uint64_t slices_per_warp;  // fused mode: each warp owns a contiguous run of slices
    CompactArgs c;         // fused mode: the match list (n = n_own, chunk = slices_per_warp * kSlice)
    const uint8_t *text;   // TXT: the ASCII text (n_avail bytes, 16-byte aligned)
    const uint4 *HR;       // uint32 images (nullable): chain-head row copies, J2 entries ALIVE|HRF|index
    uint64_t *first_bad;   // TXT (nullable): atomicMin of pos_base + the first owned non-ACGT index;
                           // bad_all set: written once from *bad_all (the owned part of it)
    const uint64_t *bad_all;  // BAR, packed input (nullable): pack's first bad index over the readable
                              // text; UINT64_MAX = no barrier anywhere, the barrier bits are not read
};

// One T row (4 cells).  Branch row: child per base.  Chain row: flag|L, then L forced bases.
template <typename CT>
struct Row;
template <>
struct Row<uint16_t> {
    uint2 r;
    uint32_t f;  // PFAC_MERGED_F: F(s) from the row's cell 4
    __device__ __forceinline__ bool chain() const { return r.x & 0x8000u; }
    __device__ __forceinline__ bool nofin() const { return r.x & 0x4000u; }
    __device__ __forceinline__ bool fstep() const { return r.x & kFStep16; }
    __device__ __forceinline__ uint32_t len() const { return r.x & 31u; }
    __device__ __forceinline__ uint32_t bits() const { return (r.x >> 16) | (r.y << 16); }
    __device__ __forceinline__ uint32_t fin() const { return r.y >> 16; }
    __device__ __forceinline__ uint32_t child(uint32_t c) const { return ((c & 2 ? r.y : r.x) >> ((c & 1) * 16)) & 0xFFFFu; }
};
template <>
struct Row<uint32_t> {
    uint4 r;
    uint32_t f;  // PFAC_MERGED_F: F(s) from the row's cell 4
    __device__ __forceinline__ bool chain() const { return r.x & 0x80000000u; }
    __device__ __forceinline__ bool nofin() const { return r.x & 0x40000000u; }
    __device__ __forceinline__ uint32_t len() const { return r.x & kChainLenMask32; }
    __device__ __forceinline__ uint32_t bits() const { return r.y; }
    __device__ __forceinline__ uint64_t bits64() const { return ((uint64_t)r.w << 32) | r.y; }  // T rows only
    __device__ __forceinline__ uint32_t fin() const { return r.z; }
    __device__ __forceinline__ uint32_t end_answer() const { return (r.x >> kEndShift) & kEndMask; }  // F(end) + 1
    __device__ __forceinline__ uint32_t child(uint32_t c) const {
        return c & 2 ? (c & 1 ? r.w : r.z) : (c & 1 ? r.y : r.x);
    }
};

// Table loads (rows, F, J2, HR): read-only for the whole launch, so ld.global.nc (L1-cached) by
// default; PFAC_TAB_CG=1 is the ablation with ld.global.cg (L2 only) -- the B200 analogue of the
// paper's -Xptxas -dlcm=cg runs.
#ifndef PFAC_TAB_CG
#define PFAC_TAB_CG 0
#endif
template <typename T>
__device__ __forceinline__ T ld_tab(const T *p) {
#if PFAC_TAB_CG
    return __ldcg(p);
#else
    return __ldg(p);
#endif
}

// L1::no_allocate forms (A/B knobs PFAC_J2_NA: J2 and HR loads; PFAC_TAB_NA: every table load): the
// lookups of large automata are random over megabytes, so an L1 line allocated per miss buys no reuse
#ifndef PFAC_J2_NA
#define PFAC_J2_NA 0
#endif
#ifndef PFAC_TAB_NA
#define PFAC_TAB_NA 0
#endif
__device__ __forceinline__ uint32_t ld_na(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_na(const uint2 *p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_na(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint16_t ld_na(const uint16_t *p) {
    uint16_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
    return v;
}
template <typename T>
__device__ __forceinline__ T ld_row(const T *p) {  // T rows and F entries
    if constexpr (PFAC_TAB_NA) return ld_na(p);
    else return ld_tab(p);
}
#ifndef PFAC_J2_NA32
#define PFAC_J2_NA32 0  // A/B knob: J2 / HR loads of uint32 images L1::no_allocate (cfg4 -0.9% warm,
                        // but a cold L2 (ncu replay) then re-reads J2 from DRAM: 2.15x the algorithmic bytes)
#endif
template <bool U32, typename T>
__device__ __forceinline__ T ld_j2(const T *p) {  // J2 entries and chain-head row copies
    if constexpr (PFAC_TAB_NA || PFAC_J2_NA || (U32 && PFAC_J2_NA32)) return ld_na(p);
    else return ld_tab(p);
}

// Shared-window loads by 32-bit shared address (the row window is read through these, so the walk
// loop does not convert a generic pointer to a shared address, an S2R, per step)
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_cell(uint32_t a, uint16_t) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_cell(uint32_t a, uint32_t) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
#ifndef PFAC_LDS_ADDR
#define PFAC_LDS_ADDR 1  // A/B knob: 0 = the row window read through generic pointers
#endif

template <typename CT, bool WIN>
struct Tab {
    const CT *Tw, *Fw, *Tg, *Fg;
    uint32_t W;
    uint32_t sTa, sFa;  // shared-window addresses of Tw and Fw
    __device__ __forceinline__ Row<CT> row(uint32_t s) const {
        Row<CT> r;
        if constexpr (sizeof(CT) == 2 && kMergedF) {  // one 16-byte row: 4 transitions, F, padding
            const uint4 v = (!WIN || s < W) ? *reinterpret_cast<const uint4 *>(Tw + (size_t)s * kRowCells)
                                            : ld_row(reinterpret_cast<const uint4 *>(Tg + (size_t)s * kRowCells));
            r.r = make_uint2(v.x, v.y);
            r.f = v.z & 0xFFFFu;
        } else if constexpr (sizeof(CT) == 2) {
            if (!WIN || s < W) r.r = PFAC_LDS_ADDR ? lds_v2(sTa + s * (kRowCells * 2)) : *reinterpret_cast<const uint2 *>(Tw + (size_t)s * kRowCells);
            else r.r = ld_row(reinterpret_cast<const uint2 *>(Tg + (size_t)s * kRowCells));
        } else {
            if (!WIN || s < W) r.r = PFAC_LDS_ADDR ? lds_v4(sTa + s * (kRowCells * 4)) : *reinterpret_cast<const uint4 *>(Tw + (size_t)s * kRowCells);
            else r.r = ld_row(reinterpret_cast<const uint4 *>(Tg + (size_t)s * kRowCells));
            if constexpr (kMergedF)
                r.f = (!WIN || s < W) ? (uint32_t)Tw[(size_t)s * kRowCells + 4] : (uint32_t)ld_row(Tg + (size_t)s * kRowCells + 4);
        }
        return r;
    }
    __device__ __forceinline__ uint32_t final_of(uint32_t s) const {
        if constexpr (kMergedF) {
            const size_t b = (size_t)s * kRowCells + 4;
            if constexpr (!WIN) return Tw[b];
            else return s < W ? (uint32_t)Tw[b] : (uint32_t)ld_row(Tg + b);
        } else if constexpr (!WIN) {
            return PFAC_LDS_ADDR ? lds_cell(sFa + s * (uint32_t)sizeof(CT), CT{}) : (uint32_t)Fw[s];
        } else {
            return s < W ? (PFAC_LDS_ADDR ? lds_cell(sFa + s * (uint32_t)sizeof(CT), CT{}) : (uint32_t)Fw[s])
                         : (uint32_t)ld_row(Fg + s);
        }
    }
};

// Rank of this lane's first set bit among the warp's 4-bit masks m (lane order), via three ballots
// of the per-lane counts (0..4); tot = the warp's total.  lt = lanes below this one.
__device__ __forceinline__ uint32_t nibble_rank(uint32_t m, uint32_t lt, uint32_t &tot) {
    const uint32_t c = __popc(m);
    const uint32_t b0 = __ballot_sync(~0u, c & 1), b1 = __ballot_sync(~0u, c & 2), b2 = __ballot_sync(~0u, c & 4);
    tot = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
    return __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
}

#ifndef PFAC_FB_LOP
#define PFAC_FB_LOP 1  // A/B knob: 0 = filter word address as base + offset (an extra IADD per lookup)
#endif
// Shared-window offset of the dynamic shared memory when the kernel has no static shared memory:
// the 1 KiB the system reserves per block comes first (cudaDevAttrReservedSharedMemoryPerBlock,
// checked by plan_match).
constexpr uint32_t kFBSmemBase = 1024;
constexpr bool kFbLop = PFAC_FB_LOP && kFilterK == 10;  // the 0x1FFFC mask is FB's 128 KiB
constexpr bool kLdsConst = PFAC_LDS_ADDR && kFbLop;  // row window at constant shared addresses

bool fb_addressing_ok(int device) {
    int reserved = -1;
    if (cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, device) != cudaSuccess) return false;
    return !kFbLop || (uint32_t)reserved == kFBSmemBase;
}

// The 4-byte filter word at byte offset (y & 0x1FFFC) of FB, the first 128 KiB of the dynamic shared
// memory: hi = the shared-window address of the dynamic region with its low 17 bits cleared, so the
// address is one LOP3 ((y & 0x1FFFC) | hi) and the region's base rides in the load's immediate.
__device__ __forceinline__ uint32_t lds_fb(uint32_t hi, uint32_t y) {
    uint32_t a, v;
    asm("lop3.b32 %0, %1, 0x1FFFC, %2, 0xEA;" : "=r"(a) : "r"(y), "r"(hi));
    asm volatile("ld.shared.u32 %0, [%1+1024];" : "=r"(v) : "r"(a));
    return v;
}

// 16 bases starting at local offset l (base i in bits 2i).
__device__ __forceinline__ uint32_t window16(const uint32_t *txt, uint32_t l) {
    const uint32_t q = l >> 4;
    return (uint32_t)(((((uint64_t)txt[q + 1]) << 32) | txt[q]) >> ((l & 15) * 2));
}

// 32 bases starting at local offset l (base i in bits 2i).
__device__ __forceinline__ uint64_t window32(const uint32_t *txt, uint32_t l) {
    const uint32_t q = l >> 4, sh = (l & 15) * 2;
    const uint32_t a = txt[q], b = txt[q + 1], c = txt[q + 2];
    return ((uint64_t)__funnelshift_r(b, c, sh) << 32) | __funnelshift_r(a, b, sh);
}

// The PFAC walk from state s reading bases l, l+1, ... (< lend): follow the goto function until the
// first missing transition.  A chain row advances over its forced bases with one
// XOR (up to 16 per uint16 row, 32 per uint32 row); the answer is F of the last state reached (the
// deepest final passed).  A walk that ends inside a NOFIN chain span returns the row's own F without
// another lookup; one that consumes a uint32 span ending in a state without transitions returns the
// row's end answer.
template <typename CT, bool WIN>
__device__ __forceinline__ uint32_t walk(const Tab<CT, WIN> &tb, const uint32_t *txt, uint32_t s, uint32_t l,
                                         uint32_t lend) {
    while (l < lend) {
        const Row<CT> r = tb.row(s);
        uint32_t m, c0;
        if constexpr (sizeof(CT) == 4) {
            const uint64_t w = window32(txt, l);
            const uint64_t d = w ^ r.bits64();
            m = d ? (uint32_t)(__ffsll((long long)d) - 1) >> 1 : 32u;  // matching leading bases
            c0 = (uint32_t)w & 3u;
        } else {
            const uint32_t w = window16(txt, l);
            const uint32_t d = w ^ r.bits();
            m = d ? (uint32_t)(__ffs(d) - 1) >> 1 : 16u;
            c0 = w & 3u;
        }
        if (r.chain()) {
            const uint32_t L = r.len();
            const uint32_t rem = lend - l;
            const uint32_t lim = L < rem ? L : rem;
            if (m < lim || lim < L) {  // the walk ends inside this span, at s + min(m, lim)
                const uint32_t mm = m < lim ? m : lim;
                if (r.nofin() || mm == 0) return r.fin();
                if constexpr (sizeof(CT) == 2) {
                    if (r.fstep()) return r.fin() + mm;  // F(s + mm) = F(s) + mm along this span
                }
                s += mm;
                break;
            }
            if constexpr (sizeof(CT) == 4) {
                if (const uint32_t e = r.end_answer()) return e - 1;  // the span ends in a dead end
            }
            s += L;
            l += L;
        } else {
            const uint32_t t = r.child(c0);
            if (!t) {
                if constexpr (kMergedF) return r.f;  // the answer came with the row
                break;
            }
            s = t;
            ++l;
        }
    }
    return tb.final_of(s);
}

// walk() from a depth-K2 chain head whose row comes from the compact copy HR (uint32 images): the
// first step reads the given row (cell 3 = the head's device id), the rest continues in T.
template <typename CT, bool WIN>
__device__ __forceinline__ uint32_t walk_head(const Tab<CT, WIN> &tb, const uint32_t *txt, const uint4 row, uint32_t l,
                                              uint32_t lend) {
    const uint32_t s = row.w;
    if (l >= lend) return tb.final_of(s);
    Row<uint32_t> r;
    r.r = row;
    const uint32_t w = window16(txt, l);
    const uint32_t L = r.len();
    const uint32_t d = w ^ r.bits();
    const uint32_t m = d ? (uint32_t)(__ffs(d) - 1) >> 1 : 16u;
    const uint32_t rem = lend - l;
    const uint32_t lim = L < rem ? L : rem;
    if (m < lim || lim < L) {  // the walk ends inside this span
        const uint32_t mm = m < lim ? m : lim;
        if (r.nofin() || mm == 0) return r.fin();
        return tb.final_of(s + mm);
    }
    if (const uint32_t e = r.end_answer()) return e - 1;  // the span ends in a dead end
    return walk(tb, txt, s + L, l + L, lend);
}

#ifndef PFAC_CONTIG
#define PFAC_CONTIG 1
#endif
#ifndef PFAC_ZERO_CONTIG
#define PFAC_ZERO_CONTIG 1
#endif
#ifndef PFAC_P16
#define PFAC_P16 0  // A/B knob: filter-path interior slices with 16 positions per lane (measured: cfg2 -1.4%, cfg3 +2.8%)
#endif
constexpr bool kP16 = PFAC_P16;
constexpr bool kContiguousSchedule = PFAC_CONTIG;
#ifndef PFAC_BALANCED
#define PFAC_BALANCED 0  // A/B knob: 1 = runs balanced to within one slice (measured slower on cfg2)
#endif
#ifndef PFAC_SPW_PAD
#define PFAC_SPW_PAD 0   // A/B knob: extra slices per warp run (probes the out[] stream spacing)
#endif  // unfused kernel: contiguous slice runs per warp (A/B)
#ifndef PFAC_DRAIN_IPL
#define PFAC_DRAIN_IPL 1
#endif
#ifndef PFAC_DRAIN_IPL_1K
#define PFAC_DRAIN_IPL_1K 2
#endif
// queued items per lane per drain round (A/B knobs): two for the 1024-position-slice kernels (large
// automata: J2 latency; cfg4 -3%), one elsewhere (cfg2/cfg3 +1% with two)
static __host__ __device__ constexpr uint32_t drain_ipl_for(uint32_t bm_words) {
    return bm_words <= 32 ? PFAC_DRAIN_IPL_1K : PFAC_DRAIN_IPL;
}
// queue of flagged positions (entries per warp): the 1024-position-slice kernels (large automata,
// ~9% of positions flagged: ~90 per 1024-position group) have the shared memory for a longer one
#ifndef PFAC_QEXTRA_1K
#define PFAC_QEXTRA_1K 96  // queue beyond one drain round (1024-position kernels): keeps 32 warps' shared
                           // memory under the 196-KB carve-out on uint32 images (more L1 for the misses)
#endif
static __host__ __device__ constexpr uint32_t qcap_for(uint32_t bm_words) {
    return 32 * drain_ipl_for(bm_words) + (bm_words <= 32 ? PFAC_QEXTRA_1K : 64);
}
#ifndef PFAC_PUSH_SCAN
#define PFAC_PUSH_SCAN 1  // A/B knob: 0 = one ballot round per queued position per lane
#endif
constexpr bool kPushScan = PFAC_PUSH_SCAN;
#ifndef PFAC_DEFER
#define PFAC_DEFER 0  // A/B knob: 1 = a group's last drain round resolved after the next group's filter
                      // step (measured slower: cfg2 +2.4%, cfg3 +2%, cfg4 +6.7%, cfg5 +5%)
#endif
constexpr bool kDeferRound = PFAC_DEFER;
#ifndef PFAC_MATCH_LOG
#define PFAC_MATCH_LOG 1  // A/B knob: 0 = no per-warp match log (a full staging area spills at once)
#endif
constexpr bool kMatchLog = PFAC_MATCH_LOG;
constexpr int kFBK = kFilterK;                         // filter length K1 (FBM)
constexpr uint32_t kFBBytes = (1u << (2 * kFBK)) / 8;  // 4^K1 bits of shared memory (4^10: 128 KiB)

static __host__ __device__ constexpr uint32_t inv_buf_words(uint32_t slice_words) {  // uint16, 16-B multiple
    return (slice_words + 8 + 7) & ~7u;
}
#ifndef PFAC_JPRE
#define PFAC_JPRE 0  // A/B knob: 1 = J2 prefetch at filter time in the 1024-position uint32 text kernels
#endif
#ifndef PFAC_JPRE_K
#define PFAC_JPRE_K 8
#endif
#ifndef PFAC_JPRE_PROBE
#define PFAC_JPRE_PROBE 0  // probe: the JPRE shared-memory buffer allocated, never used
#endif
constexpr uint32_t kJPreK = PFAC_JPRE_K;  // J2 prefetch slots per lane and 1024-position group
static_assert(kK2Max + 7 <= 24, "JPRE: a lane's K2-mers come from its 64-bit text window (>= 24 bases)");
// J2 prefetch (JPRE): the 1024-position-slice text kernels of uint32 images (large automata, ~9% of
// positions flagged) have the shared memory for a per-lane buffer of kJPreK J2 entries
static __host__ __device__ constexpr bool jpre_for(bool txt, uint32_t bm_words, uint32_t cell) {
    return PFAC_JPRE && txt && bm_words == 32 && cell == 4;
}
static __host__ __device__ constexpr uint32_t warp_bytes(uint32_t slice_words, bool bar = false, bool txt = false,
                                                         uint32_t bm_words = kBmWords, bool jpre = false) {
    // TXT: ASCII staging (slice_words * 16 bytes) + ONE packed slice and barrier-bit buffer (the warp
    // packs a slice before it prefetches the next one's bytes, so the ASCII buffer is the double buffer)
    return txt ? slice_words * 16 + (slice_words + 4) * 4 + 16 + qcap_for(bm_words) * 2 + bm_words * 4 +
                     inv_buf_words(slice_words) * 2 + (jpre ? 32 * kJPreK * 4 : 0)
               : 2 * (slice_words + 4) * 4 + 16 + qcap_for(bm_words) * 2 + bm_words * 4 +  // text, mbarriers, queue, bitmap
                     (bar ? 2 * inv_buf_words(slice_words) * 2 : 0);          // BAR: the slice's barrier bits
}

// Places one match-log record: cnt entries (offset in the slice, id) at ranks r0.. of the list, slice
// positions from pbase.  128 entries per step, the next step's loads issued before this one's stores
// (as in warp_stream): the replay is a stream, not a chain of load-use latencies.  The record was
// written by this warp in this launch (coherent L2 loads).
__device__ __forceinline__ void replay_record(const CompactArgs &c, const uint32_t *ent, uint32_t cnt, uint64_t r0,
                                              uint64_t pbase, uint32_t lane) {
    const uint32_t steps = (cnt + 127) / 128;
    if (c.pid16) {
        uint32_t e[4], en[4];
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) e[k] = lane + 32 * k < cnt ? __ldcg(ent + lane + 32 * k) : 0u;
        for (uint32_t st = 0; st < steps; ++st) {
            const uint32_t i0 = st * 128 + lane;
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) en[k] = i0 + 128 + 32 * k < cnt ? __ldcg(ent + i0 + 128 + 32 * k) : 0u;
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
                if (i0 + 32 * k < cnt) put_match(c, r0 + i0 + 32 * k, pbase + (e[k] & 0xFFFFu), e[k] >> 16);
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) e[k] = en[k];
        }
    } else {
        const uint2 *ent2 = reinterpret_cast<const uint2 *>(ent);
        uint2 e[4], en[4];
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) e[k] = lane + 32 * k < cnt ? __ldcg(ent2 + lane + 32 * k) : make_uint2(0, 0);
        for (uint32_t st = 0; st < steps; ++st) {
            const uint32_t i0 = st * 128 + lane;
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
                en[k] = i0 + 128 + 32 * k < cnt ? __ldcg(ent2 + i0 + 128 + 32 * k) : make_uint2(0, 0);
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
                if (i0 + 32 * k < cnt) put_match(c, r0 + i0 + 32 * k, pbase + e[k].x, e[k].y);
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) e[k] = en[k];
        }
    }
}

// Grid-wide barrier of a cooperative launch (every CTA resident) on a per-call zeroed counter.
__device__ __forceinline__ void grid_sync(uint64_t *ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(reinterpret_cast<unsigned long long *>(ctr), 1ull);
        while (ld_acquire_u64(ctr) < gridDim.x) __nanosleep(64);
    }
    __syncthreads();
}

constexpr uint32_t kSpillBit = 0x80000000u;  // DYN: a slice's count word, its matches not logged

template <typename CT, bool WIN, int K, bool FUSE, bool FBM, bool BAR = false, bool LIST = false, bool TXT = false,
          uint32_t SL = kSlice, bool DYN = false>
__global__ void __launch_bounds__(mt_for(SL), 1) match_kernel(const MatchArgs p) {
    constexpr int kMWarps = mt_for(SL) / 32;  // warps per CTA of this instantiation
    // positions per slice (text kernel for large automata: 1024, which leaves L1 more room)
    static_assert(SL % 1024 == 0 && SL <= 65536, "slice = whole 1024-position groups, u16 positions");
    constexpr uint32_t kSliceT = SL, kHalvesT = SL / 1024, kBmWordsT = SL / 32;
    constexpr uint32_t kQCap = qcap_for(kBmWordsT), kDrainIPL = drain_ipl_for(kBmWordsT);
    static_assert(!BAR || FBM, "barrier semantics are implemented on the filter path");
    static_assert(!LIST || (FUSE && FBM), "list-only mode is the fused kernel on the filter path");
    static_assert(!TXT || (FUSE && BAR), "text mode is the fused kernel with per-slice barriers");
    static_assert(!DYN || TXT, "dynamic slice claiming: the text kernel");
    constexpr uint32_t NJ = 1u << (2 * K);
    constexpr uint32_t MASK = NJ - 1;
    constexpr uint32_t ALIVE = sizeof(CT) == 2 ? 0x8000u : 0x80000000u;
    static_assert(kP + K - 1 <= 16, "the eight K-mers of a lane come from one 32-bit window");
    [[maybe_unused]] constexpr uint32_t FBMASK = (1u << (2 * kFBK)) - 1;
    extern __shared__ __align__(128) uint8_t smem[];
    CT *sJ = reinterpret_cast<CT *>(smem);                 // J (4^K cells) ...
    const uint32_t *sFB = reinterpret_cast<const uint32_t *>(smem);  // ... or, FBM: the K1-mer filter
    CT *sT = reinterpret_cast<CT *>(smem + (FBM ? kFBBytes : NJ * sizeof(CT)));
    CT *sF = sT + (size_t)p.window * kRowCells;
    uint8_t *wbase = reinterpret_cast<uint8_t *>(sF + (kMergedF ? 0 : p.window));  // 16-byte aligned (W % 8 == 0)
    // JPRE: each flagged position's J2 entry is fetched (cp.async, LDGSTS) into a per-lane buffer as
    // soon as the filter flags it; the drain reads it from shared memory, so the L2 latency of the
    // first sub-slices' lookups hides behind the later sub-slices' filter work
    constexpr bool JPRE = FBM && jpre_for(TXT, kBmWordsT, sizeof(CT)) && !PFAC_JPRE_PROBE;
    const uint32_t WB = warp_bytes(p.slice_words, BAR, TXT, kBmWordsT, FBM && jpre_for(TXT, kBmWordsT, sizeof(CT)));
    uint64_t *tab_bar = reinterpret_cast<uint64_t *>(wbase + kMWarps * WB);

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint8_t *asc = wbase + warp * WB;  // TXT: the slice's ASCII bytes (TMA destination)
    uint32_t *txt0 = reinterpret_cast<uint32_t *>(asc + (TXT ? p.slice_words * 16 : 0));
    uint32_t *txt1 = TXT ? txt0 : txt0 + p.slice_words + 4;
    uint64_t *bar = reinterpret_cast<uint64_t *>(txt1 + p.slice_words + 4);
    uint16_t *queue = reinterpret_cast<uint16_t *>(bar + 2);
    uint32_t *bm = reinterpret_cast<uint32_t *>(queue + kQCap);  // fused: nonzero cells of the slice
    uint16_t *inv0 = reinterpret_cast<uint16_t *>(bm + kBmWordsT);  // BAR: barrier bits of the slice
    uint16_t *inv1 = TXT ? inv0 : inv0 + inv_buf_words(p.slice_words);
    uint32_t *jbuf = reinterpret_cast<uint32_t *>(inv1 + inv_buf_words(p.slice_words));  // JPRE: [32][kJPreK]
    (void)jbuf;
    const uint32_t lt = (1u << lane) - 1;
    // grid_prefix's per-warp counts live in the dynamic region too: with no static shared memory the
    // dynamic region (FB first) starts right after the 1 KiB the system reserves, which the filter
    // lookups' addressing relies on (fb_word)
    uint64_t *s_wcount = tab_bar + 1, *s_woff = tab_bar + 1 + kMWarps;
    uint32_t fb_hi = 0;
    if constexpr (kFbLop) {
        const uint32_t fb_sa = (uint32_t)__cvta_generic_to_shared(smem);
        if ((fb_sa & 0x1FFFFu) != kFBSmemBase) __trap();  // host-checked (fb_addressing_ok); never taken
        if (kLdsConst && (fb_sa & ~0x1FFFFu) != 0) __trap();  // a non-cluster launch: CTA window high bits 0
        fb_hi = fb_sa & ~0x1FFFFu;
    }
    // the filter word of K1-mer bits [sh, sh + 2 K1) of x: bit (x >> sh) & 31 of word (x >> (sh + 5))
    auto fb_word = [&](uint64_t x, uint32_t sh) -> uint32_t {
        if constexpr (kFbLop) return lds_fb(fb_hi, (uint32_t)(x >> (sh + 3)));
        else return sFB[((uint32_t)(x >> sh) & FBMASK) >> 5];
    };

    const uint64_t TW = (uint64_t)gridDim.x * kMWarps;
    const uint64_t gw = (uint64_t)blockIdx.x * kMWarps + warp;
    // slice schedule: strided over the grid, or (fused) a contiguous run per warp so that the warp's
    // matches come out in position order
    // DYN: warps claim slices from a global counter (walk-heavy text: per-slice work varies widely)
    constexpr bool CONTIG = !DYN && (FUSE || kContiguousSchedule);
    // contiguous runs balanced to within one slice: warp gw owns [gw*N/TW, (gw+1)*N/TW) (a ceil-sized
    // run per warp would leave the last warps idle: cfg2 has 30.2 slices per warp)
#if PFAC_BALANCED
    const uint64_t s_first = CONTIG ? gw * p.nslices / TW : gw;
    const uint64_t s_end = CONTIG ? (gw + 1) * p.nslices / TW : p.nslices;
#else
    const uint64_t s_first = CONTIG ? gw * p.slices_per_warp : gw;
    const uint64_t s_end = CONTIG ? (s_first + p.slices_per_warp < p.nslices ? s_first + p.slices_per_warp : p.nslices)
                                  : p.nslices;
#endif
    const uint64_t s_stride = CONTIG ? 1 : TW;
    constexpr bool DIRECT = PFAC_TEXT_DIRECT && !BAR;
    // BAR over packed text: when pack found no bad byte at all, the barrier bits are never read
    bool no_bar = false;
    if constexpr (BAR && !TXT) {
        if (p.bad_all) {
            const uint64_t b = __ldcg(p.bad_all);  // written by the pack kernel before this launch
            no_bar = b == ~0ull;
            if (p.first_bad && blockIdx.x == 0 && tid == 0) *p.first_bad = b < p.n_own ? p.c.pos_base + b : ~0ull;
        }
    }
    auto issue = [&](uint64_t sl, uint32_t *dst, uint64_t *b) {
        if constexpr (DIRECT) return;
        if constexpr (TXT) {  // the 16-byte multiple part of the slice's readable bytes (the rest: lanes)
            const uint64_t b0 = sl * kSliceT, left = p.n_avail - b0;
            const uint32_t nb = (uint32_t)(left < p.slice_words * 16ull ? left : p.slice_words * 16ull) & ~15u;
            mbar_expect_tx(b, nb);
            if (nb) bulk_g2s(asc, p.text + b0, nb, b);
            return;
        }
        const uint64_t w0 = sl * (kSliceT / 16);
        const uint64_t left = p.avail_words - w0;
        const uint32_t nw = left < p.slice_words ? (uint32_t)left : p.slice_words;
        if (BAR && !no_bar) {  // the barrier bits of the same bases ride on the same mbarrier
            const uint32_t ni = (nw + 7) & ~7u;  // 16-byte multiple (the inv array is padded to 8 words)
            uint16_t *idst = dst == txt0 ? inv0 : inv1;
            mbar_expect_tx(b, nw * 4 + ni * 2);
            bulk_g2s(dst, p.packed + w0, nw * 4, b);
            bulk_g2s(idst, p.inv + w0, ni * 2, b);
        } else {
            mbar_expect_tx(b, nw * 4);
            bulk_g2s(dst, p.packed + w0, nw * 4, b);
        }
    };
    if (tid == 0) mbar_init(tab_bar, 1);
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    fence_mbar_init();
    __syncthreads();
    if (tid == 0) {
        const uint32_t jb = FBM ? kFBBytes : NJ * sizeof(CT), tb = p.window * kRowCells * sizeof(CT),
                       fb = kMergedF ? 0u : p.window * (uint32_t)sizeof(CT);
        mbar_expect_tx(tab_bar, jb + tb + fb);
        bulk_g2s(smem, FBM ? (const void *)p.FB : p.J, jb, tab_bar);
        if (p.window) {
            bulk_g2s(sT, p.T, tb, tab_bar);
            if (fb) bulk_g2s(sF, p.F, fb, tab_bar);
        }
    }
    // DYN: the first slice, then each next one claimed one slice ahead (its TMA is issued mid-slice)
    uint64_t sl0 = s_first, claim = 0;
    if constexpr (DYN) {
        if (lane == 0) claim = atomicAdd(reinterpret_cast<unsigned long long *>(p.c.ctl), 1ull);
        sl0 = __shfl_sync(~0u, claim, 0);
    }
    if (lane == 0 && sl0 < s_end) issue(sl0, txt0, &bar[0]);
    // the row window's shared-window address as a constant (+ the window size from the parameters):
    // the dynamic region starts at kFBSmemBase of a CTA window whose high bits are 0 (checked above),
    // so no walk step converts a generic pointer (an S2R the compiler would otherwise rematerialize)
    constexpr uint32_t kTOff = kFBSmemBase + (FBM ? kFBBytes : NJ * (uint32_t)sizeof(CT));
    const uint32_t sTa = kLdsConst ? kTOff : (uint32_t)__cvta_generic_to_shared(sT);
    const Tab<CT, WIN> tb{sT, sF, reinterpret_cast<const CT *>(p.T), reinterpret_cast<const CT *>(p.F), p.window,
                          sTa, sTa + p.window * (uint32_t)(kRowCells * sizeof(CT))};
    if constexpr (!TXT) mbar_wait(tab_bar, 0);  // TXT: after packing the first slice (overlaps the load)
    bool pred_bar = false;  // TXT: the previous slice had a barrier (FASTA text: every slice has one)

    uint32_t it = 0;
    uint64_t wcount = 0;   // fused: matches of this warp so far
    // fused: a slice's matches go to the staging area while it has room (wstaged == wcount), then
    // to the warp's match log while that has room, then are spilled (re-read after the prefix)
    uint32_t wstaged = 0;     // fused: matches staged (<= stg)
    uint32_t log_off = 0;     // fused: bytes of the warp's match log used (< 2^32: log_pw ~ run length)
    uint32_t spill_rel = ~0u; // fused: first spilled slice, relative to s_first (~0u: none)
    bool bad_done = false;    // TXT: this warp has reported its first non-ACGT byte (slices ascend)
    uint64_t *spos = FUSE ? p.c.stage_pos + gw * p.c.stg : nullptr;
    uint32_t *spid = FUSE ? p.c.stage_pid + gw * p.c.stg : nullptr;
    uint64_t sl_next = 0;
    for (uint64_t sl = sl0; sl < s_end; sl = sl_next, ++it) {
        if constexpr (DYN) {
            if (lane == 0) claim = atomicAdd(reinterpret_cast<unsigned long long *>(p.c.ctl), 1ull);
        } else {
            sl_next = sl + s_stride;
        }
        const uint32_t buf = it & 1;
        if (!TXT && lane == 0 && sl + s_stride < s_end) issue(sl + s_stride, buf ? txt0 : txt1, &bar[buf ^ 1]);
            if (FUSE) {
            for (uint32_t w = lane; w < kBmWordsT; w += 32) bm[w] = 0;
            __syncwarp();
        }
        if constexpr (TXT) mbar_wait(&bar[0], it & 1);
        else if constexpr (!DIRECT) mbar_wait(&bar[buf], (it >> 1) & 1);
        const uint32_t *txt = DIRECT ? p.packed + sl * (kSliceT / 16) : (buf ? txt1 : txt0);
        const uint16_t *inv = buf ? inv1 : inv0;
        (void)inv;
        const uint64_t base = sl * kSliceT;
        const uint64_t avail_left = p.n_avail - base;
        const uint32_t lend = avail_left < p.slice_words * 16ull ? (uint32_t)avail_left : p.slice_words * 16;
        const uint64_t own_left = p.n_own - base;
        const uint32_t lown = own_left < kSliceT ? (uint32_t)own_left : kSliceT;
        int32_t *out = p.out + base;
        // BAR: does any readable base of this slice (owned range + halo) fail to be ACGT?
        bool bar_slice = false;
        if constexpr (TXT) {
            // Pack the slice (16 bases per lane and step, PAPER.md:120's 4-letter alphabet as 2-bit
            // codes); bytes past the readable end pack as A.  Two forms, chosen by whether the previous
            // slice had a barrier (a byte outside ACGTacgt, reading R5):
            //  * plain text: the hot pass only ORs the validity residues; a slice that turns out to
            //    hold a barrier gets its exact barrier bits in a second pass over its bytes;
            //  * FASTA-like text (barriers in every slice): each word keeps its four residues and a
            //    nonzero one gives the word's barrier bits at once (badmask16) -- one pass.
            const uint32_t nb = lend & ~15u;  // bytes the TMA brought; [nb, lend) come from global
            uint32_t acc = 0;
            auto tail_word = [&](uint32_t q, uint32_t &word) -> uint32_t {  // bytes [nb, lend) of word q
                uint32_t m = 0;
                for (uint32_t j = 0; j < 16 && q * 16 + j < lend; ++j) {
                    const uint32_t i = q * 16 + j;
                    const uint8_t b = i < nb ? asc[i] : p.text[base + i];
                    m |= valid_byte(b) ? 0u : 1u << j;
                    word |= (((b >> 1) ^ (b >> 2)) & 3u) << (2 * j);
                }
                return m;
            };
            if (pred_bar) {
                for (uint32_t q = lane; q < inv_buf_words(p.slice_words); q += 32) {
                    uint32_t word = 0, m = 0;
                    if (q * 16 + 16 <= nb) {
                        const uint4 v = *reinterpret_cast<const uint4 *>(asc + q * 16);
                        uint32_t r0, r1, r2, r3;
                        const uint32_t h0 = pack4r(v.x, r0), h1 = pack4r(v.y, r1), h2 = pack4r(v.z, r2),
                                       h3 = pack4r(v.w, r3);
                        word = byte_perm(byte_perm(h0, h1, 0x0040u), byte_perm(h2, h3, 0x0040u), 0x5410u);
                        if ((r0 | r1 | r2 | r3) & kBadMask) m = badmask16(r0, r1, r2, r3);
                    } else if (q * 16 < lend) {
                        m = tail_word(q, word);
                    }
                    acc |= m;
                    if (q < p.slice_words + 4) txt0[q] = word;
                    inv0[q] = (uint16_t)m;
                }
                bar_slice = __any_sync(~0u, acc != 0);
            } else {
                for (uint32_t q = lane; q < p.slice_words + 4; q += 32) {
                    uint32_t word = 0;
                    if (q * 16 + 16 <= nb) {
                        const uint4 v = *reinterpret_cast<const uint4 *>(asc + q * 16);
                        word = pack16(v.x, v.y, v.z, v.w, acc);
                    } else if (q * 16 < lend) {
                        acc |= tail_word(q, word) ? 1u : 0u;
                    }
                    txt0[q] = word;
                }
                bar_slice = __any_sync(~0u, (acc & kBadMask) != 0);
                if (bar_slice) {  // exact barrier bits of every word of the slice
                    for (uint32_t q = lane; q < inv_buf_words(p.slice_words); q += 32) {
                        uint32_t m = 0, w = 0;
                        if (q * 16 + 16 <= nb) {
                            const uint4 v = *reinterpret_cast<const uint4 *>(asc + q * 16);
                            uint32_t r0, r1, r2, r3;
                            pack4r(v.x, r0), pack4r(v.y, r1), pack4r(v.z, r2), pack4r(v.w, r3);
                            m = badmask16(r0, r1, r2, r3);
                        } else if (q * 16 < lend) {
                            m = tail_word(q, w);
                        }
                        inv0[q] = (uint16_t)m;
                    }
                }
            }
            if (bar_slice && p.first_bad && !bad_done) {  // the first owned barrier, from the bits
                __syncwarp();
                uint32_t firstb = ~0u;
                for (uint32_t q = lane; q * 16 < lown; q += 32) {
                    const uint32_t m = inv0[q];
                    const uint32_t mo = lown - q * 16 >= 16 ? m : m & ((1u << (lown - q * 16)) - 1);
                    if (mo) {
                        firstb = q * 16 + (__ffs(mo) - 1);  // q ascends per lane
                        break;
                    }
                }
                firstb = __reduce_min_sync(~0u, firstb);
                if (firstb != ~0u) {
                    if (lane == 0)
                        atomicMin(reinterpret_cast<unsigned long long *>(p.first_bad),
                                  (unsigned long long)(p.c.pos_base + base + firstb));
                    bad_done = true;
                }
            }
            __syncwarp();  // the ASCII buffer is free: fetch the next slice while this one is matched
            if constexpr (DYN) sl_next = __shfl_sync(~0u, claim, 0);
            if (lane == 0 && sl_next < s_end) issue(sl_next, txt0, &bar[0]);
            if (it == 0) mbar_wait(tab_bar, 0);
        } else if (BAR && !no_bar) {
            uint32_t any = 0;
            for (uint32_t w = lane; w < (lend + 15) / 16; w += 32) any |= inv[w];
            bar_slice = __any_sync(~0u, any) != 0;
        }
        // BAR: local offset of the first barrier at or after l (a walk from l reads bases < it)
        auto next_barrier = [&](uint32_t l) -> uint32_t {
            uint32_t q = l >> 4;
            uint32_t bits = (uint32_t)inv[q] >> (l & 15);
            uint32_t at = l;
            while (!bits) {
                at = (q + 1) * 16;
                if (at >= lend) return lend;
                bits = inv[++q];
            }
            const uint32_t b = at + (__ffs(bits) - 1);
            return b < lend ? b : lend;
        };
        (void)next_barrier;

        uint32_t qn = 0;  // warp-uniform length of the queue of alive positions
        // Walk the queued positions 32 at a time (one per lane) until at most `keep` remain.  The
        // __syncwarp orders the queue writes and the owners' v4 stores before these patch stores.
        // A drain round: issue() takes up to 32 * kDrainIPL queued items (kDrainIPL per lane) and issues
        // all their J2 loads; resolve() consumes them (an NB check, a chain-head row, a walk) and
        // patches out[].  One L2 round trip serves the whole round.
        uint32_t dl[kDrainIPL], dg[kDrainIPL];  // position, J2 entry (the walk bound is recomputed: registers)
        auto issue = [&](uint32_t take, uint32_t qb) {
#pragma unroll
            for (uint32_t k = 0; k < kDrainIPL; ++k) {
                const uint32_t i = lane + 32 * k;
                const uint32_t e = i < take ? queue[qb + i] : 0xFFFFu;
                // JPRE entries: bit 15 = J2 prefetched into slot (bits 12-14) of the owner lane's buffer
                dl[k] = JPRE && i < take ? e & 0xFFFu : e;
                const uint32_t le = (BAR && bar_slice && i < take) ? next_barrier(dl[k]) : lend;
                if (JPRE && i < take && (e & 0x8000u))
                    dg[k] = jbuf[((dl[k] >> 3) & 31u) * kJPreK + ((e >> 12) & 7u)];
                else
                    dg[k] = (i < take && dl[k] + p.K2 <= le) ? ld_j2<sizeof(CT) == 4>(p.J2 + (window16(txt, dl[k]) & p.mask2))
                                                             : 0xFFFFFFFFu;
            }
        };
        auto resolve = [&]() {
#pragma unroll
            for (uint32_t k = 0; k < kDrainIPL; ++k) {
                const uint32_t l = dl[k], g = dg[k];
                if (l == 0xFFFFu) continue;
                const uint32_t le = (BAR && bar_slice) ? next_barrier(l) : lend;  // the walk's bound
                uint32_t res;
                if (g == 0xFFFFFFFFu) res = walk(tb, txt, p.root, l, le);  // near the end / a barrier
                else if (sizeof(CT) == 4 && p.HR && (g & kJ2HR)) {  // a chain head's row copy
                    // NB entry: unless the next 4 bases are the chain's first 4 (and readable), the walk
                    // ends inside the NOFIN span of an F = 0 head: the answer is 0 without the row load
                    // (builder.cpp, pfac_internal.h)
                    const uint32_t l2 = l + p.K2;
                    if ((g & kJ2NB) && (le - l2 < kHRBases || ((window16(txt, l2) ^ (g >> kHRIndexBitsNB)) & 0xFFu)))
                        res = 0;
                    else
                        res = walk_head(tb, txt, ld_j2<sizeof(CT) == 4>(p.HR + (g & (g & kJ2NB ? (1u << kHRIndexBitsNB) - 1 : kJ2NB - 1))),
                                        l2, le);
                }
                else if (g & 0x80000000u) res = walk(tb, txt, g & 0x7FFFFFFFu, l + p.K2, le);
                else res = g;
                if (!LIST || res) out[l] = (int32_t)res;
                if (FUSE && res) atomicOr(&bm[l >> 5], 1u << (l & 31));
            }
        };
        bool pending = false;  // a round issued at the end of one group and resolved after the next one's filter
        // Walk the queued positions (FBM: rounds as above) until at most `keep` remain.  The
        // __syncwarp orders the queue writes and the owners' v4 stores before these patch stores.
        auto drain = [&](uint32_t keep) {
            if constexpr (JPRE) cp_async_wait_all();  // this lane's prefetches (the loop's __syncwarp: all lanes')
            while (qn > keep) {
                __syncwarp();
                if constexpr (FBM) {
                    const uint32_t avail = qn - keep;
                    const uint32_t take = avail < 32 * kDrainIPL ? avail : 32 * kDrainIPL;
                    issue(take, qn - take);
                    resolve();
                    qn -= take;
                } else {
                    const uint32_t take = qn - keep < 32 ? qn - keep : 32;
                    if (lane < take) {
                        const uint32_t l = queue[qn - take + lane];
                        const uint32_t res = walk(tb, txt, (uint32_t)sJ[window16(txt, l) & MASK] & ~ALIVE, l + K, lend);
                        out[l] = (int32_t)res;
                        if (FUSE && res) atomicOr(&bm[l >> 5], 1u << (l & 31));
                    }
                    qn -= take;
                }
                __syncwarp();
            }
        };
        // the end of a group: drain to at most one round; with `defer`, issue that round's loads and leave
        // it pending (resolved after the next group's filter step, which hides the L2 latency)
        auto finish = [&](bool defer) {
            if (kDeferRound && FBM && defer) {
                drain(32 * kDrainIPL);
                if (qn) {
                    __syncwarp();
                    issue(qn, 0);
                    __syncwarp();  // the queue reads above before the next group's queue writes
                    qn = 0;
                    pending = true;
                }
            } else {
                drain(0);
            }
        };
        auto resolve_pending = [&]() {
            if (kDeferRound && FBM && pending) {
                resolve();
                pending = false;
            }
        };
        // Queue this lane's alive positions (bit r*8+j of `am` = position r*256 + lane*8 + j), one per
        // lane and round: a round costs one ballot, and there are max-over-lanes(popc(am)) rounds.
        // lg: log2 of the positions per lane per sub-slice of the bits in am (3: 8 positions, 4: 16)
        // pf (JPRE): the lane's flagged positions of this group had their J2 entries prefetched, the k-th
        // (in bit order) into slot k of its buffer (k < kJPreK)
        auto push = [&](uint32_t am, uint32_t gbase, uint32_t lg = 3, bool defer = false, bool pf = false) {
            uint32_t kk = 0;
            auto tag = [&]() -> uint32_t {
                const uint32_t t = (JPRE && pf && kk < kJPreK) ? 0x8000u | (kk << 12) : 0u;  // (kJPreK <= 8)
                ++kk;
                return t;
            };
            // The lanes' slots are the exclusive prefix of their counts c: from two ballots of the bits
            // of c when every c <= 3 (sparse groups: no shuffle chain), else a shuffle scan.  Each lane
            // then writes its own positions -- no ballot round per queued position.
            const uint32_t c = __popc(am);
            uint32_t excl = 0, total = 0;
            if (kPushScan) {
                if (!__ballot_sync(~0u, c > 3)) {
                    const uint32_t b0 = __ballot_sync(~0u, c & 1u), b1 = __ballot_sync(~0u, c & 2u);
                    excl = __popc(b0 & lt) + 2 * __popc(b1 & lt);
                    total = __popc(b0) + 2 * __popc(b1);
                    if (total == 0) return;
                } else {
                    uint32_t incl = c;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_up_sync(~0u, incl, d);
                        if (lane >= (uint32_t)d) incl += y;
                    }
                    excl = incl - c;
                    total = __shfl_sync(~0u, incl, 31);
                }
            }
            if (kPushScan && qn + total <= kQCap) {  // the group fits: each lane writes its own
                uint32_t slot = qn + excl;
                while (am) {
                    const uint32_t bit = __ffs(am) - 1;
                    am &= am - 1;
                    queue[slot++] =
                        (uint16_t)((gbase + (bit >> lg) * (32u << lg) + (lane << lg) + (bit & ((1u << lg) - 1))) | tag());
                }
                qn += total;
                finish(defer);
                return;
            }
            // dense groups (repetitive text): one queued position per lane and ballot round
            while (true) {
                const uint32_t b = __ballot_sync(~0u, am != 0);
                if (!b) break;
                if (qn + 32 > kQCap) drain(qn & 31);  // keep < 32: every drained round is full
                if (am) {
                    const uint32_t bit = __ffs(am) - 1;
                    am &= am - 1;
                    queue[qn + __popc(b & lt)] =
                        (uint16_t)((gbase + (bit >> lg) * (32u << lg) + (lane << lg) + (bit & ((1u << lg) - 1))) | tag());
                }
                qn += __popc(b);
            }
            finish(defer);
        };
        if (FBM && kP16 && lown == kSliceT && lend >= kSliceT + 16 + 16 && !(BAR && bar_slice)) {
            // interior slice, filter path, 16 positions per lane: one 64-bit window holds the 16
            // K1-mers of a lane (25 bases), and the warp's zero stores are four contiguous 512-B runs
#pragma unroll 1
          for (uint32_t hg = 0; hg < kHalvesT; ++hg) {
            uint32_t am = 0;
#pragma unroll
            for (uint32_t r = 0; r < 2; ++r) {
                const uint32_t q = hg * 64 + r * 32 + lane;  // l0 = 16 q
                const uint64_t x64 = (((uint64_t)txt[q + 1]) << 32) | txt[q];
                uint32_t m = 0;
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j)
                    m |= ((fb_word(x64, 2 * j) >> ((uint32_t)(x64 >> (2 * j)) & 31)) & 1u) << j;
                if constexpr (!LIST) {
                    const uint32_t z0 = hg * 1024 + r * 512 + lane * 4;
#pragma unroll
                    for (uint32_t k = 0; k < 4; ++k) st_stream_v4(out + z0 + 128 * k, 0u, 0u, 0u, 0u);
                }
                am |= m << (r * 16);
            }
            push(am, hg * 1024, 4);
          }
        } else if (lown == kSliceT && lend >= kSliceT + kP - 1 + (FBM ? 16 : K) && !(BAR && bar_slice)) {
            // interior slice: every position owned, every K-mer (K1-mer, K2-mer) readable
#pragma unroll 1
          for (uint32_t hg = 0; hg < kHalvesT; ++hg) {
            uint32_t am = 0;
            [[maybe_unused]] uint32_t kc = 0;  // JPRE: this lane's flagged positions so far in the group
#pragma unroll kPh1Unroll
            for (uint32_t r = 0; r < 4; ++r) {
                const uint32_t l0 = hg * 1024 + r * kSubN + lane * kP;
                if constexpr (FBM) {
                    // One filter bit per position: is the K1-mer at l0+j the start of a walk that survives
                    // K1 bases or completes a pattern?  Almost every answer is 0 and stored right away;
                    // the flagged positions are queued and resolved by J2 (+ a rare walk) in drain().
                    const uint32_t q = l0 >> 4;
                    const uint64_t x64 = ((((uint64_t)txt[q + 1]) << 32) | txt[q]) >> ((l0 & 15) * 2);
                    uint32_t m = 0;
                    if constexpr (PFAC_FMA_SHR && !TXT && !LIST) {
                    // the same lookups with the shifts on the FMA pipe (packed-input dense kernels: +3.5%
                    // on cfg2; the text kernel, whose packing loads the ALU pipe differently, loses 2.5%,
                    // the compute-bound list-only kernel ~5%):
                    // positions 0-5 from the low word y, 6-7 from z = x64 >> 12; K1-mer j of src =
                    // bits [2jj, 2jj + 2 K1) of it
                    static_assert(kFBK == 10 && kP == 8, "window split assumes 10-mers and 8 positions");
                    const uint32_t y = (uint32_t)x64, z = (uint32_t)(x64 >> 12);
#pragma unroll
                    for (uint32_t j = 0; j < kP; ++j) {
                        const uint32_t src = j < 6 ? y : z, jj = j < 6 ? j : j - 6;
                        const uint32_t a = shr_fma(src, 2 * jj + 3) & 0x1FFFCu;  // byte offset of the word
                        const uint32_t w = *reinterpret_cast<const uint32_t *>(reinterpret_cast<const uint8_t *>(sFB) + a);
                        const uint32_t s = jj ? shr_fma(src, 2 * jj) : src;       // low 5 bits: the bit
                        m |= ((w >> (s & 31)) & 1u) << j;
                    }
                    } else {
#pragma unroll
                    for (uint32_t j = 0; j < kP; ++j)
                        m |= ((fb_word(x64, 2 * j) >> ((uint32_t)(x64 >> (2 * j)) & 31)) & 1u) << j;
                    }
                    if constexpr (JPRE) {  // the flagged positions' J2 entries (K2-mer at l0 + j, in x64)
                        for (uint32_t mm = m; mm; mm &= mm - 1) {
                            const uint32_t j = __ffs(mm) - 1;
                            if (kc < kJPreK)
                                cp_async4(jbuf + lane * kJPreK + kc, p.J2 + ((uint32_t)(x64 >> (2 * j)) & p.mask2));
                            ++kc;
                        }
                    }
                    if constexpr (!LIST) {  // the sub-slice's zeros: every store is zeros, so the warp
                        // writes two contiguous 512-B runs (A/B knob: each lane its own 8 positions)
#if PFAC_ZERO_CONTIG
                        const uint32_t z0 = hg * 1024 + r * kSubN + lane * 4;
                        st_stream_v4(out + z0, 0u, 0u, 0u, 0u);
                        st_stream_v4(out + z0 + 128, 0u, 0u, 0u, 0u);
#else
                        st_stream_v4(out + l0, 0u, 0u, 0u, 0u);
                        st_stream_v4(out + l0 + 4, 0u, 0u, 0u, 0u);
#endif
                    }
                    am |= m << (r * kP);
                } else {
                    uint32_t e[kP];
                    const uint32_t x = window16(txt, l0);
#pragma unroll
                    for (uint32_t j = 0; j < kP; ++j) {
                        e[j] = sJ[(x >> (2 * j)) & MASK];
                        am |= (e[j] & ALIVE) ? (1u << (r * kP + j)) : 0u;
                    }
                    st_stream_v4(out + l0, e[0], e[1], e[2], e[3]);  // alive cells are patched by drain()
                    st_stream_v4(out + l0 + 4, e[4], e[5], e[6], e[7]);
                    if (FUSE && p.short_pat) {  // dead walks with an answer (a pattern shorter than K)
                        uint32_t nz = 0;
#pragma unroll
                        for (uint32_t j = 0; j < kP; ++j)
                            nz |= (e[j] != 0 && !(e[j] & ALIVE)) ? (1u << j) : 0u;
                        if (nz) atomicOr(&bm[l0 >> 5], nz << (l0 & 31));
                    }
                }
            }
            resolve_pending();  // the previous group's round: its J2 loads had this filter step to land
            push(am, hg * 1024, 3, FBM, JPRE);
          }
          resolve_pending();
        } else if (BAR && bar_slice) {
            // Barrier path: a position whose K1-mer window touches a non-ACGT base cannot use the filter;
            // it is queued with the filter-flagged ones, and drain() bounds every walk at the next
            // barrier (reading R5: a non-ACGT byte has no transition).  Zeros are stored first.
#pragma unroll 1
          for (uint32_t hg = 0; hg < kHalvesT; ++hg) {
            uint32_t am = 0;
#pragma unroll 1
            for (uint32_t r = 0; r < 4; ++r) {
                const uint32_t l0 = hg * 1024 + r * kSubN + lane * kP;
                if (l0 >= lown) continue;
                const uint32_t own = lown - l0 >= kP ? 0xFFu : (1u << (lown - l0)) - 1;
                uint32_t m = own;  // default: every owned position goes through drain()
                if (l0 + kP - 1 + kFBK <= lend) {
                    const uint32_t q = l0 >> 4, sh = (l0 & 15) * 2;
                    const uint64_t x64 = ((((uint64_t)txt[q + 1]) << 32) | txt[q]) >> sh;
                    const uint32_t ib = (uint32_t)((((uint64_t)inv[q + 2] << 32) | ((uint32_t)inv[q + 1] << 16) |
                                                    inv[q]) >> (l0 & 15));  // barrier bits of l0..l0+31
                    // near (bit j): a barrier within K1 bases of l0+j -- the filter cannot answer, the
                    // walk in drain() does; dead: a barrier within min(minlen, K1) bases -- no pattern
                    // fits before it, out = 0.  Both as smears of the barrier bits, branch-free.
                    uint32_t fb = 0, near = 0, dead = 0;
#pragma unroll
                    for (uint32_t j = 0; j < kP; ++j)
                        fb |= ((fb_word(x64, 2 * j) >> ((uint32_t)(x64 >> (2 * j)) & 31)) & 1u) << j;
#pragma unroll
                    for (uint32_t t = 0; t < (uint32_t)kFBK; ++t) {
                        near |= ib >> t;
                        dead |= (ib >> t) & (0u - ((p.bar_dead >> t) & 1u));
                    }
                    m = ((fb & ~near) | (near & ~dead)) & 0xFFu;
                    m &= own;
                }
                if (LIST) {
                } else if (l0 + kP <= lown) {
                    st_stream_v4(out + l0, 0u, 0u, 0u, 0u);
                    st_stream_v4(out + l0 + 4, 0u, 0u, 0u, 0u);
                } else {
                    for (uint32_t j = 0; j < kP; ++j)
                        if (l0 + j < lown) out[l0 + j] = 0;
                }
                am |= m << (r * kP);
            }
            push(am, hg * 1024);
          }
        } else if (FBM) {  // slice at the end of the text: every owned position goes through drain()
#pragma unroll 1
          for (uint32_t hg = 0; hg < kHalvesT; ++hg) {
            uint32_t am = 0;
#pragma unroll 1
            for (uint32_t r = 0; r < 4; ++r) {
                const uint32_t l0 = hg * 1024 + r * kSubN + lane * kP;
                if (l0 >= lown) continue;
                const uint32_t own = lown - l0 >= kP ? 0xFFu : (1u << (lown - l0)) - 1;
                am |= own << (r * kP);
            }
            push(am, hg * 1024);
          }
        } else {
#pragma unroll 1
          for (uint32_t hg = 0; hg < kHalvesT; ++hg) {
            uint32_t am = 0;
#pragma unroll 1
            for (uint32_t r = 0; r < 4; ++r) {
                const uint32_t l0 = hg * 1024 + r * kSubN + lane * kP;
                if (l0 >= lown) continue;
                uint32_t e[kP];
                uint32_t alive = 0;
                if (l0 + kP - 1 + K <= lend) {  // all eight K-mers readable: one J lookup each
                    const uint32_t x = window16(txt, l0);
#pragma unroll
                    for (uint32_t j = 0; j < kP; ++j) {
                        e[j] = sJ[(x >> (2 * j)) & MASK];
                        alive |= (e[j] & ALIVE) ? (1u << j) : 0u;
                    }
                } else {  // the last bases of the readable text: plain walks from the root
#pragma unroll
                    for (uint32_t j = 0; j < kP; ++j)
                        e[j] = l0 + j < lend ? walk(tb, txt, p.root, l0 + j, lend) : 0u;
                }
                if (l0 + kP <= lown) {
                    st_stream_v4(out + l0, e[0], e[1], e[2], e[3]);
                    st_stream_v4(out + l0 + 4, e[4], e[5], e[6], e[7]);
                } else {
#pragma unroll
                    for (uint32_t j = 0; j < kP; ++j)
                        if (l0 + j < lown) out[l0 + j] = (int32_t)e[j];
                    alive &= (1u << (lown - l0)) - 1;
                }
                if (FUSE) {
                    uint32_t nz = 0;
#pragma unroll
                    for (uint32_t j = 0; j < kP; ++j)
                        nz |= (l0 + j < lown && e[j] != 0 && !(e[j] & ALIVE)) ? (1u << j) : 0u;
                    if (nz) atomicOr(&bm[l0 >> 5], nz << (l0 & 31));
                }
                am |= alive << (r * kP);
            }
            push(am, hg * 1024);
          }
        }
        __syncwarp();  // all lanes done with `txt` before lane 0 refills it next iteration
        if constexpr (TXT) pred_bar = bar_slice;
        if (FUSE) {  // stage this slice's matches in position order (word w = positions 32w..32w+31)
            uint32_t any = 0;
            for (uint32_t w = lane; w < kBmWordsT; w += 32) any |= bm[w];
            uint32_t cnt = 0;
            if (__any_sync(~0u, any)) {  // most slices have no match (cfg2: 0.5 per slice)
                for (uint32_t w = lane; w < kBmWordsT; w += 32) cnt += __popc(bm[w]);
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(~0u, cnt, d);
            }
            if constexpr (DYN) {
                // every slice's count (bit 31: spilled, placed by the owner of its chunk after the scan);
                // a slice with matches is logged as [slice, count, entries] when the log has room
                const uint32_t eb = p.c.pid16 ? 4u : 8u;
                const uint32_t rec = log_record_bytes(cnt, eb);
                const bool logged = cnt && kMatchLog && log_off + rec <= p.c.log_pw;
                if (lane == 0) p.c.scnt[sl] = cnt | (cnt && !logged ? kSpillBit : 0u);
                if (cnt && !logged && LIST)  // out[] is valid only at matches: keep the slice's bitmap
                    for (uint32_t w = lane; w < kBmWordsT; w += 32) p.c.bitmap[sl * kBmWordsT + w] = bm[w];
                if (!logged) cnt = 0;  // nothing to log below
            }
            if (!cnt) {  // after a spill, list-only mode still needs this slice's (empty) bitmap
                if (!DYN && LIST && spill_rel != ~0u)
                    for (uint32_t w = lane; w < kBmWordsT; w += 32) p.c.bitmap[sl * kBmWordsT + w] = 0u;
            } else if (!DYN && wstaged == wcount && wcount + cnt <= p.c.stg) {  // (stg < 2^32)
#pragma unroll 1
                for (uint32_t w0 = 0; w0 < kBmWordsT; w0 += 32) {
                    uint32_t w = bm[w0 + lane];
                    const uint32_t c = __popc(w);
                    uint32_t incl = c;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_up_sync(~0u, incl, d);
                        if (lane >= (uint32_t)d) incl += y;
                    }
                    uint64_t r = wcount + incl - c;
                    while (w) {
                        const uint32_t bit = __ffs(w) - 1;
                        w &= w - 1;
                        const uint32_t l = (w0 + lane) * 32 + bit;
                        spos[r] = p.c.pos_base + base + l;
                        spid[r] = ld_cg_u32(out + l);  // written by this warp before the __syncwarp above
                        ++r;
                    }
                    wcount += __shfl_sync(~0u, incl, 31);
                }
                wstaged = (uint32_t)wcount;
            } else {
                const uint32_t eb = p.c.pid16 ? 4u : 8u;
                const uint32_t rec = log_record_bytes(cnt, eb);
                if (DYN || (kMatchLog && spill_rel == ~0u && log_off + rec <= p.c.log_pw)) {
                    // the staging is full: log the slice -- header [slice (relative), count], then
                    // (offset, pid) per match in position order -- to be placed after the prefix by a
                    // coalesced copy instead of re-reading out[]
                    uint32_t *hdr = reinterpret_cast<uint32_t *>(p.c.log + gw * p.c.log_pw + log_off);
                    uint32_t *ent = hdr + 4;
                    if (lane == 0) {
                        hdr[0] = (uint32_t)(DYN ? sl : sl - s_first);  // DYN: the absolute slice
                        hdr[1] = cnt;
                    }
                    // 128 positions per step: lane t owns positions 4t..4t+3 (one 16-byte read of the
                    // out[] cells this warp just wrote, L2 hits); ranks from three ballots, so a step's
                    // stores cover a contiguous rank range
                    uint32_t run = 0;
                    // the out[] cells of the next step are loaded while this step is written (__ldcg: L2,
                    // coherent with this warp's stores before the __syncwarp above; not volatile)
                    auto ld4 = [&](uint32_t ch) -> uint4 {
                        const uint32_t l0 = ch * 128 + lane * 4;
                        return ch < kSliceT / 128 && l0 + 4 <= lown ? __ldcg(reinterpret_cast<const uint4 *>(out + l0))
                                                                    : make_uint4(0, 0, 0, 0);
                    };
                    uint4 q = ld4(0);
#pragma unroll 1
                    for (uint32_t ch = 0; ch < kSliceT / 128; ++ch) {
                        const uint4 qn = ld4(ch + 1);
                        const uint32_t m = (bm[ch * 4 + (lane >> 3)] >> ((lane & 7) * 4)) & 0xFu;
                        if (__any_sync(~0u, m)) {
                            uint32_t tot;
                            uint32_t r = run + nibble_rank(m, lt, tot);
                            if (m) {
                                const uint32_t l0 = ch * 128 + lane * 4;
                                uint32_t v[4] = {q.x, q.y, q.z, q.w};
                                if (l0 + 4 > lown) {  // the slice's last owned cells
#pragma unroll
                                    for (int e = 0; e < 4; ++e) v[e] = (m >> e) & 1 ? (uint32_t)__ldcg(out + l0 + e) : 0u;
                                }
#pragma unroll
                                for (uint32_t e = 0; e < 4; ++e) {
                                    if (!((m >> e) & 1)) continue;
                                    if (p.c.pid16) ent[r] = (l0 + e) | (v[e] << 16);
                                    else reinterpret_cast<uint2 *>(ent)[r] = make_uint2(l0 + e, v[e]);
                                    ++r;
                                }
                            }
                            run += tot;
                        }
                        q = qn;
                    }
                    log_off += rec;
                } else {  // staging and log are full: spill, emit by re-reading out[] after the prefix
                    if (spill_rel == ~0u) spill_rel = (uint32_t)(sl - s_first);
                    if (LIST)  // out[] is valid only at matches: keep the slice's bitmap
                        for (uint32_t w = lane; w < kBmWordsT; w += 32) p.c.bitmap[sl * kBmWordsT + w] = bm[w];
                }
                wcount += cnt;
            }
        }
    }
    // TXT: a warp that had no slice never waited for the table copy; no CTA may retire while its
    // bulk copy into shared memory is in flight
    if (TXT && it == 0) mbar_wait(tab_bar, 0);
    if constexpr (DYN) {
        // every slice is matched: scan the per-slice counts (a contiguous chunk of slices per warp, the
        // warps' chunk totals by grid_prefix), then replay this warp's log records at their slices'
        // offsets; the spilled slices of each chunk are re-read from out[] by the chunk's warp
        grid_sync(p.c.ctl + 1);
        const uint64_t C = (p.nslices + TW - 1) / TW, lo = gw * C < p.nslices ? gw * C : p.nslices,
                       hi = lo + C < p.nslices ? lo + C : p.nslices;
        uint64_t sum = 0;
        for (uint64_t s = lo + lane; s < hi; s += 32) sum += p.c.scnt[s] & ~kSpillBit;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(~0u, sum, d);
        uint64_t run = grid_prefix<kMWarps>(sum, p.c.counts, p.c.d_count, s_wcount, s_woff);
        for (uint64_t s0 = lo; s0 < hi; s0 += 32) {
            const uint64_t s = s0 + lane;
            const uint32_t c = s < hi ? p.c.scnt[s] & ~kSpillBit : 0u;
            uint32_t incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(~0u, incl, d);
                if (lane >= (uint32_t)d) incl += y;
            }
            if (s < hi) p.c.soff[s] = run + incl - c;
            run += __shfl_sync(~0u, incl, 31);
        }
        grid_sync(p.c.ctl + 2);
        for (uint32_t off = 0; kMatchLog && off < log_off;) {
            const uint32_t *hdr = reinterpret_cast<const uint32_t *>(p.c.log + gw * p.c.log_pw + off);
            const uint32_t s = __ldcg(hdr), cnt = __ldcg(hdr + 1);
            replay_record(p.c, hdr + 4, cnt, __ldcg(p.c.soff + s), p.c.pos_base + (uint64_t)s * kSliceT, lane);
            off += log_record_bytes(cnt, p.c.pid16 ? 4u : 8u);
        }
        for (uint64_t s = lo; s < hi; ++s) {
            const uint32_t c = __ldcg(p.c.scnt + s);
            if (!(c & kSpillBit)) continue;
            const uint64_t a = s * kSliceT, b = a + kSliceT < p.n_own ? a + kSliceT : p.n_own;
            warp_stream<false>(
                p.c, a, b, __ldcg(p.c.soff + s),
                [&](uint64_t rr, uint64_t i, uint32_t val) { put_match(p.c, rr, p.c.pos_base + i, val); },
                LIST ? p.c.bitmap : nullptr);
        }
    } else if (FUSE) {  // grid-wide placement of the staged lists (cooperative launch: all CTAs resident)
        const uint64_t prefix = grid_prefix<kMWarps>(wcount, p.c.counts, p.c.d_count, s_wcount, s_woff);
        for (uint64_t i = lane; i < wstaged; i += 32) put_match(p.c, prefix + i, spos[i], spid[i]);
        // logged slices, in slice order: positions from each record's bitmap, pids from its list
        __syncwarp();
        uint64_t r0 = prefix + wstaged;
        for (uint32_t off = 0; kMatchLog && off < log_off;) {
            const uint32_t *hdr = reinterpret_cast<const uint32_t *>(p.c.log + gw * p.c.log_pw + off);
            const uint32_t rel = __ldcg(hdr), cnt = __ldcg(hdr + 1);  // this warp's own log (coherent L2 loads)
            replay_record(p.c, hdr + 4, cnt, r0, p.c.pos_base + (s_first + rel) * kSliceT, lane);
            r0 += cnt;
            off += log_record_bytes(cnt, p.c.pid16 ? 4u : 8u);
        }
        // spilled slices (dense matches): stream this warp's out[] from the first spilled slice
        // (list-only: masked by the spilled slice bitmaps, the scratch holds values only at matches)
        if (spill_rel != ~0u) {
            const uint64_t spill_first = s_first + spill_rel;
            const uint64_t lo = spill_first * kSliceT < p.n_own ? spill_first * kSliceT : p.n_own;
            const uint64_t hi = s_end * kSliceT < p.n_own ? s_end * kSliceT : p.n_own;
            warp_stream<false>(
                p.c, lo, hi, r0,  // after the staged and the logged matches
                [&](uint64_t rr, uint64_t i, uint32_t val) { put_match(p.c, rr, p.c.pos_base + i, val); },
                LIST ? p.c.bitmap : nullptr);
        }
    }
}

// ---------------------------------------------------------------------------------- host side
static uint32_t halo_words_for(int K, uint32_t maxlen) {
    const uint32_t need = (maxlen > (uint32_t)K ? maxlen : (uint32_t)K) + 16;  // +16: a window16 read
    return ((need + 63) / 64) * 4;
}

static int g_sms[64], g_optin[64];

static void dev_props(int device, int &sms, int &optin) {
    int &s = g_sms[device & 63], &o = g_optin[device & 63];
    if (!s) {
        cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, device);
        cudaDeviceGetAttribute(&o, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    }
    sms = s;
    optin = o;
}

#ifndef PFAC_WINDOW_MIN_SHARE
#define PFAC_WINDOW_MIN_SHARE 4
#endif
constexpr uint32_t kWindowMinShare = PFAC_WINDOW_MIN_SHARE;  // keep a row window only if rows <= this x window
constexpr size_t kStaticSmemReserve = 1024;
constexpr uint32_t kWinCells = kRowCells + (kMergedF ? 0 : 1);  // shared-memory cells per window row (T + F)
#ifndef PFAC_TXT_MAX_ROWS
#define PFAC_TXT_MAX_ROWS (1u << 20)
#endif
constexpr uint32_t kTxtMaxRows = PFAC_TXT_MAX_ROWS;  // larger automata: the text kernel with small slices
constexpr uint32_t kSliceSmall = 1024;  // the fused kernel's static shared arrays (grid_prefix)

static size_t match_smem(size_t table_bytes, uint32_t cell, uint32_t window, uint32_t slice_words,
                         bool bar = false, bool txt = false, uint32_t bm_words = kBmWords, bool jpre = false) {
    const size_t nw = (size_t)mt_for(bm_words * 32) / 32;
    return table_bytes + (size_t)window * kWinCells * cell + nw * warp_bytes(slice_words, bar, txt, bm_words, jpre) +
           16 + 2 * nw * 8;  // + the table mbarrier and grid_prefix's per-warp counts
}

MatchPlan plan_match(int device, const HostImage &h, uint32_t maxlen) {
    MatchPlan pl;
    int sms = 0, optin = 0;
    dev_props(device, sms, optin);
    pl.cell = h.cell;
    pl.slice_words = kSlice / 16 + halo_words_for(h.K2 > h.K ? h.K2 : h.K, maxlen);
    const size_t table = h.K2 ? (size_t)kFBBytes : ((size_t)1 << (2 * h.K)) * pl.cell;
    const size_t fixed = match_smem(table, pl.cell, 0, pl.slice_words) + kStaticSmemReserve;
    const size_t budget = (size_t)optin > fixed ? (size_t)optin - fixed : 0;
    uint32_t w = (uint32_t)(budget / (kWinCells * pl.cell)) & ~7u;
#ifdef PFAC_WINDOW_MAX
    if (w > (uint32_t)(PFAC_WINDOW_MAX)) w = (uint32_t)(PFAC_WINDOW_MAX) & ~7u;
#endif
    // A window that holds only a small share of the rows (huge uint32 automata, cfg4: 5.4 M states vs
    // ~3 k rows) costs more than it saves: lanes split between the shared and the global row path,
    // and its shared memory is better left to L1, which then caches the hot rows itself
    // (profiles/r01_ablations.md: window0 is 18% faster on cfg4, neutral elsewhere).
    if (w < h.rows && (uint64_t)h.rows > (uint64_t)kWindowMinShare * w) w = 0;
    pl.all_smem = w >= h.rows;
    pl.window = pl.all_smem ? h.rows : w;
    pl.smem = match_smem(table, pl.cell, pl.window, pl.slice_words);
    // barrier-mode variant (BAR): per-warp barrier bits take room from the row window
    const size_t fixed_b = match_smem(table, pl.cell, 0, pl.slice_words, true) + kStaticSmemReserve;
    const size_t budget_b = (size_t)optin > fixed_b ? (size_t)optin - fixed_b : 0;
    uint32_t wb = (uint32_t)(budget_b / (kWinCells * pl.cell)) & ~7u;
    if (wb < h.rows && (uint64_t)h.rows > (uint64_t)kWindowMinShare * wb) wb = 0;
#ifdef PFAC_WINDOW_MAX
    if (wb > (uint32_t)(PFAC_WINDOW_MAX)) wb = (uint32_t)(PFAC_WINDOW_MAX) & ~7u;
#endif
    pl.all_smem_bar = wb >= h.rows;
    pl.window_bar = pl.all_smem_bar ? h.rows : wb;
    pl.smem_bar = match_smem(table, pl.cell, pl.window_bar, pl.slice_words, true);
    // text-input variant (TXT): the ASCII staging buffers take the room of the row window; it exists
    // only when the filter image fits beside them (halo <= 112 bases at 896 threads per CTA)
    const size_t fixed_t = match_smem(table, pl.cell, 0, pl.slice_words, true, true) + kStaticSmemReserve;
    pl.txt_ok = h.K2 != 0 && (size_t)optin >= fixed_t;
    uint32_t wt = pl.txt_ok ? (uint32_t)(((size_t)optin - fixed_t) / (kWinCells * pl.cell)) & ~7u : 0u;
    if (wt < h.rows && (uint64_t)h.rows > (uint64_t)kWindowMinShare * wt) wt = 0;
#ifdef PFAC_WINDOW_MAX
    if (wt > (uint32_t)(PFAC_WINDOW_MAX)) wt = (uint32_t)(PFAC_WINDOW_MAX) & ~7u;
#endif
    pl.all_smem_txt = wt >= h.rows;
    pl.window_txt = pl.all_smem_txt ? h.rows : wt;
    pl.smem_txt = match_smem(table, pl.cell, pl.window_txt, pl.slice_words, true, true);
    // Measured (profiles/): the one-kernel text path wins where the step is HBM-bound
    // (cfg2 +11%, cfg3 +13%); it loses where walks dominate and the two-kernel plan holds every row in
    // shared memory (cfg5 -5%) or the rows are many and L1 caches them (cfg4, 5.4 M states: -12%;
    // the text buffers take that L1).
    pl.txt_pref = pl.txt_ok && !(pl.all_smem && !pl.all_smem_txt) && h.rows <= kTxtMaxRows;
    // the text kernel with 1024-position slices (uint32 images): half the staging, so L1 keeps room for
    // the rows of large automata (cfg4: 1.84 vs 2.16 ms for 2048-position slices, vs 1.92 for pack +
    // fused); 2% slower on cfg2-like automata, so it serves only those the 2048 plan is not used for
    pl.slice_words_1k = kSliceSmall / 16 + halo_words_for(h.K2 > h.K ? h.K2 : h.K, maxlen);
    const bool jpre = jpre_for(true, kSliceSmall / 32, pl.cell);
    const size_t fixed_k = match_smem(table, pl.cell, 0, pl.slice_words_1k, true, true, kSliceSmall / 32, jpre) +
                           kStaticSmemReserve;
    pl.txt1k_ok = h.K2 != 0 && (size_t)optin >= fixed_k;
    uint32_t wk = pl.txt1k_ok ? (uint32_t)(((size_t)optin - fixed_k) / (kWinCells * pl.cell)) & ~7u : 0u;
    if (wk < h.rows && (uint64_t)h.rows > (uint64_t)kWindowMinShare * wk) wk = 0;
#ifdef PFAC_WINDOW_MAX
    if (wk > (uint32_t)(PFAC_WINDOW_MAX)) wk = (uint32_t)(PFAC_WINDOW_MAX) & ~7u;
#endif
    pl.all_smem_txt1k = wk >= h.rows;
    pl.window_txt1k = pl.all_smem_txt1k ? h.rows : wk;
    pl.smem_txt1k = match_smem(table, pl.cell, pl.window_txt1k, pl.slice_words_1k, true, true, kSliceSmall / 32, jpre);
    pl.txt1k_pref = pl.txt1k_ok && !pl.txt_pref && pl.txt_ok && h.rows > kTxtMaxRows;
    pl.sms = sms;
    return pl;
}

static void fill_args(MatchArgs &a, const DeviceImage &img, const uint32_t *d_packed, uint64_t n_own,
                      uint64_t n_avail, int32_t *d_out, uint32_t slice = kSlice) {
    a.packed = d_packed;
    a.out = d_out;
    a.n_own = n_own;
    a.n_avail = n_avail;
    a.nslices = (n_own + slice - 1) / slice;
    a.avail_words = ((n_avail + 15) / 16 + 3) & ~3ull;
    a.J = img.d_J;
    a.T = img.d_T;
    a.F = img.d_F;
    a.window = img.plan.window;
    a.root = img.root;
    a.slice_words = slice == kSlice ? img.plan.slice_words : img.plan.slice_words_1k;
    a.short_pat = img.short_pat;
    a.bar_dead = (1u << (img.minlen < (uint32_t)kFBK ? img.minlen : (uint32_t)kFBK)) - 1;
    a.J2 = img.d_J2;
    a.FB = img.d_FB;
    a.K2 = (uint32_t)img.K2;
    a.mask2 = img.K2 ? (uint32_t)((1ull << (2 * img.K2)) - 1) : 0u;
    a.slices_per_warp = 0;
    a.inv = nullptr;
    a.c = CompactArgs{};
    a.text = nullptr;
    a.first_bad = nullptr;
    a.bad_all = nullptr;
    a.HR = reinterpret_cast<const uint4 *>(img.d_HR);
}

template <typename CT, bool LIST, uint32_t SL = kSlice, bool DYN = false>
static const void *txt_kernel(bool all_smem) {
    return all_smem ? (const void *)match_kernel<CT, false, sizeof(CT) == 2 ? kJumpK16 : kJumpK32, true, true, true, LIST, true, SL, DYN>
                    : (const void *)match_kernel<CT, true, sizeof(CT) == 2 ? kJumpK16 : kJumpK32, true, true, true, LIST, true, SL, DYN>;
}

template <bool FUSE>
static const void *kernel_for(const DeviceImage &img, bool bar, bool list = false, bool txt = false,
                              bool small = false, bool dyn = false) {
    const MatchPlan &pl = img.plan;
    if constexpr (FUSE) {
        if (txt && small && dyn) {  // text input, 1024-position slices claimed dynamically
            if (pl.cell == 2)
                return list ? txt_kernel<uint16_t, true, kSliceSmall, true>(pl.all_smem_txt1k)
                            : txt_kernel<uint16_t, false, kSliceSmall, true>(pl.all_smem_txt1k);
            return list ? txt_kernel<uint32_t, true, kSliceSmall, true>(pl.all_smem_txt1k)
                        : txt_kernel<uint32_t, false, kSliceSmall, true>(pl.all_smem_txt1k);
        }
        if (txt && small) {  // text input, 1024-position slices
            if (pl.cell == 2)
                return list ? txt_kernel<uint16_t, true, kSliceSmall>(pl.all_smem_txt1k)
                            : txt_kernel<uint16_t, false, kSliceSmall>(pl.all_smem_txt1k);
            return list ? txt_kernel<uint32_t, true, kSliceSmall>(pl.all_smem_txt1k)
                        : txt_kernel<uint32_t, false, kSliceSmall>(pl.all_smem_txt1k);
        }
        if (txt) {  // text input (filter path; checked by the launcher)
            if (pl.cell == 2) return list ? txt_kernel<uint16_t, true>(pl.all_smem_txt) : txt_kernel<uint16_t, false>(pl.all_smem_txt);
            return list ? txt_kernel<uint32_t, true>(pl.all_smem_txt) : txt_kernel<uint32_t, false>(pl.all_smem_txt);
        }
        if (list) {  // list-only (filter path only; checked by the launcher)
            if (bar) {
                if (pl.cell == 2) return pl.all_smem_bar ? (const void *)match_kernel<uint16_t, false, kJumpK16, true, true, true, true>
                                                         : (const void *)match_kernel<uint16_t, true, kJumpK16, true, true, true, true>;
                return pl.all_smem_bar ? (const void *)match_kernel<uint32_t, false, kJumpK32, true, true, true, true>
                                       : (const void *)match_kernel<uint32_t, true, kJumpK32, true, true, true, true>;
            }
            if (pl.cell == 2) return pl.all_smem ? (const void *)match_kernel<uint16_t, false, kJumpK16, true, true, false, true>
                                                 : (const void *)match_kernel<uint16_t, true, kJumpK16, true, true, false, true>;
            return pl.all_smem ? (const void *)match_kernel<uint32_t, false, kJumpK32, true, true, false, true>
                               : (const void *)match_kernel<uint32_t, true, kJumpK32, true, true, false, true>;
        }
    }
    if (bar) {  // barrier semantics (non-ACGT bytes present): filter path only
        if (pl.cell == 2) return pl.all_smem_bar ? (const void *)match_kernel<uint16_t, false, kJumpK16, FUSE, true, true>
                                                 : (const void *)match_kernel<uint16_t, true, kJumpK16, FUSE, true, true>;
        return pl.all_smem_bar ? (const void *)match_kernel<uint32_t, false, kJumpK32, FUSE, true, true>
                               : (const void *)match_kernel<uint32_t, true, kJumpK32, FUSE, true, true>;
    }
    if (pl.cell == 2 && img.K2) return pl.all_smem ? (const void *)match_kernel<uint16_t, false, kJumpK16, FUSE, true>
                                                   : (const void *)match_kernel<uint16_t, true, kJumpK16, FUSE, true>;
    if (pl.cell == 2) return pl.all_smem ? (const void *)match_kernel<uint16_t, false, kJumpK16, FUSE, false>
                                         : (const void *)match_kernel<uint16_t, true, kJumpK16, FUSE, false>;
    if (img.K2) return pl.all_smem ? (const void *)match_kernel<uint32_t, false, kJumpK32, FUSE, true>
                                   : (const void *)match_kernel<uint32_t, true, kJumpK32, FUSE, true>;
    return pl.all_smem ? (const void *)match_kernel<uint32_t, false, kJumpK32, FUSE, false>
                       : (const void *)match_kernel<uint32_t, true, kJumpK32, FUSE, false>;
}

// Launch with the image's L2 access-policy window (J2 persisting in L2) and, for the fused kernel,
// as a cooperative launch (every CTA resident: the grid-wide prefix spins on its predecessors).
static int launch(const DeviceImage &img, const void *fn, uint64_t grid, MatchArgs &a, bool cooperative,
                  cudaStream_t st, bool small = false) {
    const MatchPlan &pl = img.plan;
    const size_t smem = a.text ? (small ? pl.smem_txt1k : pl.smem_txt) : a.inv ? pl.smem_bar : pl.smem;
    if (a.text) a.window = small ? pl.window_txt1k : pl.window_txt;
    else if (a.inv) a.window = pl.window_bar;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(small ? mt_for(kSliceSmall) : kMT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (cooperative) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    if (img.d_J2 && img.l2_persist_bytes) {
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = img.d_base;  // J2, then the deep-first T rows
        attr[na].val.accessPolicyWindow.num_bytes = img.l2_persist_bytes;
        attr[na].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    void *args[] = {&a};
    e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

int launch_match(const DeviceImage &img, const uint32_t *d_packed, const uint16_t *d_inv, uint64_t n_own,
                 uint64_t n_avail, int32_t *d_out, void *stream) {
    if (n_own == 0) return cudaSuccess;
    MatchArgs a;
    fill_args(a, img, d_packed, n_own, n_avail, d_out);
    if (d_inv && !img.K2) return cudaErrorNotSupported;  // barrier mode lives on the filter path
    a.inv = d_inv;
    uint64_t grid = (a.nslices + kMWarps - 1) / kMWarps;
    if (grid > (uint64_t)img.plan.sms) grid = img.plan.sms;
    a.slices_per_warp = (a.nslices + grid * kMWarps - 1) / (grid * kMWarps);
    return launch(img, kernel_for<false>(img, d_inv != nullptr), grid, a, false, (cudaStream_t)stream);
}

// Fused match + compact: out[] and the ordered match list in one pass.
int launch_match_compact(const DeviceImage &img, uint32_t k, const uint32_t *d_packed, const uint16_t *d_inv,
                         uint64_t n_own, uint64_t n_avail, int32_t *d_out, uint64_t pos_base, uint64_t *d_pos,
                         uint32_t *d_pid, uint64_t capacity, uint64_t *d_count, uint64_t *d_hist, void *d_workspace,
                         void *stream, bool list_only, const uint8_t *d_text, uint64_t *d_first_bad,
                         const uint64_t *d_bad_all, bool small, bool dyn) {
    small = small && d_text;  // 1024-position slices: the text kernel only
    dyn = dyn && small;       // dynamic slice claiming: its 1024-position form only
    cudaStream_t st = (cudaStream_t)stream;
    if (d_first_bad && (d_text || n_own == 0)) {
        cudaError_t e = cudaMemsetAsync(d_first_bad, 0xFF, 8, st);
        if (e != cudaSuccess) return e;
    }
    if (n_own == 0) return cudaMemsetAsync(d_count, 0, 8, st);
    MatchArgs a;
    const uint32_t slice = small ? kSliceSmall : kSlice;
    fill_args(a, img, d_packed, n_own, n_avail, d_out, slice);
    if ((d_inv || list_only || d_text) && !img.K2) return cudaErrorNotSupported;  // filter path only
    if (d_text && !(small ? img.plan.txt1k_ok : img.plan.txt_ok)) return cudaErrorNotSupported;
    a.inv = d_inv;
    a.text = d_text;
    a.first_bad = d_text || d_bad_all ? d_first_bad : nullptr;
    a.bad_all = d_text ? nullptr : d_bad_all;
    const MatchPlan &pl = img.plan;
    const uint64_t grid = (uint64_t)pl.sms < a.nslices ? (uint64_t)pl.sms : a.nslices;
    const uint64_t warps = grid * (uint64_t)(mt_for(slice) / 32);
    a.slices_per_warp = (a.nslices + warps - 1) / warps + PFAC_SPW_PAD;
    CompactArgs &c = a.c;
    c.out = d_out;
    c.n = n_own;
    c.pos_base = pos_base;
    c.pos = d_pos;
    c.pid = d_pid;
    c.cap = capacity;
    c.d_count = d_count;
    c.k = k;
    c.hist = d_hist;
    c.counts = reinterpret_cast<uint64_t *>(d_workspace);
    const uint64_t entries = stage_entries(n_own);
    c.stg = entries / warps;
    c.stage_pos = c.counts + kGMax;
    c.stage_pid = reinterpret_cast<uint32_t *>(c.stage_pos + entries);
    c.bitmap = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(d_workspace) + kGMax * 8 +
                                            ((entries * 12 + 15) & ~15ull));
    c.log = reinterpret_cast<uint8_t *>(c.bitmap) + spill_bitmap_bytes(n_own);
    c.log_pw = kMatchLog ? (match_log_bytes(n_own) / warps) & ~15ull : 0;
    c.pid16 = k < 65536u;
    c.chunk = a.slices_per_warp * slice;
    // DYN: the per-slice offsets and counts after the logs (dyn_area_bytes), the claim counter and the
    // two grid barriers at the end of the CTA-count array
    c.soff = reinterpret_cast<uint64_t *>(c.log + match_log_bytes(n_own));
    c.scnt = reinterpret_cast<uint32_t *>(c.soff + a.nslices);
    c.ctl = c.counts + kGMax - 4;
    cudaError_t e = cudaMemsetAsync(c.counts, 0, dyn ? (size_t)kGMax * 8 : (size_t)grid * 8, st);
    if (e != cudaSuccess) return e;
    return launch(img, kernel_for<true>(img, d_inv != nullptr, list_only, d_text != nullptr, small, dyn), grid, a,
                  true, st, small);
}

}  // namespace pfac
