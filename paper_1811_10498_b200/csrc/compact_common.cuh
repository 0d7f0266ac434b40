// Pieces of the stream compaction shared by compact_kernel (compact.cu) and the fused
// match+compact kernel (match.cu).
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace pfac {

constexpr uint32_t kStep = 512;           // ints per warp step (4 x 16 B per lane)
constexpr uint32_t kGMax = 2048;          // max CTAs (size of the CTA-count array)
constexpr uint64_t kStageBytes = 32ull << 20;
constexpr uint64_t kFlag = 1ull << 63;

struct CompactArgs {
    const int32_t *out;
    uint64_t n, pos_base;
    uint64_t *pos;
    uint32_t *pid;
    uint64_t cap;
    uint64_t *d_count;
    uint32_t k;
    uint64_t *hist;
    uint64_t *counts;     // kGMax flagged CTA counts (zeroed per call)
    uint64_t *stage_pos;  // total_warps * stg entries
    uint32_t *stage_pid;
    uint64_t stg;         // staging entries per warp
    uint64_t chunk;       // ints per warp (multiple of kStep)
    uint32_t *bitmap;     // fused kernel: match bitmaps of the slices its staging and log could not hold
    uint8_t *log;         // fused kernel: per-warp match logs (log_pw bytes each, 16-byte multiple)
    uint64_t log_pw;
    uint32_t pid16;       // log pids as uint16 (every id < 2^16)
    uint32_t *scnt;       // DYN: per-slice match count (bit 31: spilled)
    uint64_t *soff;       // DYN: per-slice list offset (the scan of scnt)
    uint64_t *ctl;        // DYN: [0] slice claim counter, [1], [2] grid barriers (zeroed per call)
};

// NC: out[] was written by an earlier launch (read-only here: ld.global.nc); otherwise (the fused
// kernels' spill path re-reading cells written in this launch) coherent L2 loads.
template <bool NC>
__device__ __forceinline__ void load_step(const int32_t *out, uint64_t n, uint64_t b, uint32_t lane, uint4 (&v)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint64_t idx = b + (uint64_t)(32 * q + lane) * 4;
        if (idx + 4 <= n) {
            v[q] = NC ? ld_stream_v4(out + idx) : ld_cg_v4(out + idx);
        } else {
            v[q].x = idx + 0 < n ? (NC ? (uint32_t)out[idx + 0] : ld_cg_u32(out + idx + 0)) : 0u;
            v[q].y = idx + 1 < n ? (NC ? (uint32_t)out[idx + 1] : ld_cg_u32(out + idx + 1)) : 0u;
            v[q].z = idx + 2 < n ? (NC ? (uint32_t)out[idx + 2] : ld_cg_u32(out + idx + 2)) : 0u;
            v[q].w = 0;
        }
    }
}

// Streams [lo, hi) of out[] with one warp; emit(rank, position, value) for every nonzero entry in
// position order, rank counted from wbase.  Returns the number of nonzero entries.
// bits (nullable): a position-indexed bitmap (bit i%32 of word i/32); when given, only entries whose
// bit is set count (the list-only kernel's out[] scratch holds values only there).  lo is a multiple of 32.
template <bool NC, typename Emit>
__device__ __forceinline__ uint64_t warp_stream(const CompactArgs &a, uint64_t lo, uint64_t hi, uint64_t wbase,
                                                Emit emit, const uint32_t *bits = nullptr) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1;
    uint64_t local = 0;
    uint4 v[4], vn[4];
    if (lo < hi && !bits) load_step<NC>(a.out, a.n, lo, lane, v);
    for (uint64_t b = lo; b < hi; b += kStep) {
        if (b + kStep < hi && !bits) load_step<NC>(a.out, a.n, b + kStep, lane, vn);
        if (bits) {  // lane's 4 positions b + 128q + 4 lane .. +3: a nibble of word (b + 128q)/32 + lane/8;
                     // only the cells whose bit is set are read (the others were never written)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint64_t p0 = b + 128 * q + 4 * lane;
                const uint32_t m = p0 < hi ? (ld_cg_u32(reinterpret_cast<const int32_t *>(bits + (p0 >> 5))) >>
                                              (p0 & 31)) & 0xFu
                                           : 0u;
                v[q].x = m & 1 ? ld_cg_u32(a.out + p0) : 0u;
                v[q].y = m & 2 ? ld_cg_u32(a.out + p0 + 1) : 0u;
                v[q].z = m & 4 ? ld_cg_u32(a.out + p0 + 2) : 0u;
                v[q].w = m & 8 ? ld_cg_u32(a.out + p0 + 3) : 0u;
            }
        }
        uint32_t any = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) any |= v[q].x | v[q].y | v[q].z | v[q].w;
        if (__any_sync(~0u, any)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t vals[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
                const uint32_t c = (vals[0] != 0) + (vals[1] != 0) + (vals[2] != 0) + (vals[3] != 0);
                const uint32_t b0 = __ballot_sync(~0u, c & 1), b1 = __ballot_sync(~0u, c & 2),
                               b2 = __ballot_sync(~0u, c & 4);
                if (b0 | b1 | b2) {
                    uint64_t r = wbase + local + __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
                    const uint64_t idx = b + (uint64_t)(32 * q + lane) * 4;
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (vals[e]) emit(r++, idx + e, vals[e]);
                    local += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = vn[q];
    }
    return local;
}

// Grid-level placement after every warp of every (co-resident) CTA has counted its matches:
// returns this warp's global exclusive offset.  Block-uniform call; NW = warps per CTA (<= 32).
// The CTA total is published in counts[blockIdx.x] (flag | count); the last CTA writes *d_count.
template <int NW>
__device__ __forceinline__ uint64_t grid_prefix(uint64_t warp_count, uint64_t *counts, uint64_t *d_count,
                                                uint64_t *s_wcount /*[NW]*/, uint64_t *s_woff /*[NW + 1]*/) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_wcount[warp] = warp_count;
    __syncthreads();
    if (warp == 0) {
        const uint64_t c = lane < (uint32_t)NW ? s_wcount[lane] : 0;
        uint64_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t y = __shfl_up_sync(~0u, incl, d);
            if (lane >= (uint32_t)d) incl += y;
        }
        const uint64_t cta_total = __shfl_sync(~0u, incl, 31);
        if (lane == 0) st_release_u64(counts + blockIdx.x, kFlag | cta_total);
        uint64_t sum = 0;  // exclusive prefix over the predecessor CTAs (co-resident: no deadlock)
        for (uint32_t j = 0; j < blockIdx.x; j += 32) {
            const uint32_t q = j + lane;
            uint64_t x = 0;
            if (q < blockIdx.x) {
                do x = ld_acquire_u64(counts + q);
                while (!(x & kFlag));
            }
            sum += x & ~kFlag;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(~0u, sum, d);
        if (lane < (uint32_t)NW) s_woff[lane] = sum + incl - c;
        if (lane == 0 && blockIdx.x == gridDim.x - 1) *d_count = sum + cta_total;
    }
    __syncthreads();
    return s_woff[warp];
}

// The final write of one match (rank r): list entry (if within capacity) + histogram.
__device__ __forceinline__ void put_match(const CompactArgs &a, uint64_t r, uint64_t p, uint32_t val) {
    if (r < a.cap) {
        a.pos[r] = p;
        a.pid[r] = val;
    }
    if (a.hist && val <= a.k) atomicAdd(reinterpret_cast<unsigned long long *>(a.hist + val), 1ull);
}

// Workspace of the fused kernel's spilled slice bitmaps: one bit per position, whole slices
// (a slice is <= 65536 positions), 16-byte multiple.
inline uint64_t spill_bitmap_bytes(uint64_t n) { return (((n + 65536) / 32) * 4 + 15) & ~15ull; }

// The fused kernels' per-warp match logs: a slice's record is a header (slice, count) and one entry
// per match in position order -- (offset in the slice | pid << 16) as 4 bytes when every id fits in
// 16 bits, else (offset, pid) as 8 bytes -- so placing it after the prefix is a coalesced copy.
// 5/4 bytes per position: every slice of a warp's run fits up to ~31% (4-byte entries) / ~15%
// (8-byte) match density; denser runs spill their remaining slices to the out[] re-read.
inline uint64_t match_log_bytes(uint64_t n) { return (n + n / 4 + 15) & ~15ull; }
__host__ __device__ constexpr uint32_t log_record_bytes(uint32_t cnt, uint32_t entry_bytes) {
    return (16 + cnt * entry_bytes + 15) & ~15u;
}

// The dynamic-slice text kernel's per-slice arrays (1024-position slices): list offset (8 B) and
// count word (4 B) per slice, after the match logs.
inline uint64_t dyn_area_bytes(uint64_t n) { return (((n + 1023) / 1024) * 12 + 15) & ~15ull; }

inline uint64_t stage_entries(uint64_t n) {
    const uint64_t cap = kStageBytes / 12;
    return n < cap ? n : cap;
}

}  // namespace pfac
