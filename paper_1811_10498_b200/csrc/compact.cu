// Compact kernel: the ordered match list {(pos_base + i, out[i]) : out[i] != 0}.
//
// Warp-ballot ranks + a block scan of the warp counts, inside a persistent cooperative grid:
//  * CTA b owns one contiguous chunk of out[] and streams it tile by tile (4096 ints per tile, the
//    next tile's 16-byte loads in flight while the current one is ranked), appending its matches in
//    order to a CTA-private staging area and counting them;
//  * it publishes its count, then sums the counts of CTAs 0..b-1 (all co-resident -- cooperative
//    launch -- so there is no chained look-back), and copies the staged entries to their final
//    place.  Only a CTA whose matches overflow its staging area re-reads its chunk (dense outputs).
// HBM-bound: 4 B read per base + 12 B written per match.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "pfac_internal.h"
#include "ptx.cuh"

namespace pfac {

constexpr int kCT = 256;                     // threads per CTA
constexpr int kCI = 4;                       // int4 loads per thread per tile
constexpr int kCW = kCT / 32;                // warps
constexpr uint32_t kCTile = kCT * kCI * 4;   // 4096 ints per tile
constexpr uint32_t kGMax = 1024;             // max CTAs (counts array size)
constexpr uint64_t kStageBytes = 16ull << 20;
constexpr uint64_t kFlag = 1ull << 63;
static_assert(kCI * kCW == 32, "one warp scans the per-(load, warp) counts");

struct CompactArgs {
    const int32_t *out;
    uint64_t n, pos_base;
    uint64_t *pos;
    uint32_t *pid;
    uint64_t cap;
    uint64_t *d_count;
    uint32_t k;
    uint64_t *hist;
    uint64_t *counts;     // kGMax flagged counts (zeroed per call)
    uint64_t *stage_pos;  // gridDim.x * stg entries
    uint32_t *stage_pid;
    uint64_t stg;         // staging entries per CTA
    uint64_t chunk;       // ints per CTA (multiple of kCTile)
};

struct Shared {
    uint32_t cnt[32], off[32], tot;
    uint64_t prefix;
};

__device__ __forceinline__ void load_tile(const int32_t *out, uint64_t n, uint64_t tb, uint32_t tid, uint4 (&v)[kCI]) {
#pragma unroll
    for (int i = 0; i < kCI; ++i) {
        const uint64_t idx = tb + ((uint64_t)i * kCT + tid) * 4;
        if (idx + 4 <= n) {
            v[i] = ld_stream_v4(out + idx);
        } else {
            v[i].x = idx + 0 < n ? (uint32_t)out[idx + 0] : 0u;
            v[i].y = idx + 1 < n ? (uint32_t)out[idx + 1] : 0u;
            v[i].z = idx + 2 < n ? (uint32_t)out[idx + 2] : 0u;
            v[i].w = 0;
        }
    }
}

// Ranks the nonzero entries of one tile (already loaded in v) and hands each one to emit(rank, pos, val)
// with rank counted from `wbase`.  Returns the tile's match count.  Block-uniform call.
template <typename Emit>
__device__ __forceinline__ uint32_t rank_tile(Shared &sh, const uint4 (&v)[kCI], uint64_t tb, uint64_t wbase,
                                              uint32_t tid, Emit emit) {
    const uint32_t lane = tid & 31, warp = tid >> 5, lt = (1u << lane) - 1;
    uint32_t any = 0;
#pragma unroll
    for (int i = 0; i < kCI; ++i) any |= v[i].x | v[i].y | v[i].z | v[i].w;
    if (!__syncthreads_or(any)) return 0;  // common case: no match in the tile
    uint32_t lex[kCI];
#pragma unroll
    for (int i = 0; i < kCI; ++i) {
        const uint32_t c = (v[i].x != 0) + (v[i].y != 0) + (v[i].z != 0) + (v[i].w != 0);
        const uint32_t b0 = __ballot_sync(~0u, c & 1), b1 = __ballot_sync(~0u, c & 2), b2 = __ballot_sync(~0u, c & 4);
        lex[i] = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
        if (lane == 0) sh.cnt[i * kCW + warp] = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t x = sh.cnt[lane];
        uint32_t incl = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(~0u, incl, d);
            if (lane >= (uint32_t)d) incl += y;
        }
        sh.off[lane] = incl - x;
        if (lane == 31) sh.tot = incl;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kCI; ++i) {
        const uint32_t vals[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
        if ((vals[0] | vals[1] | vals[2] | vals[3]) == 0) continue;
        uint64_t r = wbase + sh.off[i * kCW + warp] + lex[i];
        const uint64_t idx = tb + ((uint64_t)i * kCT + tid) * 4;
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (vals[e]) emit(r++, idx + e, vals[e]);
    }
    const uint32_t tot = sh.tot;
    __syncthreads();  // sh.cnt / sh.off / sh.tot are reused by the next tile
    return tot;
}

template <typename Emit>
__device__ __forceinline__ uint64_t stream_chunk(Shared &sh, const CompactArgs &a, uint64_t lo, uint64_t hi,
                                                 uint64_t wbase, Emit emit) {
    const uint32_t tid = threadIdx.x;
    uint64_t local = 0;
    uint4 v[kCI], vn[kCI];
    if (lo < hi) load_tile(a.out, a.n, lo, tid, v);
    for (uint64_t tb = lo; tb < hi; tb += kCTile) {
        if (tb + kCTile < hi) load_tile(a.out, a.n, tb + kCTile, tid, vn);
        local += rank_tile(sh, v, tb, wbase + local, tid, emit);
#pragma unroll
        for (int i = 0; i < kCI; ++i) v[i] = vn[i];
    }
    return local;
}

__global__ void __launch_bounds__(kCT) compact_kernel(const CompactArgs a) {
    __shared__ Shared sh;
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    const uint32_t b = blockIdx.x;
    const uint64_t lo = (uint64_t)b * a.chunk < a.n ? (uint64_t)b * a.chunk : a.n;
    const uint64_t hi = lo + a.chunk < a.n ? lo + a.chunk : a.n;
    uint64_t *spos = a.stage_pos + (uint64_t)b * a.stg;
    uint32_t *spid = a.stage_pid + (uint64_t)b * a.stg;
    const uint64_t stg = a.stg, pos_base = a.pos_base;

    // pass 1: count + stage in order
    const uint64_t local = stream_chunk(sh, a, lo, hi, 0, [&](uint64_t r, uint64_t i, uint32_t val) {
        if (r < stg) {
            spos[r] = pos_base + i;
            spid[r] = val;
        }
    });
    if (tid == 0) st_release_u64(a.counts + b, kFlag | local);
    // exclusive prefix over the (co-resident) predecessors
    if (tid < 32) {
        uint64_t sum = 0;
        for (uint32_t j = 0; j < b; j += 32) {
            const uint32_t q = j + lane;
            uint64_t c = 0;
            if (q < b) {
                do c = ld_acquire_u64(a.counts + q);
                while (!(c & kFlag));
            }
            sum += c & ~kFlag;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(~0u, sum, d);
        if (lane == 0) sh.prefix = sum;
    }
    __syncthreads();
    const uint64_t prefix = sh.prefix;
    auto put = [&](uint64_t r, uint64_t p, uint32_t val) {
        if (r < a.cap) {
            a.pos[r] = p;
            a.pid[r] = val;
        }
        if (a.hist && val <= a.k) atomicAdd(reinterpret_cast<unsigned long long *>(a.hist + val), 1ull);
    };
    // pass 2: place the staged entries (or re-read the chunk if they overflowed the staging area)
    if (local <= stg) {
        for (uint64_t i = tid; i < local; i += kCT) put(prefix + i, spos[i], spid[i]);
    } else {
        stream_chunk(sh, a, lo, hi, prefix, [&](uint64_t r, uint64_t i, uint32_t val) { put(r, pos_base + i, val); });
    }
    if (b == gridDim.x - 1 && tid == 0) *a.d_count = prefix + local;
}

static uint64_t stage_entries(uint64_t n) {
    const uint64_t cap = kStageBytes / 12;
    return n < cap ? n : cap;
}

uint64_t compact_workspace_bytes(uint64_t n) {
    return (uint64_t)kGMax * 8 + ((stage_entries(n) * 12 + 15) & ~15ull);
}

int launch_compact(const int32_t *d_out, uint64_t n, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                   uint64_t capacity, uint64_t *d_count, uint32_t k, uint64_t *d_hist, void *d_workspace,
                   void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) return cudaMemsetAsync(d_count, 0, 8, st);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, compact_kernel, kCT, 0);
    if (e != cudaSuccess) return e;
    const uint64_t tiles = (n + kCTile - 1) / kCTile;
    uint64_t G = (uint64_t)sms * (per_sm > 4 ? 4 : per_sm);
    if (G > kGMax) G = kGMax;
    if (G > tiles) G = tiles;
    if (G == 0) G = 1;
    CompactArgs a;
    a.out = d_out;
    a.n = n;
    a.pos_base = pos_base;
    a.pos = d_pos;
    a.pid = d_pid;
    a.cap = capacity;
    a.d_count = d_count;
    a.k = k;
    a.hist = d_hist;
    a.counts = reinterpret_cast<uint64_t *>(d_workspace);
    const uint64_t entries = stage_entries(n);
    a.stg = entries / G;
    a.stage_pos = a.counts + kGMax;
    a.stage_pid = reinterpret_cast<uint32_t *>(a.stage_pos + entries);
    a.chunk = ((tiles + G - 1) / G) * kCTile;
    e = cudaMemsetAsync(a.counts, 0, (size_t)G * 8, st);
    if (e != cudaSuccess) return e;
    void *args[] = {&a};
    e = cudaLaunchCooperativeKernel((const void *)compact_kernel, dim3((unsigned)G), dim3(kCT), args, 0, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace pfac
