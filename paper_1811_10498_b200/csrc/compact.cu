// Compact kernel: the ordered match list {(pos_base + i, out[i]) : out[i] != 0}.
//
// Warp-ballot ranks inside a persistent cooperative grid, with no block barrier in the stream:
//  * every warp owns one contiguous chunk of out[] and streams it 512 ints at a time (four
//    coalesced 16-byte loads per lane, the next step's loads in flight while the current one is
//    ranked); a step with no match costs one vote;
//  * matches are ranked with three ballots per 16-byte load and appended, in order, to the warp's
//    staging area in global memory, and counted;
//  * once its chunk is done a CTA adds up its warps' counts, publishes the CTA count, sums the counts
//    of CTAs 0..b-1 (all co-resident -- cooperative launch -- so there is no chained look-back) and
//    its warps copy their staged entries to the final positions.  Only a warp whose matches
//    overflow its staging area re-reads its chunk (dense outputs).
// HBM-bound: 4 B read per base + 12 B written per match.
#include <cuda_runtime.h>

#include <cstdint>

#include "pfac_internal.h"
#include "ptx.cuh"

namespace pfac {

constexpr int kCT = 256;                  // threads per CTA
constexpr int kCW = kCT / 32;             // warps per CTA
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
};

__device__ __forceinline__ void load_step(const int32_t *out, uint64_t n, uint64_t b, uint32_t lane, uint4 (&v)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint64_t idx = b + (uint64_t)(32 * q + lane) * 4;
        if (idx + 4 <= n) {
            v[q] = ld_stream_v4(out + idx);
        } else {
            v[q].x = idx + 0 < n ? (uint32_t)out[idx + 0] : 0u;
            v[q].y = idx + 1 < n ? (uint32_t)out[idx + 1] : 0u;
            v[q].z = idx + 2 < n ? (uint32_t)out[idx + 2] : 0u;
            v[q].w = 0;
        }
    }
}

// Streams [lo, hi) of out[] with one warp; emit(rank, position, value) for every nonzero entry in
// position order, rank counted from wbase.  Returns the number of nonzero entries.
template <typename Emit>
__device__ __forceinline__ uint64_t warp_stream(const CompactArgs &a, uint64_t lo, uint64_t hi, uint64_t wbase,
                                                Emit emit) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1;
    uint64_t local = 0;
    uint4 v[4], vn[4];
    if (lo < hi) load_step(a.out, a.n, lo, lane, v);
    for (uint64_t b = lo; b < hi; b += kStep) {
        if (b + kStep < hi) load_step(a.out, a.n, b + kStep, lane, vn);
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

__global__ void __launch_bounds__(kCT) compact_kernel(const CompactArgs a) {
    __shared__ uint64_t s_wcount[kCW], s_woff[kCW];
    __shared__ uint64_t s_prefix;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * kCW + warp;
    const uint64_t lo = gw * a.chunk < a.n ? gw * a.chunk : a.n;
    const uint64_t hi = lo + a.chunk < a.n ? lo + a.chunk : a.n;
    uint64_t *spos = a.stage_pos + gw * a.stg;
    uint32_t *spid = a.stage_pid + gw * a.stg;
    const uint64_t stg = a.stg, pos_base = a.pos_base;

    // pass 1: count + stage in order
    const uint64_t local = warp_stream(a, lo, hi, 0, [&](uint64_t r, uint64_t i, uint32_t val) {
        if (r < stg) {
            spos[r] = pos_base + i;
            spid[r] = val;
        }
    });
    if (lane == 0) s_wcount[warp] = local;
    __syncthreads();
    if (warp == 0) {
        const uint64_t c = lane < kCW ? s_wcount[lane] : 0;
        uint64_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t y = __shfl_up_sync(~0u, incl, d);
            if (lane >= (uint32_t)d) incl += y;
        }
        if (lane < kCW) s_woff[lane] = incl - c;
        const uint64_t cta_total = __shfl_sync(~0u, incl, 31);
        if (lane == 0) st_release_u64(a.counts + blockIdx.x, kFlag | cta_total);
        // exclusive prefix over the (co-resident) predecessor CTAs
        uint64_t sum = 0;
        for (uint32_t j = 0; j < blockIdx.x; j += 32) {
            const uint32_t q = j + lane;
            uint64_t x = 0;
            if (q < blockIdx.x) {
                do x = ld_acquire_u64(a.counts + q);
                while (!(x & kFlag));
            }
            sum += x & ~kFlag;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(~0u, sum, d);
        if (lane == 0) {
            s_prefix = sum;
            if (blockIdx.x == gridDim.x - 1) *a.d_count = sum + cta_total;
        }
    }
    __syncthreads();
    const uint64_t prefix = s_prefix + s_woff[warp];
    auto put = [&](uint64_t r, uint64_t p, uint32_t val) {
        if (r < a.cap) {
            a.pos[r] = p;
            a.pid[r] = val;
        }
        if (a.hist && val <= a.k) atomicAdd(reinterpret_cast<unsigned long long *>(a.hist + val), 1ull);
    };
    // pass 2: place the staged entries (or re-read the chunk if they overflowed the staging area)
    if (local <= stg) {
        for (uint64_t i = lane; i < local; i += 32) put(prefix + i, spos[i], spid[i]);
    } else {
        warp_stream(a, lo, hi, prefix, [&](uint64_t r, uint64_t i, uint32_t val) { put(r, pos_base + i, val); });
    }
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
    const uint64_t steps = (n + kStep - 1) / kStep;
    uint64_t G = (uint64_t)sms * (per_sm < 1 ? 1 : per_sm);
    if (G > kGMax) G = kGMax;
    if (G * kCW > steps) G = (steps + kCW - 1) / kCW;
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
    const uint64_t warps = G * kCW;
    a.stg = entries / warps;
    a.stage_pos = a.counts + kGMax;
    a.stage_pid = reinterpret_cast<uint32_t *>(a.stage_pos + entries);
    a.chunk = ((steps + warps - 1) / warps) * kStep;
    e = cudaMemsetAsync(a.counts, 0, (size_t)G * 8, st);
    if (e != cudaSuccess) return e;
    void *args[] = {&a};
    e = cudaLaunchCooperativeKernel((const void *)compact_kernel, dim3((unsigned)G), dim3(kCT), args, 0, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace pfac
