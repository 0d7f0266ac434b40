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

#include "compact_common.cuh"
#include "pfac_internal.h"
#include "ptx.cuh"

namespace pfac {

constexpr int kCT = 256;                  // threads per CTA
constexpr int kCW = kCT / 32;             // warps per CTA

__global__ void __launch_bounds__(kCT) compact_kernel(const CompactArgs a) {
    __shared__ uint64_t s_wcount[kCW], s_woff[kCW];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * kCW + warp;
    const uint64_t lo = gw * a.chunk < a.n ? gw * a.chunk : a.n;
    const uint64_t hi = lo + a.chunk < a.n ? lo + a.chunk : a.n;
    uint64_t *spos = a.stage_pos + gw * a.stg;
    uint32_t *spid = a.stage_pid + gw * a.stg;
    const uint64_t stg = a.stg, pos_base = a.pos_base;

    // pass 1: count + stage in order
    const uint64_t local = warp_stream<true>(a, lo, hi, 0, [&](uint64_t r, uint64_t i, uint32_t val) {
        if (r < stg) {
            spos[r] = pos_base + i;
            spid[r] = val;
        }
    });
    const uint64_t prefix = grid_prefix<kCW>(local, a.counts, a.d_count, s_wcount, s_woff);
    auto put = [&](uint64_t r, uint64_t p, uint32_t val) { put_match(a, r, p, val); };
    // pass 2: place the staged entries (or re-read the chunk if they overflowed the staging area)
    if (local <= stg) {
        for (uint64_t i = lane; i < local; i += 32) put(prefix + i, spos[i], spid[i]);
    } else {
        warp_stream<true>(a, lo, hi, prefix, [&](uint64_t r, uint64_t i, uint32_t val) { put(r, pos_base + i, val); });
    }
}

// [counts kGMax | staging pos | staging pid | spilled slice bitmaps (fused kernel) | match logs (fused kernel)]
uint64_t compact_workspace_bytes(uint64_t n) {
    return (uint64_t)kGMax * 8 + ((stage_entries(n) * 12 + 15) & ~15ull) + spill_bitmap_bytes(n) + match_log_bytes(n) +
           dyn_area_bytes(n);
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
