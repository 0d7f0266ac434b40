// Expand kernel: the longest-only match list -> every occurrence.
//
// PFAC reports only the longest pattern at each position.  Every pattern that occurs
// at i is a prefix of that longest one (its bases are the first bases of the same walk), so the
// all-occurrence set of the serial Aho-Corasick machine is
//   {(i, q) : (i, p) in the list, q on the prefix chain of p},
// where the chain of p is p, then the longest pattern that is a proper prefix of p, and so on
// (built on the host, pfac_internal.h `chain`).  Output order: ascending position, and at one
// position ascending pattern length (the order in which a walk from i completes them).
//
// One persistent cooperative grid; each warp owns a contiguous run of input entries:
//   pass 1: the warp sums the chain lengths of its entries;
//   grid_prefix: ordered offsets across warps and CTAs (compact_common.cuh);
//   pass 2: 32 entries per round; their outputs form one contiguous range, which the lanes fill
//           with stride 32 (coalesced 8-byte and 4-byte stores): output r of the round belongs to
//           the entry whose inclusive chain-length scan first exceeds r (a 5-step shuffle search),
//           and its pattern id is element t of that entry's flattened chain (prefix_flat, shortest
//           first, built on the host).  Long chains (cfg5: ~80 per match) and short ones (1) both
//           keep every lane busy.
// HBM-bound on the output: 12 B per occurrence written, 12 B per input entry read.
#include <cuda_runtime.h>

#include <cstdint>

#include "compact_common.cuh"
#include "pfac_internal.h"

namespace pfac {

constexpr int kEWarps = 16;  // warps per CTA

struct ExpandArgs {
    const uint64_t *pos;
    const uint32_t *pid;
    const uint64_t *count;  // device: entries in the input list (read at run time)
    uint64_t in_cap;        // entries readable from pos/pid
    const uint4 *prefix;    // k+1: (chain length, parent, flat base lo, hi)
    const uint32_t *flat;   // chains, shortest first
    uint32_t k;
    uint64_t *pos_all;
    uint32_t *pid_all;
    uint64_t cap;
    uint64_t *count_all;
    uint64_t *counts;       // kGMax flagged CTA totals (zeroed per call)
};

__global__ void __launch_bounds__(kEWarps * 32) expand_kernel(ExpandArgs a) {
    __shared__ uint64_t s_wcount[kEWarps], s_woff[kEWarps + 1];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t m = *a.count < a.in_cap ? *a.count : a.in_cap;
    const uint64_t nw = (uint64_t)gridDim.x * kEWarps, gw = (uint64_t)blockIdx.x * kEWarps + warp;
    const uint64_t per = ((m + nw - 1) / nw + 31) & ~31ull;
    const uint64_t lo = gw * per < m ? gw * per : m, hi = lo + per < m ? lo + per : m;
    uint64_t wcount = 0;
    for (uint64_t j = lo + lane; j < hi; j += 32) {
        const uint32_t p = __ldg(a.pid + j);
        wcount += p && p <= a.k ? __ldg(&a.prefix[p].x) : 0u;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) wcount += __shfl_xor_sync(~0u, wcount, d);
    uint64_t run = grid_prefix<kEWarps>(wcount, a.counts, a.count_all, s_wcount, s_woff);
    for (uint64_t j0 = lo; j0 < hi; j0 += 32) {
        const uint64_t j = j0 + lane;
        uint32_t c = 0;
        uint64_t x = 0, base = 0;
        if (j < hi) {
            const uint32_t p = __ldg(a.pid + j);
            if (p && p <= a.k) {
                const uint4 e = __ldg(&a.prefix[p]);
                c = e.x;
                base = e.z | ((uint64_t)e.w << 32);
            }
            x = __ldg(a.pos + j);
        }
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(~0u, incl, d);
            if (lane >= (uint32_t)d) incl += y;
        }
        const uint32_t total = __shfl_sync(~0u, incl, 31);
        const uint64_t first = base - (incl - c);  // flat index of output (incl - c) + t, per entry
        for (uint32_t r0 = 0; r0 < total; r0 += 32) {
            const uint32_t r = r0 + lane;
            // entry e = the first lane whose inclusive scan exceeds r
            uint32_t e = 0;
#pragma unroll
            for (uint32_t step = 16; step > 0; step >>= 1) {
                const uint32_t v = __shfl_sync(~0u, incl, e + step - 1);
                if (v <= r) e += step;
            }
            const uint64_t xe = __shfl_sync(~0u, x, e), fe = __shfl_sync(~0u, first, e);
            const uint64_t o = run + r;
            if (r < total && o < a.cap) {
                a.pos_all[o] = xe;
                a.pid_all[o] = __ldg(a.flat + fe + r);
            }
        }
        run += total;
    }
}

uint64_t expand_workspace_bytes() { return kGMax * sizeof(uint64_t); }

int launch_expand(const DeviceImage &img, uint32_t k, const uint64_t *d_pos, const uint32_t *d_pid,
                  const uint64_t *d_count, uint64_t in_capacity, uint64_t *d_pos_all, uint32_t *d_pid_all,
                  uint64_t capacity, uint64_t *d_count_all, void *d_workspace, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(d_workspace, 0, expand_workspace_bytes(), st);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expand_kernel, kEWarps * 32, 0);
    if (e != cudaSuccess) return e;
    int grid = img.plan.sms * (per_sm < 2 ? per_sm : 2);
    if (grid > (int)kGMax) grid = kGMax;
    if (grid < 1) return cudaErrorLaunchOutOfResources;
    ExpandArgs a;
    a.pos = d_pos;
    a.pid = d_pid;
    a.count = d_count;
    a.in_cap = in_capacity;
    a.prefix = reinterpret_cast<const uint4 *>(img.d_prefix);
    a.flat = img.d_prefix_flat;
    a.k = k;
    a.pos_all = d_pos_all;
    a.pid_all = d_pid_all;
    a.cap = capacity;
    a.count_all = d_count_all;
    a.counts = reinterpret_cast<uint64_t *>(d_workspace);
    void *args[] = {&a};
    // cooperative: grid_prefix waits on predecessor CTAs, so all CTAs must be resident
    return cudaLaunchCooperativeKernel((const void *)expand_kernel, dim3(grid), dim3(kEWarps * 32), args, 0, st);
}

}  // namespace pfac
