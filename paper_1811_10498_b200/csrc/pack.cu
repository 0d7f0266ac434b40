// Pack kernel: ASCII bases -> 2-bit codes + validation status.
// HBM-bound: 1 B read + 0.25 B written per base.
#include <cuda_runtime.h>

#include <cstdint>

#include "pfac_internal.h"
#include "pack_common.cuh"
#include "ptx.cuh"

namespace pfac {

// ============================================================================ pack
// A warp packs 128 consecutive words (2048 bases) per iteration: for q = 0..3 lane l reads the 16
// bytes of word 32q + l (one coalesced 512-byte load per q) and writes that word (a coalesced
// 128-byte store per q).  Grid-stride over the padded word range.
// inv (nullable): one bit per base, set for a byte outside ACGTacgt (the barriers of reading R5),
// as one uint16 per packed word; words past the text are written as 0 (their bytes count as valid).
// first_bad: a warp reports only the first bad index it meets (its iterations ascend), one atomicMin,
// so a text full of barriers (FASTA newlines) costs one atomic per warp.
#ifndef PFAC_PACK_MINB
#define PFAC_PACK_MINB 8  // 8 CTAs of 256 threads per SM: caps the kernel at 32 registers
#endif
template <bool INV>
__global__ void __launch_bounds__(256, PFAC_PACK_MINB) pack_kernel(const uint8_t *__restrict__ text, uint64_t n,
                                                   uint32_t *__restrict__ packed, uint64_t nwords,
                                                   uint64_t *first_bad, bool aligned, uint16_t *__restrict__ inv) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    bool wdone = false;  // warp-uniform: this warp has reported its first bad byte
    for (uint64_t wb = warp * 128; wb < nwords; wb += nwarps * 128) {
        uint32_t bad = 0;  // nonzero: one of this lane's 4 words holds a byte outside ACGTacgt
        uint32_t mlo = 0, mhi = 0;  // INV: the 4 words' 16-bit masks (q = 0, 1 in mlo; 2, 3 in mhi)
        if (aligned && (wb + 128) * 16 <= n) {
            uint4 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = ld_stream_v4(text + (wb + 32 * q + lane) * 16);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if constexpr (INV) {
                    uint32_t bq = 0;
                    packed[wb + 32 * q + lane] = pack16(v[q].x, v[q].y, v[q].z, v[q].w, bq);
                    const uint32_t m = (bq & kBadMask) ? bad16(v[q]) : 0u;
                    inv[wb + 32 * q + lane] = (uint16_t)m;
                    if (q < 2) mlo |= m << (16 * q);
                    else mhi |= m << (16 * (q - 2));
                    bad |= m;
                } else {  // one residue accumulator (tested against kBadMask below)
                    packed[wb + 32 * q + lane] = pack16(v[q].x, v[q].y, v[q].z, v[q].w, bad);
                }
            }
        } else {
#pragma unroll 1
            for (int q = 0; q < 4; ++q) {
                const uint64_t w = wb + 32 * q + lane;
                if (w >= nwords) break;
                uint32_t word = 0, m = 0;
                for (int j = 0; j < 16; ++j) {
                    const uint64_t i = w * 16 + j;
                    if (i < n) {
                        const uint8_t b = text[i];
                        if (!valid_byte(b)) m |= 1u << j;
                        const uint32_t t = (b >> 1) & 3u;
                        word |= (t ^ (t >> 1)) << (2 * j);
                    }
                }
                bad |= m ? 1u : 0u;  // bit 0 lies in kBadMask
                packed[w] = word;
                if (INV) {
                    inv[w] = (uint16_t)m;
                    if (q < 2) mlo |= m << (16 * q);
                    else mhi |= m << (16 * (q - 2));
                }
            }
        }
        if (!INV) bad &= kBadMask;  // INV: bad already holds exact masks
        if (first_bad && !wdone && __any_sync(~0u, bad != 0)) {
            // rare (once per warp): this lane's first bad byte (its words ascend with q)
            uint32_t off = ~0u;
            if constexpr (INV) {  // from the masks in registers
                for (uint32_t q = 0; q < 4 && off == ~0u; ++q) {
                    const uint32_t m = ((q < 2 ? mlo : mhi) >> (16 * (q & 1))) & 0xFFFFu;
                    if (m) off = (32u * q + lane) * 16u + (__ffs(m) - 1);
                }
            } else {  // rescan this lane's bytes (pfac_pack_async on a text with barriers)
                for (uint32_t q = 0; bad && q < 4 && off == ~0u; ++q) {
                    const uint64_t w = wb + 32 * q + lane;
                    for (uint32_t j = 0; j < 16; ++j)
                        if (w * 16 + j < n && !valid_byte(text[w * 16 + j])) {
                            off = (32u * q + lane) * 16u + j;
                            break;
                        }
                }
            }
            off = __reduce_min_sync(~0u, off);
            if (lane == 0) atomicMin(reinterpret_cast<unsigned long long *>(first_bad), (unsigned long long)(wb * 16 + off));
            wdone = true;  // later iterations of this warp only see larger positions
        }
    }
}

int launch_pack(const uint8_t *d_text, uint64_t n, uint32_t *d_packed, uint64_t nwords_padded,
                uint64_t *d_first_bad, uint16_t *d_inv, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (d_first_bad) {
        cudaError_t e = cudaMemsetAsync(d_first_bad, 0xFF, sizeof(uint64_t), st);
        if (e != cudaSuccess) return e;
    }
    const uint64_t inv_words = (nwords_padded + 7) & ~7ull;
    if (d_inv && inv_words > nwords_padded) {  // the padding words past the packed range
        cudaError_t e = cudaMemsetAsync(d_inv + nwords_padded, 0, (inv_words - nwords_padded) * 2, st);
        if (e != cudaSuccess) return e;
    }
    if (nwords_padded == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t blocks = (nwords_padded + 1023) / 1024;  // 8 warps x 128 words per block and pass
    const uint64_t cap = (uint64_t)sms * 8;
    if (blocks > cap) blocks = cap;
    const bool aligned = (reinterpret_cast<uintptr_t>(d_text) & 15) == 0;
    if (d_inv)
        pack_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(d_text, n, d_packed, nwords_padded, d_first_bad, aligned,
                                                            d_inv);
    else
        pack_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(d_text, n, d_packed, nwords_padded, d_first_bad, aligned,
                                                             nullptr);
    return cudaGetLastError();
}

}  // namespace pfac
