// Pack kernel: ASCII bases -> 2-bit codes + validation status.
// HBM-bound: 1 B read + 0.25 B written per base.
#include <cuda_runtime.h>

#include <cstdint>

#include "pfac_internal.h"
#include "ptx.cuh"

namespace pfac {

// ============================================================================ pack
// ASCII -> 2-bit codes (A0 C1 G2 T3), 16 bases per uint32, base j at bits 2(j mod 16).
// Four bytes at a time (one 32-bit word x):
//   t = (x >> 1) & 3 per byte gives A0 C1 T2 G3 for upper and lower case;
//   validity: the byte must equal "acgt"[t] after |0x20 -- one PRMT builds the expected word;
//   code = t ^ (t >> 1) swaps G and T; one multiply gathers the four 2-bit codes into a byte.
// Integer ALU (LOP3/SHF/PRMT) is the scarce pipe here (half rate), so the multiply does the gather.
__device__ __forceinline__ uint32_t expect4(uint32_t x, uint32_t t) {  // nonzero bytes = bad bytes
    uint32_t sel = t | (t >> 4);                    // nibble selectors at bits 0, 4, 16, 20
    sel = (sel & 0xFFu) | ((sel >> 8) & 0xFF00u);   // -> bits 0, 4, 8, 12
    return __byte_perm(0x67746361u, 0u, sel) ^ (x | 0x20202020u);  // "acgt"[t] vs the byte
}
__device__ __forceinline__ uint32_t pack4(uint32_t x, uint32_t &bad) {
    const uint32_t t = (x >> 1) & 0x03030303u;
    bad |= expect4(x, t);
    const uint32_t c = t ^ ((t >> 1) & 0x01010101u);
    return (c * 0x01041040u) >> 24;                 // c0 | c1 << 2 | c2 << 4 | c3 << 6
}
// 4-bit mask of the bad bytes of x (bit b = byte b): the 0x01 bits of the nonzero-byte mask gathered
// by one multiply (partial products land on distinct bits, none in 24..27 but the wanted four).
__device__ __forceinline__ uint32_t bad4(uint32_t x) {
    const uint32_t m = __vcmpne4(expect4(x, (x >> 1) & 0x03030303u), 0u) & 0x01010101u;
    return (m * 0x01020408u) >> 24;
}
__device__ __forceinline__ uint32_t bad16(uint4 v) {
    return bad4(v.x) | (bad4(v.y) << 4) | (bad4(v.z) << 8) | (bad4(v.w) << 12);
}
__device__ __forceinline__ bool valid_byte(uint8_t b) {
    uint8_t y = b | 0x20;
    return y == 'a' || y == 'c' || y == 'g' || y == 't';
}

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
                    packed[wb + 32 * q + lane] = pack4(v[q].x, bq) | (pack4(v[q].y, bq) << 8) |
                                                 (pack4(v[q].z, bq) << 16) | (pack4(v[q].w, bq) << 24);
                    const uint32_t m = bq ? bad16(v[q]) : 0u;
                    inv[wb + 32 * q + lane] = (uint16_t)m;
                    if (q < 2) mlo |= m << (16 * q);
                    else mhi |= m << (16 * (q - 2));
                    bad |= bq;
                } else {  // one accumulator: the integer pipe is this kernel's limit
                    packed[wb + 32 * q + lane] = pack4(v[q].x, bad) | (pack4(v[q].y, bad) << 8) |
                                                 (pack4(v[q].z, bad) << 16) | (pack4(v[q].w, bad) << 24);
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
                bad |= m;
                packed[w] = word;
                if (INV) {
                    inv[w] = (uint16_t)m;
                    if (q < 2) mlo |= m << (16 * q);
                    else mhi |= m << (16 * (q - 2));
                }
            }
        }
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
