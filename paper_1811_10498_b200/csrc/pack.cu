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
// first_bad: the warp keeps the first bad index it meets (its iterations ascend) and issues one
// atomicMin at the end, so a text full of barriers (FASTA newlines) costs one atomic per warp.
__global__ void __launch_bounds__(256) pack_kernel(const uint8_t *__restrict__ text, uint64_t n,
                                                   uint32_t *__restrict__ packed, uint64_t nwords,
                                                   uint64_t *first_bad, bool aligned, uint16_t *__restrict__ inv,
                                                   uint64_t inv_words) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t wfirst = ~0ull;  // warp-uniform
    for (uint64_t wb = warp * 128; wb < nwords; wb += nwarps * 128) {
        uint32_t im[4] = {0u, 0u, 0u, 0u};
        if (aligned && (wb + 128) * 16 <= n) {
            uint4 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = ld_stream_v4(text + (wb + 32 * q + lane) * 16);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t bq = 0;
                packed[wb + 32 * q + lane] = pack4(v[q].x, bq) | (pack4(v[q].y, bq) << 8) |
                                             (pack4(v[q].z, bq) << 16) | (pack4(v[q].w, bq) << 24);
                if (bq) im[q] = bad16(v[q]);
                if (inv) inv[wb + 32 * q + lane] = (uint16_t)im[q];
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
                im[q] = m;
                packed[w] = word;
                if (inv) inv[w] = (uint16_t)m;
            }
        }
        if (first_bad && wfirst == ~0ull) {
            // this lane's first bad byte: its first word with one (offsets of later q are larger)
            uint32_t off = ~0u;
#pragma unroll
            for (int q = 3; q >= 0; --q)
                if (im[q]) off = (32u * q + lane) * 16u + (__ffs(im[q]) - 1);
            off = __reduce_min_sync(~0u, off);
            if (off != ~0u) wfirst = wb * 16 + off;
        }
    }
    if (first_bad && lane == 0 && wfirst != ~0ull)
        atomicMin(reinterpret_cast<unsigned long long *>(first_bad), (unsigned long long)wfirst);
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
    pack_kernel<<<(unsigned)blocks, 256, 0, st>>>(d_text, n, d_packed, nwords_padded, d_first_bad, aligned, d_inv,
                                                   inv_words);
    return cudaGetLastError();
}

}  // namespace pfac
