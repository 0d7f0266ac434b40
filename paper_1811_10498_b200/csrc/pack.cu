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
__device__ __forceinline__ uint32_t pack4(uint32_t x, uint32_t &bad) {
    const uint32_t t = (x >> 1) & 0x03030303u;
    uint32_t sel = t | (t >> 4);                    // nibble selectors at bits 0, 4, 16, 20
    sel = (sel & 0xFFu) | ((sel >> 8) & 0xFF00u);   // -> bits 0, 4, 8, 12
    bad |= __byte_perm(0x67746361u, 0u, sel) ^ (x | 0x20202020u);  // "acgt"[t] vs the byte
    const uint32_t c = t ^ ((t >> 1) & 0x01010101u);
    return (c * 0x01041040u) >> 24;                 // c0 | c1 << 2 | c2 << 4 | c3 << 6
}
__device__ __forceinline__ bool valid_byte(uint8_t b) {
    uint8_t y = b | 0x20;
    return y == 'a' || y == 'c' || y == 'g' || y == 't';
}

// A warp packs 128 consecutive words (2048 bases) per iteration: for q = 0..3 lane l reads the 16
// bytes of word 32q + l (one coalesced 512-byte load per q) and writes that word (a coalesced
// 128-byte store per q).  Grid-stride over the padded word range.
__global__ void __launch_bounds__(256) pack_kernel(const uint8_t *__restrict__ text, uint64_t n,
                                                   uint32_t *__restrict__ packed, uint64_t nwords,
                                                   uint64_t *first_bad, bool aligned) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t wb = warp * 128; wb < nwords; wb += nwarps * 128) {
        bool ok = true;
        if (aligned && (wb + 128) * 16 <= n) {
            uint4 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = ld_stream_v4(text + (wb + 32 * q + lane) * 16);
            uint32_t bad = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                packed[wb + 32 * q + lane] = pack4(v[q].x, bad) | (pack4(v[q].y, bad) << 8) |
                                             (pack4(v[q].z, bad) << 16) | (pack4(v[q].w, bad) << 24);
            ok = (bad == 0);
        } else {
#pragma unroll 1
            for (int q = 0; q < 4; ++q) {
                const uint64_t w = wb + 32 * q + lane;
                if (w >= nwords) break;
                uint32_t word = 0;
                for (int j = 0; j < 16; ++j) {
                    const uint64_t i = w * 16 + j;
                    if (i < n) {
                        const uint8_t b = text[i];
                        ok &= valid_byte(b);
                        const uint32_t t = (b >> 1) & 3u;
                        word |= (t ^ (t >> 1)) << (2 * j);
                    }
                }
                packed[w] = word;
            }
        }
        if (!ok && first_bad) {  // rare: locate this lane's first bad byte exactly
            for (int q = 0; q < 4; ++q) {
                const uint64_t w = wb + 32 * q + lane;
                bool found = false;
                for (int j = 0; j < 16 && !found; ++j) {
                    const uint64_t i = w * 16 + j;
                    if (i < n && !valid_byte(text[i])) {
                        atomicMin(reinterpret_cast<unsigned long long *>(first_bad), (unsigned long long)i);
                        found = true;
                    }
                }
                if (found) break;
            }
        }
    }
}

int launch_pack(const uint8_t *d_text, uint64_t n, uint32_t *d_packed, uint64_t nwords_padded,
                uint64_t *d_first_bad, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (d_first_bad) {
        cudaError_t e = cudaMemsetAsync(d_first_bad, 0xFF, sizeof(uint64_t), st);
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
    pack_kernel<<<(unsigned)blocks, 256, 0, st>>>(d_text, n, d_packed, nwords_padded, d_first_bad, aligned);
    return cudaGetLastError();
}

}  // namespace pfac
