// Pack kernel: ASCII bases -> 2-bit codes + validation status.
// HBM-bound: 1 B read + 0.25 B written per base.
#include <cuda_runtime.h>

#include <cstdint>

#include "pfac_internal.h"
#include "ptx.cuh"

namespace pfac {

// ============================================================================ pack
// ASCII -> 2-bit codes (A0 C1 G2 T3), 16 bases per uint32, base j at bits 2(j mod 16).
// (b >> 1) & 3 gives A0 C1 T2 G3 for upper and lower case; t ^ (t >> 1) swaps G and T.
__device__ __forceinline__ uint32_t pack4(uint32_t x) {
    uint32_t t = (x >> 1) & 0x03030303u;
    uint32_t c = t ^ ((t >> 1) & 0x01010101u);
    c = (c | (c >> 6)) & 0x000F000Fu;
    return (c | (c >> 12)) & 0xFFu;
}
// 0xFF in each byte lane that holds one of ACGTacgt.
__device__ __forceinline__ uint32_t valid4(uint32_t x) {
    uint32_t y = x | 0x20202020u;
    return __vcmpeq4(y, 0x61616161u) | __vcmpeq4(y, 0x63636363u) | __vcmpeq4(y, 0x67676767u) |
           __vcmpeq4(y, 0x74747474u);
}
__device__ __forceinline__ bool valid_byte(uint8_t b) {
    uint8_t y = b | 0x20;
    return y == 'a' || y == 'c' || y == 'g' || y == 't';
}

__global__ void __launch_bounds__(256) pack_kernel(const uint8_t *__restrict__ text, uint64_t n,
                                                   uint32_t *__restrict__ packed, uint64_t ngroups,
                                                   uint64_t *first_bad, bool aligned) {
    // one group = 4 packed words = 64 bases; grid-stride
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < ngroups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b0 = g * 64;
        uint32_t w[4];
        bool ok = true;
        if (aligned && b0 + 64 <= n) {
            uint32_t m = 0xFFFFFFFFu;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint4 v = ld_stream_v4(text + b0 + 16 * q);
                m &= valid4(v.x) & valid4(v.y) & valid4(v.z) & valid4(v.w);
                w[q] = pack4(v.x) | (pack4(v.y) << 8) | (pack4(v.z) << 16) | (pack4(v.w) << 24);
            }
            ok = (m == 0xFFFFFFFFu);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t word = 0;
                for (int j = 0; j < 16; ++j) {
                    uint64_t i = b0 + 16 * q + j;
                    if (i < n) {
                        uint8_t b = text[i];
                        ok &= valid_byte(b);
                        uint32_t t = (b >> 1) & 3u;
                        word |= (t ^ (t >> 1)) << (2 * j);
                    }
                }
                w[q] = word;
            }
        }
        if (!ok && first_bad) {
            for (int j = 0; j < 64; ++j) {
                uint64_t i = b0 + j;
                if (i < n && !valid_byte(text[i])) {
                    atomicMin(reinterpret_cast<unsigned long long *>(first_bad), (unsigned long long)i);
                    break;
                }
            }
        }
        *reinterpret_cast<uint4 *>(packed + 4 * g) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

int launch_pack(const uint8_t *d_text, uint64_t n, uint32_t *d_packed, uint64_t nwords_padded,
                uint64_t *d_first_bad, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (d_first_bad) {
        cudaError_t e = cudaMemsetAsync(d_first_bad, 0xFF, sizeof(uint64_t), st);
        if (e != cudaSuccess) return e;
    }
    const uint64_t ngroups = nwords_padded / 4;
    if (ngroups == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t blocks = (ngroups + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8;
    if (blocks > cap) blocks = cap;
    const bool aligned = (reinterpret_cast<uintptr_t>(d_text) & 15) == 0;
    pack_kernel<<<(unsigned)blocks, 256, 0, st>>>(d_text, n, d_packed, ngroups, d_first_bad, aligned);
    return cudaGetLastError();
}

}  // namespace pfac
