// Microbenchmarks for the peaks SURVEY.md §8(d) asks to measure beside the roofline (measurement
// tooling only; not part of libpfac): write-only / read-only / copy HBM bandwidth with 16-byte
// accesses, L2 random 32-byte gathers over 4-64 MB windows, shared-memory random-lookup rate, and the
// device attributes the design depends on.  Prints one JSON object.
//
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o microbench scripts/microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cmath>
#include <cstdio>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

// Four independent 16-byte accesses per thread and iteration (bytes in flight), grid-stride.
__global__ void k_write(uint4 *p, size_t n, bool stream) {
    const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    const size_t T = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += 4 * T) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const size_t j = i + u * T;
            if (j >= n) break;
            if (stream) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p + j), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
            else p[j] = v;
        }
    }
}
__global__ void k_read(const uint4 *p, size_t n, uint32_t *sink) {
    uint32_t acc = 0;
    const size_t T = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += 4 * T) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const size_t j = i + u * T < n ? i + u * T : i;
            asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + j));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}
__global__ void k_copy(const uint4 *a, uint4 *b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
// Random 32-byte-sector gathers (one 16-byte load per sector) inside a window of `mask+1` sectors.
__global__ void k_gather(const uint4 *p, uint32_t mask, int iters, uint32_t *sink) {
    uint32_t x = blockIdx.x * blockDim.x + threadIdx.x + 1, acc = 0;
    for (int it = 0; it < iters; it += 4) {
        uint32_t idx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            x = x * 1664525u + 1013904223u;
            idx[u] = (x >> 3) & mask;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint4 v = __ldg(p + 2 * (size_t)idx[u]);
            acc += v.x;
        }
    }
    if (acc == 0x12345678u) *sink = acc;
}
// Random 4-byte lookups in a 128 KiB shared-memory table (the size of the match kernel's filter).
__global__ void k_smem(int iters, uint32_t *sink) {
    extern __shared__ uint32_t tab[];
    for (uint32_t i = threadIdx.x; i < 32768; i += blockDim.x) tab[i] = i * 2654435761u;
    __syncthreads();
    uint32_t x = blockIdx.x * blockDim.x + threadIdx.x + 1, acc = 0;
    for (int it = 0; it < iters; it += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x = x * 1664525u + 1013904223u;
            acc += tab[(x >> 9) & 32767];
        }
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <typename F>
static float time_ms(F f, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

int main() {
    int dev = 0, sms = 0, l2 = 0, persist = 0, smem_optin = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const size_t bytes = 2ull << 30, n = bytes / 16;
    uint4 *a = nullptr, *b = nullptr;
    uint32_t *sink = nullptr;
    CK(cudaMalloc(&a, bytes));
    CK(cudaMalloc(&b, bytes));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(a, 1, bytes));
    // best over launch shapes (blocks per SM x threads per block)
    float w_cs = 1e30f, w_wb = 1e30f, rd = 1e30f, cp = 1e30f;
    for (int bps : {2, 4, 8, 16}) {
        for (int block : {256, 512, 1024}) {
            if (bps * block > 2048) continue;
            const int grid = sms * bps;
            w_cs = fminf(w_cs, time_ms([&] { k_write<<<grid, block>>>(a, n, true); }, 5));
            w_wb = fminf(w_wb, time_ms([&] { k_write<<<grid, block>>>(a, n, false); }, 5));
            rd = fminf(rd, time_ms([&] { k_read<<<grid, block>>>(a, n, sink); }, 5));
            cp = fminf(cp, time_ms([&] { k_copy<<<grid, block>>>(a, b, n / 2); }, 5));  // 1 GiB read + 1 GiB write
        }
    }
    CK(cudaGetLastError());
    printf("{\"device_attrs\": {\"sms\": %d, \"l2_bytes\": %d, \"max_persisting_l2_bytes\": %d, "
           "\"smem_per_block_optin\": %d, \"sm_clock_khz\": %d},\n",
           sms, l2, persist, smem_optin, clk);
    printf(" \"hbm_gbs\": {\"write_st_cs_v4\": %.1f, \"write_st_v4\": %.1f, \"read_ld_cs_v4\": %.1f, "
           "\"copy_read_plus_write\": %.1f, \"buffer_bytes\": %zu},\n",
           bytes / (w_cs * 1e-3) / 1e9, bytes / (w_wb * 1e-3) / 1e9, bytes / (rd * 1e-3) / 1e9,
           bytes / (cp * 1e-3) / 1e9, bytes);
    printf(" \"l2_gather_32B\": [");
    const int gth = 512, giters = 256;
    const size_t gthreads = (size_t)sms * 4 * gth;
    const uint32_t wins_mb[] = {4, 16, 64};
    for (int wi = 0; wi < 3; ++wi) {
        const uint32_t sectors = wins_mb[wi] * (1u << 20) / 32;
        k_gather<<<sms * 4, gth>>>(a, sectors - 1, giters, sink);  // warm the window into L2
        const float ms = time_ms([&] { k_gather<<<sms * 4, gth>>>(a, sectors - 1, giters, sink); }, 5);
        const double loads = (double)gthreads * giters;
        printf("%s{\"window_mb\": %u, \"gsectors_per_s\": %.2f, \"gbs_32B\": %.1f}", wi ? ", " : "", wins_mb[wi],
               loads / (ms * 1e-3) / 1e9, loads * 32 / (ms * 1e-3) / 1e9);
    }
    printf("],\n");
    CK(cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    const int siters = 4096;
    const float sm_ms = time_ms([&] { k_smem<<<sms, 1024, 131072>>>(siters, sink); }, 5);
    CK(cudaGetLastError());
    const double lookups = (double)sms * 1024 * siters;
    printf(" \"smem_random_lookup\": {\"table_bytes\": 131072, \"glookups_per_s\": %.1f, \"per_sm_per_clk\": %.2f}}\n",
           lookups / (sm_ms * 1e-3) / 1e9, lookups / (sm_ms * 1e-3) / sms / (clk * 1e3));
    cudaFree(a);
    cudaFree(b);
    cudaFree(sink);
    return 0;
}
