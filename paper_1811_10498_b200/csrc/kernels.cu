// sm_100a kernels of the PFAC hot path: pack, match, compact.
// DESIGN.md §5 gives the data layout in HBM/shared memory and the roofline of each kernel.
#include <cuda_runtime.h>

#include <cstdint>

#include "pfac_internal.h"

namespace pfac {

// ============================================================================ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
// TMA 1-D bulk copy global -> shared, completion signalled on `bar` (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void st_stream_v4(int32_t *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_stream_v4(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t *p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

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

// ============================================================================ match
// One persistent CTA per SM.  Shared memory holds the jump table J (4^K uint32), the first W rows
// of the device transition table and of F, and a double-buffered text tile (+ halo) that a TMA
// bulk copy brings in one tile ahead.  Lane l of warp w handles 4 consecutive positions of each of
// R 128-position slices, so every slice is stored with one coalesced 512-byte st.global.v4.
struct MatchParams {
    const uint32_t *packed;
    int32_t *out;
    uint64_t n_own, n_avail;
    uint64_t ntiles;
    uint64_t avail_words;  // packed words readable (pfac_packed_words(n_avail))
    const uint32_t *J, *T, *F;
    uint32_t window;  // device ids [0, window) have their T row / F entry in smem
    uint32_t root;
    uint32_t txt_words;  // words per text buffer = TILE/16 + halo words
};

template <int K>
struct Tables {
    const uint32_t *J;   // smem
    const uint32_t *Tw;  // smem, rows [0, W)
    const uint32_t *Fw;  // smem
    const uint32_t *Tg;  // global
    const uint32_t *Fg;  // global
    uint32_t W;
    __device__ __forceinline__ uint32_t next(uint32_t s, uint32_t c) const {
        return s < W ? Tw[s * 4 + c] : __ldg(Tg + (size_t)s * 4 + c);
    }
    __device__ __forceinline__ uint32_t final_of(uint32_t s) const { return s < W ? Fw[s] : __ldg(Fg + s); }
};

__device__ __forceinline__ uint32_t base_at(const uint32_t *txt, uint32_t l) {
    return (txt[l >> 4] >> ((l & 15) * 2)) & 3u;
}

// Continue a walk in state s from local text offset l until the first missing transition or the
// end of the readable text (lend); the answer is the deepest final state on the path (F).
template <int K>
__device__ __forceinline__ uint32_t walk_from(const Tables<K> &tb, const uint32_t *txt, uint32_t s, uint32_t l,
                                              uint32_t lend) {
    while (l < lend) {
        uint32_t t = tb.next(s, base_at(txt, l));
        if (!t) break;
        s = t;
        ++l;
    }
    return tb.final_of(s);
}

template <int K, int NT, int R>
__global__ void __launch_bounds__(NT, 1) match_kernel(const MatchParams p) {
    constexpr uint32_t TILE = NT / 32 * R * 128;
    constexpr uint32_t NJ = 1u << (2 * K);
    constexpr uint32_t MASK = NJ - 1;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t *sJ = reinterpret_cast<uint32_t *>(smem);
    uint32_t *sT = sJ + NJ;
    uint32_t *sF = sT + (size_t)p.window * 4;
    uint32_t *sTxt0 = sF + p.window;
    uint32_t *sTxt1 = sTxt0 + p.txt_words;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sTxt1 + p.txt_words);  // [0]=tables, [1],[2]=text

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto issue_text = [&](uint64_t tile, uint32_t *dst, uint64_t *bar) {
        const uint64_t w0 = tile * (TILE / 16);
        const uint64_t left = p.avail_words - w0;
        const uint32_t nw = left < p.txt_words ? (uint32_t)left : p.txt_words;
        mbar_expect_tx(bar, nw * 4);
        bulk_g2s(dst, p.packed + w0, nw * 4, bar);
    };
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        const uint32_t jb = NJ * 4, tb = p.window * 16, fb = p.window * 4;
        mbar_expect_tx(&bars[0], jb + tb + fb);
        bulk_g2s(sJ, p.J, jb, &bars[0]);
        if (p.window) {
            bulk_g2s(sT, p.T, tb, &bars[0]);
            bulk_g2s(sF, p.F, fb, &bars[0]);
        }
        if (blockIdx.x < p.ntiles) issue_text(blockIdx.x, sTxt0, &bars[1]);
    }
    const Tables<K> tb{sJ, sT, sF, p.T, p.F, p.window};
    mbar_wait(&bars[0], 0);

    uint32_t it = 0;
    for (uint64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++it) {
        const uint32_t buf = it & 1;
        if (tid == 0 && tile + gridDim.x < p.ntiles)
            issue_text(tile + gridDim.x, buf ? sTxt0 : sTxt1, &bars[1 + (buf ^ 1)]);
        mbar_wait(&bars[1 + buf], (it >> 1) & 1);
        const uint32_t *txt = buf ? sTxt1 : sTxt0;
        const uint64_t tile_base = tile * TILE;
        const uint64_t avail_left = p.n_avail - tile_base;
        const uint32_t lend = avail_left < p.txt_words * 16ull ? (uint32_t)avail_left : p.txt_words * 16;
        const uint64_t own_left = p.n_own - tile_base;
        const uint32_t lown = own_left < TILE ? (uint32_t)own_left : TILE;
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
            const uint32_t l0 = (warp * R + r) * 128 + lane * 4;
            if (l0 >= lown) continue;
            const uint32_t q = l0 >> 4;
            const uint64_t w64 = ((((uint64_t)txt[q + 1]) << 32) | txt[q]) >> ((l0 & 15) * 2);
            uint32_t e0, e1, e2, e3;
            uint32_t alive = 0;
            if (l0 + 3 + K <= lend) {  // all four K-mers readable: one J lookup each
                e0 = sJ[(uint32_t)w64 & MASK];
                e1 = sJ[(uint32_t)(w64 >> 2) & MASK];
                e2 = sJ[(uint32_t)(w64 >> 4) & MASK];
                e3 = sJ[(uint32_t)(w64 >> 6) & MASK];
                alive = (e0 >> 31) | ((e1 >> 31) << 1) | ((e2 >> 31) << 2) | ((e3 >> 31) << 3);
            } else {  // near the end of the readable text: walk from the root
                e0 = l0 + 0 < lend ? walk_from(tb, txt, p.root, l0 + 0, lend) : 0;
                e1 = l0 + 1 < lend ? walk_from(tb, txt, p.root, l0 + 1, lend) : 0;
                e2 = l0 + 2 < lend ? walk_from(tb, txt, p.root, l0 + 2, lend) : 0;
                e3 = l0 + 3 < lend ? walk_from(tb, txt, p.root, l0 + 3, lend) : 0;
            }
            while (alive) {  // walks that survived K bases continue in the automaton
                const int j = __ffs(alive) - 1;
                alive &= alive - 1;
                const uint32_t s = (j == 0 ? e0 : j == 1 ? e1 : j == 2 ? e2 : e3) & ~kAlive;
                const uint32_t res = walk_from(tb, txt, s, l0 + j + K, lend);
                e0 = j == 0 ? res : e0;
                e1 = j == 1 ? res : e1;
                e2 = j == 2 ? res : e2;
                e3 = j == 3 ? res : e3;
            }
            int32_t *o = p.out + tile_base + l0;
            if (l0 + 4 <= lown) {
                st_stream_v4(o, e0, e1, e2, e3);
            } else {
                o[0] = (int32_t)e0;
                if (l0 + 1 < lown) o[1] = (int32_t)e1;
                if (l0 + 2 < lown) o[2] = (int32_t)e2;
            }
        }
        __syncthreads();  // everyone is done with `txt` before it is refilled
    }
}

constexpr int kMatchThreads = 512;
constexpr int kMatchR = 4;
constexpr uint32_t kMatchTile = kMatchThreads / 32 * kMatchR * 128;

static uint32_t halo_words_for(int K, uint32_t maxlen) {
    uint32_t need = (maxlen > (uint32_t)K ? maxlen : (uint32_t)K) + 16;  // +16: the w64 read of word q+1
    return ((need + 63) / 64) * 4;
}

static size_t match_smem_bytes(int K, uint32_t window, uint32_t txt_words) {
    return ((size_t)1 << (2 * K)) * 4 + (size_t)window * 20 + (size_t)txt_words * 8 + 3 * 8;
}

struct DevProps {
    int sms = 0;
    int smem_optin = 0;
    bool attr_set = false;
};
static DevProps g_props[64];

static DevProps &props(int device) {
    DevProps &d = g_props[device & 63];
    if (!d.sms) {
        cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device);
        cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    }
    return d;
}

uint32_t match_window_rows(int device, int K, uint32_t maxlen, uint32_t S) {
    DevProps &d = props(device);
    const uint32_t txt_words = kMatchTile / 16 + halo_words_for(K, maxlen);
    const size_t fixed = match_smem_bytes(K, 0, txt_words);
    size_t budget = (size_t)d.smem_optin > fixed ? (size_t)d.smem_optin - fixed : 0;
    uint32_t w = (uint32_t)(budget / 20) & ~3u;
    const uint32_t all = ((S + 1) + 3) & ~3u;
    return w < all ? w : all;
}

int launch_match(const DeviceImage &img, const uint32_t *d_packed, uint64_t n_own, uint64_t n_avail,
                 int32_t *d_out, void *stream) {
    if (n_own == 0) return cudaSuccess;
    DevProps &d = props(img.device);
    MatchParams p;
    p.packed = d_packed;
    p.out = d_out;
    p.n_own = n_own;
    p.n_avail = n_avail;
    p.ntiles = (n_own + kMatchTile - 1) / kMatchTile;
    p.avail_words = ((n_avail + 15) / 16 + 3) & ~3ull;
    p.J = img.d_J;
    p.T = img.d_T;
    p.F = img.d_F;
    p.window = img.window;
    p.root = img.root;
    p.txt_words = kMatchTile / 16 + halo_words_for(img.K, img.maxlen);
    const size_t smem = match_smem_bytes(img.K, img.window, p.txt_words);
    auto kern = match_kernel<kJumpK, kMatchThreads, kMatchR>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMatchThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)d.sms * per_sm;
    if (grid > p.ntiles) grid = p.ntiles;
    kern<<<(unsigned)grid, kMatchThreads, smem, (cudaStream_t)stream>>>(p);
    return cudaGetLastError();
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
    int dev = 0;
    cudaGetDevice(&dev);
    DevProps &d = props(dev);
    uint64_t blocks = (ngroups + 255) / 256;
    const uint64_t cap = (uint64_t)d.sms * 8;
    if (blocks > cap) blocks = cap;
    const bool aligned = (reinterpret_cast<uintptr_t>(d_text) & 15) == 0;
    pack_kernel<<<(unsigned)blocks, 256, 0, st>>>(d_text, n, d_packed, ngroups, d_first_bad, aligned);
    return cudaGetLastError();
}

// ============================================================================ compact
// Single pass, order preserving: per tile a warp-ballot rank + a block scan of warp counts, then a
// decoupled look-back over the predecessors' published (aggregate | inclusive prefix) words.
constexpr int kCT = 256;                  // threads
constexpr int kCI = 4;                    // int4 chunks per thread
constexpr int kCW = kCT / 32;             // warps
constexpr uint32_t kCTile = kCT * kCI * 4;  // 4096 elements per tile
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagIncl = 2ull << 62, kValMask = (1ull << 62) - 1;
static_assert(kCI * kCW == 32, "the look-back warp scans one count per lane");

__global__ void __launch_bounds__(kCT) compact_kernel(const int32_t *__restrict__ out, uint64_t n,
                                                      uint64_t pos_base, uint64_t *__restrict__ pos,
                                                      uint32_t *__restrict__ pid, uint64_t cap,
                                                      uint64_t *d_count, uint32_t k, uint64_t *hist,
                                                      uint64_t *ws, uint64_t ntiles) {
    __shared__ uint64_t s_tile, s_prefix;
    __shared__ uint32_t s_cnt[32], s_off[32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(reinterpret_cast<unsigned long long *>(ws), 1ull);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * kCTile;
    const uint32_t lt = (1u << lane) - 1;
    uint4 v[kCI];
    uint32_t lex[kCI];
#pragma unroll
    for (int i = 0; i < kCI; ++i) {
        const uint64_t idx = base + ((uint64_t)i * kCT + tid) * 4;
        if (idx + 4 <= n) {
            v[i] = ld_stream_v4(out + idx);
        } else {
            v[i].x = idx + 0 < n ? out[idx + 0] : 0;
            v[i].y = idx + 1 < n ? out[idx + 1] : 0;
            v[i].z = idx + 2 < n ? out[idx + 2] : 0;
            v[i].w = 0;
        }
        const uint32_t c = (v[i].x != 0) + (v[i].y != 0) + (v[i].z != 0) + (v[i].w != 0);
        const uint32_t b0 = __ballot_sync(~0u, c & 1), b1 = __ballot_sync(~0u, c & 2),
                       b2 = __ballot_sync(~0u, c & 4);
        lex[i] = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
        if (lane == 0) s_cnt[i * kCW + warp] = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t x = s_cnt[lane];
        uint32_t incl = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t y = __shfl_up_sync(~0u, incl, d);
            if (lane >= (uint32_t)d) incl += y;
        }
        s_off[lane] = incl - x;
        const uint64_t total = __shfl_sync(~0u, incl, 31);
        uint64_t prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_release_u64(ws + 1, kFlagIncl | total);
        } else {
            if (lane == 0) st_release_u64(ws + 1 + tile, kFlagAgg | total);
            int64_t j = (int64_t)tile - 1;
            while (true) {
                const int64_t idx = j - (int64_t)lane;
                uint64_t st = idx >= 0 ? ld_acquire_u64(ws + 1 + idx) : kFlagIncl;
                while (__any_sync(~0u, (st >> 62) == 0)) {
                    if ((st >> 62) == 0) st = ld_acquire_u64(ws + 1 + idx);
                }
                const uint32_t incl_mask = __ballot_sync(~0u, (st >> 62) == 2);
                const int first = incl_mask ? __ffs(incl_mask) - 1 : 32;
                uint64_t val = (int)lane <= first ? (st & kValMask) : 0;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) val += __shfl_xor_sync(~0u, val, d);
                prefix += val;
                if (incl_mask) break;
                j -= 32;
            }
            if (lane == 0) st_release_u64(ws + 1 + tile, kFlagIncl | (prefix + total));
        }
        if (lane == 0) {
            s_prefix = prefix;
            if (tile == ntiles - 1) *d_count = prefix + total;
        }
    }
    __syncthreads();
    const uint64_t prefix = s_prefix;
#pragma unroll
    for (int i = 0; i < kCI; ++i) {
        const uint32_t vals[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
        if ((vals[0] | vals[1] | vals[2] | vals[3]) == 0) continue;
        uint64_t r = prefix + s_off[i * kCW + warp] + lex[i];
        const uint64_t idx = base + ((uint64_t)i * kCT + tid) * 4;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (!vals[e]) continue;
            if (r < cap) {
                pos[r] = pos_base + idx + e;
                pid[r] = vals[e];
            }
            if (hist && vals[e] <= k) atomicAdd(reinterpret_cast<unsigned long long *>(hist + vals[e]), 1ull);
            ++r;
        }
    }
}

uint64_t compact_workspace_bytes(uint64_t n) { return ((n + kCTile - 1) / kCTile + 1) * 8; }

int launch_compact(const int32_t *d_out, uint64_t n, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                   uint64_t capacity, uint64_t *d_count, uint32_t k, uint64_t *d_hist, void *d_workspace,
                   void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t ntiles = (n + kCTile - 1) / kCTile;
    if (ntiles == 0) return cudaMemsetAsync(d_count, 0, 8, st);
    cudaError_t e = cudaMemsetAsync(d_workspace, 0, compact_workspace_bytes(n), st);
    if (e != cudaSuccess) return e;
    if (ntiles > 0x7fffffffull) return cudaErrorInvalidValue;
    compact_kernel<<<(unsigned)ntiles, kCT, 0, st>>>(d_out, n, pos_base, d_pos, d_pid, capacity, d_count, k,
                                                     d_hist, reinterpret_cast<uint64_t *>(d_workspace), ntiles);
    return cudaGetLastError();
}

}  // namespace pfac
