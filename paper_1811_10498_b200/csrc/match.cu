// Match kernel: out[i] = id of the longest pattern starting at i.
//
// Layout and schedule:
//  * One persistent CTA of 1024 threads per SM.  Shared memory holds the jump table J (4^K cells),
//    the first W rows of the device transition table T and of F (all of them when they fit), and
//    per warp a double-buffered text slice that the warp's lane 0 fetches with a TMA bulk copy.
//  * A warp owns "slices" of 512 positions (strided over the grid) + a halo of >= maxlen bases.
//    Lane l handles 4 consecutive positions of each 128-position sub-slice: one J lookup per
//    position answers every walk that dies within K bases; the answers are stored right away with
//    one coalesced 512-byte st.global.cs.v4 per sub-slice.
//  * Walks still alive after K bases are pushed (position, state) into a warp-private queue and
//    walked 32 at a time, one per lane, so the rare long walks do not serialise the warp; their
//    results patch out[] after a __syncwarp (which orders them after the v4 stores).
// The walk itself is PAPER.md:91-93 / :204: follow the goto function from the start state, stop at
// the first missing transition; the answer is the deepest final state passed (F).
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "pfac_internal.h"
#include "ptx.cuh"

namespace pfac {

constexpr int kMT = 1024;               // threads per CTA
constexpr int kMWarps = kMT / 32;
constexpr uint32_t kSlice = 512;        // positions per warp slice
constexpr uint32_t kSub = kSlice / 128; // 128-position sub-slices per slice
constexpr uint32_t kQCap = 160;         // >= 31 + 128 queue entries

struct MatchArgs {
    const uint32_t *packed;
    int32_t *out;
    uint64_t n_own, n_avail, nslices, avail_words;
    const void *J, *T, *F;
    uint32_t window;       // device ids [0, window) have T row / F entry in smem
    uint32_t root;         // device id of the start state
    uint32_t slice_words;  // kSlice/16 + halo words
};

template <typename CT>
struct QItem {
    using type = typename std::conditional<sizeof(CT) == 2, uint32_t, uint64_t>::type;
    static __device__ __forceinline__ type make(uint32_t l, uint32_t s) {
        if constexpr (sizeof(CT) == 2) return (l << 16) | s;
        else return ((uint64_t)l << 32) | s;
    }
    static __device__ __forceinline__ uint32_t pos(type q) { return (uint32_t)(q >> (sizeof(CT) == 2 ? 16 : 32)); }
    static __device__ __forceinline__ uint32_t state(type q) {
        if constexpr (sizeof(CT) == 2) return q & 0xFFFFu;
        else return (uint32_t)q;
    }
};

template <typename CT, bool WIN>
struct Tab {
    const CT *Tw, *Fw, *Tg, *Fg;
    uint32_t W;
    __device__ __forceinline__ uint32_t next(uint32_t s, uint32_t c) const {
        if constexpr (!WIN) return Tw[s * 4 + c];
        else return s < W ? (uint32_t)Tw[s * 4 + c] : (uint32_t)__ldg(Tg + (size_t)s * 4 + c);
    }
    __device__ __forceinline__ uint32_t final_of(uint32_t s) const {
        if constexpr (!WIN) return Fw[s];
        else return s < W ? (uint32_t)Fw[s] : (uint32_t)__ldg(Fg + s);
    }
};

__device__ __forceinline__ uint32_t base_at(const uint32_t *txt, uint32_t l) {
    return (txt[l >> 4] >> ((l & 15) * 2)) & 3u;
}

// Walk from state s reading bases l, l+1, ... (< lend); returns F of the last state reached.
template <typename CT, bool WIN>
__device__ __forceinline__ uint32_t walk(const Tab<CT, WIN> &tb, const uint32_t *txt, uint32_t s, uint32_t l,
                                         uint32_t lend) {
    while (l < lend) {
        const uint32_t t = tb.next(s, base_at(txt, l));
        if (!t) break;
        s = t;
        ++l;
    }
    return tb.final_of(s);
}

static __host__ __device__ constexpr uint32_t warp_bytes(uint32_t slice_words, uint32_t qitem) {
    return ((2 * slice_words * 4 + 16 + kQCap * qitem) + 15) & ~15u;
}

template <typename CT, bool WIN, int K>
__global__ void __launch_bounds__(kMT, 1) match_kernel(const MatchArgs p) {
    constexpr uint32_t NJ = 1u << (2 * K);
    constexpr uint32_t MASK = NJ - 1;
    constexpr uint32_t ALIVE = sizeof(CT) == 2 ? 0x8000u : 0x80000000u;
    using Q = QItem<CT>;
    using QT = typename Q::type;
    extern __shared__ __align__(128) uint8_t smem[];
    CT *sJ = reinterpret_cast<CT *>(smem);
    CT *sT = sJ + NJ;
    CT *sF = sT + (size_t)p.window * 4;
    uint8_t *wbase = reinterpret_cast<uint8_t *>(sF + p.window);  // 16-byte aligned (W % 8 == 0)
    const uint32_t WB = warp_bytes(p.slice_words, sizeof(QT));
    uint64_t *tab_bar = reinterpret_cast<uint64_t *>(wbase + kMWarps * WB);

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint8_t *mine = wbase + warp * WB;
    uint32_t *txt0 = reinterpret_cast<uint32_t *>(mine);
    uint32_t *txt1 = txt0 + p.slice_words;
    uint64_t *bar = reinterpret_cast<uint64_t *>(txt1 + p.slice_words);
    QT *queue = reinterpret_cast<QT *>(bar + 2);

    const uint64_t TW = (uint64_t)gridDim.x * kMWarps;
    const uint64_t gw = (uint64_t)blockIdx.x * kMWarps + warp;
    auto issue = [&](uint64_t sl, uint32_t *dst, uint64_t *b) {
        const uint64_t w0 = sl * (kSlice / 16);
        const uint64_t left = p.avail_words - w0;
        const uint32_t nw = left < p.slice_words ? (uint32_t)left : p.slice_words;
        mbar_expect_tx(b, nw * 4);
        bulk_g2s(dst, p.packed + w0, nw * 4, b);
    };
    if (tid == 0) mbar_init(tab_bar, 1);
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    fence_mbar_init();
    __syncthreads();
    if (tid == 0) {
        const uint32_t jb = NJ * sizeof(CT), tb = p.window * 4 * sizeof(CT), fb = p.window * sizeof(CT);
        mbar_expect_tx(tab_bar, jb + tb + fb);
        bulk_g2s(sJ, p.J, jb, tab_bar);
        if (p.window) {
            bulk_g2s(sT, p.T, tb, tab_bar);
            bulk_g2s(sF, p.F, fb, tab_bar);
        }
    }
    if (lane == 0 && gw < p.nslices) issue(gw, txt0, &bar[0]);
    const Tab<CT, WIN> tb{sT, sF, reinterpret_cast<const CT *>(p.T), reinterpret_cast<const CT *>(p.F), p.window};
    mbar_wait(tab_bar, 0);

    const uint32_t lt = (1u << lane) - 1;
    uint32_t it = 0;
    for (uint64_t sl = gw; sl < p.nslices; sl += TW, ++it) {
        const uint32_t buf = it & 1;
        if (lane == 0 && sl + TW < p.nslices) issue(sl + TW, buf ? txt0 : txt1, &bar[buf ^ 1]);
        mbar_wait(&bar[buf], (it >> 1) & 1);
        const uint32_t *txt = buf ? txt1 : txt0;
        const uint64_t base = sl * kSlice;
        const uint64_t avail_left = p.n_avail - base;
        const uint32_t lend = avail_left < p.slice_words * 16ull ? (uint32_t)avail_left : p.slice_words * 16;
        const uint64_t own_left = p.n_own - base;
        const uint32_t lown = own_left < kSlice ? (uint32_t)own_left : kSlice;
        int32_t *out = p.out + base;
        uint32_t qn = 0;  // warp-uniform queue length

        auto drain = [&](uint32_t keep) {  // walk queued items 32 at a time until <= keep remain
            while (qn > keep) {
                __syncwarp();
                const uint32_t take = qn - keep < 32 ? qn - keep : 32;
                if (lane < take) {
                    const QT q = queue[qn - take + lane];
                    const uint32_t l = Q::pos(q);
                    out[l] = (int32_t)walk(tb, txt, Q::state(q), l + K, lend);
                }
                qn -= take;
                __syncwarp();
            }
        };

#pragma unroll 1
        for (uint32_t r = 0; r < kSub; ++r) {
            const uint32_t l0 = r * 128 + lane * 4;
            uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0, alive = 0;
            if (l0 < lown) {
                if (l0 + 3 + K <= lend) {  // all four K-mers readable: one J lookup each
                    const uint32_t q = l0 >> 4;
                    const uint32_t x = (uint32_t)(((((uint64_t)txt[q + 1]) << 32) | txt[q]) >> ((l0 & 15) * 2));
                    e0 = sJ[x & MASK];
                    e1 = sJ[(x >> 2) & MASK];
                    e2 = sJ[(x >> 4) & MASK];
                    e3 = sJ[(x >> 6) & MASK];
                    alive = (e0 & ALIVE ? 1u : 0u) | (e1 & ALIVE ? 2u : 0u) | (e2 & ALIVE ? 4u : 0u) |
                            (e3 & ALIVE ? 8u : 0u);
                } else {  // the last bases of the readable text: plain walks from the root
                    e0 = walk(tb, txt, p.root, l0, lend);
                    e1 = l0 + 1 < lend ? walk(tb, txt, p.root, l0 + 1, lend) : 0;
                    e2 = l0 + 2 < lend ? walk(tb, txt, p.root, l0 + 2, lend) : 0;
                    e3 = l0 + 3 < lend ? walk(tb, txt, p.root, l0 + 3, lend) : 0;
                }
                if (l0 + 4 <= lown) {
                    st_stream_v4(out + l0, e0, e1, e2, e3);  // alive cells are patched below
                } else {
                    out[l0] = (int32_t)e0;
                    if (l0 + 1 < lown) out[l0 + 1] = (int32_t)e1;
                    if (l0 + 2 < lown) out[l0 + 2] = (int32_t)e2;
                }
            }
            // warp-exclusive prefix of popc(alive) (0..4) with three ballots
            const uint32_t c = __popc(alive);
            const uint32_t b0 = __ballot_sync(~0u, c & 1), b1 = __ballot_sync(~0u, c & 2),
                           b2 = __ballot_sync(~0u, c & 4);
            if (b0 | b1 | b2) {
                uint32_t at = qn + __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
                if (alive & 1) queue[at++] = Q::make(l0 + 0, e0 & ~ALIVE);
                if (alive & 2) queue[at++] = Q::make(l0 + 1, e1 & ~ALIVE);
                if (alive & 4) queue[at++] = Q::make(l0 + 2, e2 & ~ALIVE);
                if (alive & 8) queue[at++] = Q::make(l0 + 3, e3 & ~ALIVE);
                qn += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
                if (qn >= 32) drain(qn & 31);
            }
        }
        drain(0);
        __syncwarp();  // all lanes done with `txt` before lane 0 refills it next iteration
    }
}

// ---------------------------------------------------------------------------------- host side
static uint32_t halo_words_for(int K, uint32_t maxlen) {
    const uint32_t need = (maxlen > (uint32_t)K ? maxlen : (uint32_t)K) + 16;  // +16: word q+1 read
    return ((need + 63) / 64) * 4;
}

static int g_sms[64], g_optin[64];

static void dev_props(int device, int &sms, int &optin) {
    int &s = g_sms[device & 63], &o = g_optin[device & 63];
    if (!s) {
        cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, device);
        cudaDeviceGetAttribute(&o, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    }
    sms = s;
    optin = o;
}

static size_t match_smem(int K, uint32_t cell, uint32_t window, uint32_t slice_words) {
    const uint32_t qitem = cell == 2 ? 4 : 8;
    return ((size_t)1 << (2 * K)) * cell + (size_t)window * 5 * cell + (size_t)kMWarps * warp_bytes(slice_words, qitem) +
           16;
}

MatchPlan plan_match(int device, int K, uint32_t maxlen, uint32_t S, uint32_t k) {
    MatchPlan pl;
    int sms = 0, optin = 0;
    dev_props(device, sms, optin);
    pl.cell = (S < 32768u && k < 32768u) ? 2 : 4;
    pl.slice_words = kSlice / 16 + halo_words_for(K, maxlen);
    const size_t fixed = match_smem(K, pl.cell, 0, pl.slice_words);
    const size_t budget = (size_t)optin > fixed ? (size_t)optin - fixed : 0;
    uint32_t w = (uint32_t)(budget / (5 * pl.cell)) & ~7u;
    const uint32_t all = ((S + 1) + 7) & ~7u;
    pl.all_smem = w >= all;
    pl.window = pl.all_smem ? all : w;
    pl.smem = match_smem(K, pl.cell, pl.window, pl.slice_words);
    pl.sms = sms;
    return pl;
}

int launch_match(const DeviceImage &img, const uint32_t *d_packed, uint64_t n_own, uint64_t n_avail,
                 int32_t *d_out, void *stream) {
    if (n_own == 0) return cudaSuccess;
    MatchArgs a;
    a.packed = d_packed;
    a.out = d_out;
    a.n_own = n_own;
    a.n_avail = n_avail;
    a.nslices = (n_own + kSlice - 1) / kSlice;
    a.avail_words = ((n_avail + 15) / 16 + 3) & ~3ull;
    a.J = img.d_J;
    a.T = img.d_T;
    a.F = img.d_F;
    a.window = img.plan.window;
    a.root = img.root;
    a.slice_words = img.plan.slice_words;
    const MatchPlan &pl = img.plan;
    void *args[] = {&a};
    const void *fn;
    if (pl.cell == 2) fn = pl.all_smem ? (const void *)match_kernel<uint16_t, false, kJumpK>
                                       : (const void *)match_kernel<uint16_t, true, kJumpK>;
    else fn = pl.all_smem ? (const void *)match_kernel<uint32_t, false, kJumpK>
                          : (const void *)match_kernel<uint32_t, true, kJumpK>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
    if (e != cudaSuccess) return e;
    uint64_t grid = (a.nslices + kMWarps - 1) / kMWarps;
    if (grid > (uint64_t)pl.sms) grid = pl.sms;
    e = cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(kMT), args, pl.smem, (cudaStream_t)stream);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace pfac
