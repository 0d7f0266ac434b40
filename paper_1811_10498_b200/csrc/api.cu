// C-ABI of libpfac (declared and documented in include/pfac.h).  Argument checking, device
// selection from the buffers' owning device, device-image upload, and error reporting.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/pfac.h"
#include "pfac_internal.h"

namespace pfac {
static thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

static int cuda_fail(int e, const char *where) {
    char msg[256];
    snprintf(msg, sizeof msg, "%s: CUDA error %d (%s)", where, e, cudaGetErrorString((cudaError_t)e));
    return fail(e == cudaErrorMemoryAllocation ? PFAC_E_OOM : PFAC_E_CUDA, msg);
}

// Restores the calling thread's current device on scope exit: entry points switch to the device that
// owns their buffers and must not leave it current for the caller (pfac.h conventions).
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard &) = delete;
    DeviceGuard &operator=(const DeviceGuard &) = delete;
};

// Make the device that owns `p` current for this runtime on this thread (torch's runtime and ours
// keep separate "current device" state).  Returns the device or -1 if p is not device memory.
static int device_of(const void *p) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged) return -1;
    if (cudaSetDevice(attr.device) != cudaSuccess) return -1;
    return attr.device;
}

static inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// The automaton's image on `device`, uploading it on first use.
static int get_image(const pfac_automaton *ca, int device, DeviceImage **out) {
    auto *a = const_cast<pfac_automaton *>(ca);
    std::lock_guard<std::mutex> lock(a->mu);
    for (DeviceImage *im : a->images)
        if (im->device == device) {
            *out = im;
            return PFAC_OK;
        }
    const HostImage &h = a->host_image;
    auto *im = new (std::nothrow) DeviceImage();
    if (!im) return fail(PFAC_E_OOM, "device image: host allocation failed");
    im->device = device;
    im->K = h.K;
    im->S = h.S;
    im->root = h.root;
    im->maxlen = a->maxlen;
    im->minlen = a->minlen;
    im->short_pat = h.short_pat;
    if (!fb_addressing_ok(device)) {
        delete im;
        return fail(PFAC_E_CUDA, "device image: unexpected reserved shared memory per block (match.cu kFBSmemBase)");
    }
    im->plan = plan_match(device, h, a->maxlen);
    // One allocation [J2 | T | F | J | FB] (256-byte aligned parts); the L2 access-policy window
    // covers the J2 prefix.
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    // J2 and the chain-head row copies HR together form the L2-persisting prefix
    const size_t bJ2only = al(h.J2.size() * 4), bJ2 = bJ2only + al(h.HR.size() * 4), bT = al(h.T.size()), bF = al(h.F.size()), bJ = al(h.J.size()),
                 bFB = al(h.FB.size() * 4), bC = al(a->prefix_dev.size() * 4),
                 bCF = al(a->prefix_flat.size() * 4);
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaMalloc(&im->d_base, bJ2 + bT + bF + bJ + bFB + bC + bCF);
    if (e == cudaSuccess) {
        uint8_t *b = reinterpret_cast<uint8_t *>(im->d_base);
        im->d_J2 = h.K2 ? reinterpret_cast<uint32_t *>(b) : nullptr;
        im->d_HR = h.HR.empty() ? nullptr : reinterpret_cast<const uint32_t *>(b + bJ2only);
        im->d_T = b + bJ2;
        im->d_F = b + bJ2 + bT;
        im->d_J = b + bJ2 + bT + bF;
        im->d_FB = h.K2 ? reinterpret_cast<uint32_t *>(b + bJ2 + bT + bF + bJ) : nullptr;
        uint32_t *dp = reinterpret_cast<uint32_t *>(b + bJ2 + bT + bF + bJ + bFB);
        uint32_t *dpf = reinterpret_cast<uint32_t *>(b + bJ2 + bT + bF + bJ + bFB + bC);
        im->d_prefix = dp;
        im->d_prefix_flat = dpf;
        e = cudaMemcpy(dp, a->prefix_dev.data(), a->prefix_dev.size() * 4, cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cudaMemcpy(dpf, a->prefix_flat.data(), a->prefix_flat.size() * 4, cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cudaMemcpy(im->d_T, h.T.data(), h.T.size(), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(im->d_F, h.F.data(), h.F.size(), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(im->d_J, h.J.data(), h.J.size(), cudaMemcpyHostToDevice);
        if (e == cudaSuccess && h.K2) e = cudaMemcpy(im->d_J2, h.J2.data(), h.J2.size() * 4, cudaMemcpyHostToDevice);
        if (e == cudaSuccess && !h.HR.empty())
            e = cudaMemcpy(const_cast<uint32_t *>(im->d_HR), h.HR.data(), h.HR.size() * 4, cudaMemcpyHostToDevice);
        if (e == cudaSuccess && h.K2) e = cudaMemcpy(im->d_FB, h.FB.data(), h.FB.size() * 4, cudaMemcpyHostToDevice);
    }
    im->K2 = h.K2;
#ifndef PFAC_NO_PERSIST
    if (e == cudaSuccess && h.K2) {
#else
    if (false) {
#endif
        // persisting L2 set-aside (device-wide limit; only grown, never shrunk) for J2 only: a larger
        // set-aside (J2 + the T prefix, up to 79 MB) halved cfg4 and slowed the streaming kernels
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device);
        size_t want = bJ2;
        if (want > (size_t)max_window) want = (size_t)max_window;
        if (want > (size_t)max_persist) want = (size_t)max_persist;
        size_t cur = 0;
        if (want > 0 && cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) == cudaSuccess) {
            if (cur < want && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
                cudaGetLastError();
                want = cur;
            }
            im->l2_persist_bytes = want;
        }
    }
    if (e != cudaSuccess) {
        cudaFree(im->d_base);
        delete im;
        return cuda_fail(e, "device image upload");
    }
    a->images.push_back(im);
    *out = im;
    return PFAC_OK;
}
}  // namespace pfac

using namespace pfac;

extern "C" {

int pfac_build(const uint8_t *bytes, const uint64_t *offsets, uint32_t k, pfac_automaton **out) {
    try {
        return build_automaton(bytes, offsets, k, out);
    } catch (...) {
        return fail(PFAC_E_OOM, "pfac_build: exception");
    }
}

void pfac_free(pfac_automaton *a) {
    if (!a) return;
    for (DeviceImage *im : a->images) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(im->device);
        if (im->scan) free_scan_ctx(im->scan);
        cudaFree(im->d_base);
        cudaSetDevice(prev);
        delete im;
    }
    delete a;
}

uint32_t pfac_num_states(const pfac_automaton *a) { return a ? a->S : 0; }
uint32_t pfac_num_patterns(const pfac_automaton *a) { return a ? a->k : 0; }
uint32_t pfac_max_len(const pfac_automaton *a) { return a ? a->maxlen : 0; }
const uint32_t *pfac_table(const pfac_automaton *a) { return a ? a->table.data() : nullptr; }

int pfac_prepare(const pfac_automaton *a, int device) {
    DeviceGuard guard;
    if (!a) return fail(PFAC_E_ARG, "pfac_prepare: null automaton");
    DeviceImage *im = nullptr;
    return get_image(a, device, &im);
}

uint64_t pfac_packed_words(uint64_t n) { return (((n + 15) / 16) + 3) & ~3ull; }

int pfac_pack_async(const uint8_t *d_text, uint64_t n, uint32_t *d_packed, uint64_t *d_first_bad, void *stream) {
    DeviceGuard guard;
    if (n == 0) {  // nothing to pack; still report "no bad byte"
        if (!d_first_bad) return PFAC_OK;
        if (device_of(d_first_bad) < 0) return fail(PFAC_E_ARG, "pfac_pack_async: d_first_bad is not device memory");
        int e = cudaMemsetAsync(d_first_bad, 0xFF, 8, (cudaStream_t)stream);
        return e ? cuda_fail(e, "pfac_pack_async") : PFAC_OK;
    }
    if (!d_packed || !d_text) return fail(PFAC_E_ARG, "pfac_pack_async: null buffer");
    if (!aligned16(d_packed)) return fail(PFAC_E_ARG, "pfac_pack_async: d_packed must be 16-byte aligned");
    if (device_of(d_packed) < 0) return fail(PFAC_E_ARG, "pfac_pack_async: d_packed is not device memory");
    int e = launch_pack(d_text, n, d_packed, pfac_packed_words(n), d_first_bad, nullptr, stream);
    return e ? cuda_fail(e, "pfac_pack_async") : PFAC_OK;
}

uint64_t pfac_inv_words(uint64_t n) { return (pfac_packed_words(n) + 7) & ~7ull; }

int pfac_pack_barriers_async(const uint8_t *d_text, uint64_t n, uint32_t *d_packed, uint16_t *d_inv,
                             uint64_t *d_first_bad, void *stream) {
    DeviceGuard guard;
    if (!d_inv) return fail(PFAC_E_ARG, "pfac_pack_barriers_async: null d_inv");
    if (n == 0) return pfac_pack_async(d_text, n, d_packed, d_first_bad, stream);
    if (!d_packed || !d_text) return fail(PFAC_E_ARG, "pfac_pack_barriers_async: null buffer");
    if (!aligned16(d_packed) || !aligned16(d_inv))
        return fail(PFAC_E_ARG, "pfac_pack_barriers_async: d_packed and d_inv must be 16-byte aligned");
    if (device_of(d_packed) < 0) return fail(PFAC_E_ARG, "pfac_pack_barriers_async: d_packed is not device memory");
    int e = launch_pack(d_text, n, d_packed, pfac_packed_words(n), d_first_bad, d_inv, stream);
    return e ? cuda_fail(e, "pfac_pack_barriers_async") : PFAC_OK;
}

int pfac_match_packed_async(const pfac_automaton *a, const uint32_t *d_packed, uint64_t n_own, uint64_t n_avail,
                            int32_t *d_out, void *stream) {
    DeviceGuard guard;
    if (!a) return fail(PFAC_E_ARG, "pfac_match_packed_async: null automaton");
    if (n_avail < n_own) return fail(PFAC_E_ARG, "pfac_match_packed_async: n_avail < n_own");
    if (n_own == 0) return PFAC_OK;
    if (!d_packed || !d_out) return fail(PFAC_E_ARG, "pfac_match_packed_async: null buffer");
    if (!aligned16(d_packed) || !aligned16(d_out))
        return fail(PFAC_E_ARG, "pfac_match_packed_async: d_packed and d_out must be 16-byte aligned");
    const int dev = device_of(d_out);
    if (dev < 0) return fail(PFAC_E_ARG, "pfac_match_packed_async: d_out is not device memory");
    DeviceImage *im = nullptr;
    int rc = get_image(a, dev, &im);
    if (rc) return rc;
    int e = launch_match(*im, d_packed, nullptr, n_own, n_avail, d_out, stream);
    return e ? cuda_fail(e, "pfac_match_packed_async") : PFAC_OK;
}

int pfac_match_barriers_async(const pfac_automaton *a, const uint32_t *d_packed, const uint16_t *d_inv,
                              uint64_t n_own, uint64_t n_avail, int32_t *d_out, void *stream) {
    DeviceGuard guard;
    if (!a) return fail(PFAC_E_ARG, "pfac_match_barriers_async: null automaton");
    if (n_avail < n_own) return fail(PFAC_E_ARG, "pfac_match_barriers_async: n_avail < n_own");
    if (n_own == 0) return PFAC_OK;
    if (!d_packed || !d_out || !d_inv) return fail(PFAC_E_ARG, "pfac_match_barriers_async: null buffer");
    if (!aligned16(d_packed) || !aligned16(d_out) || !aligned16(d_inv))
        return fail(PFAC_E_ARG, "pfac_match_barriers_async: buffers must be 16-byte aligned");
    const int dev = device_of(d_out);
    if (dev < 0) return fail(PFAC_E_ARG, "pfac_match_barriers_async: d_out is not device memory");
    DeviceImage *im = nullptr;
    int rc = get_image(a, dev, &im);
    if (rc) return rc;
    int e = launch_match(*im, d_packed, d_inv, n_own, n_avail, d_out, stream);
    return e ? cuda_fail(e, "pfac_match_barriers_async") : PFAC_OK;
}

int pfac_match_checked(const pfac_automaton *a, const uint8_t *d_text, uint64_t n, int32_t *d_out, uint64_t *first_bad,
                       void *stream) {
    if (!a) return fail(PFAC_E_ARG, "pfac_match_checked: null automaton");
    if (first_bad) *first_bad = ~0ull;
    if (n == 0) return PFAC_OK;
    if (!d_text || !d_out) return fail(PFAC_E_ARG, "pfac_match_checked: null buffer");
    if (!aligned16(d_out)) return fail(PFAC_E_ARG, "pfac_match_checked: d_out must be 16-byte aligned");
    const int dev = device_of(d_out);
    if (dev < 0) return fail(PFAC_E_ARG, "pfac_match_checked: d_out is not device memory");
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t words = pfac_packed_words(n), iw = pfac_inv_words(n);
    void *scratch = nullptr;
    cudaError_t e = cudaMallocAsync(&scratch, words * 4 + iw * 2 + 16, st);
    if (e != cudaSuccess) return cuda_fail(e, "pfac_match_checked: scratch allocation");
    uint32_t *d_packed = reinterpret_cast<uint32_t *>(scratch);
    uint16_t *d_inv = reinterpret_cast<uint16_t *>(d_packed + words);
    uint64_t *d_bad = reinterpret_cast<uint64_t *>(d_inv + iw);
    DeviceImage *im = nullptr;
    int rc = get_image(a, dev, &im);
    int ce = rc ? 0 : launch_pack(d_text, n, d_packed, words, d_bad, im->K2 ? d_inv : nullptr, stream);
    uint64_t bad = ~0ull;
    if (!rc && !ce) ce = cudaMemcpyAsync(&bad, d_bad, 8, cudaMemcpyDeviceToHost, st);
    if (!rc && !ce) ce = cudaStreamSynchronize(st);
    if (!rc && !ce) {
        if (first_bad) *first_bad = bad;
        if (bad != ~0ull && !im->K2) {  // barrier semantics live on the filter path
            rc = fail(PFAC_E_NON_ACGT, "pfac_match_checked: non-ACGT text needs the filter image (PFAC_FB16=1)");
        } else {
            ce = launch_match(*im, d_packed, bad != ~0ull ? d_inv : nullptr, n, n, d_out, stream);
            if (!ce) ce = cudaStreamSynchronize(st);
        }
    }
    cudaFreeAsync(scratch, st);
    if (ce) return cuda_fail(ce, "pfac_match_checked");
    return rc;
}

int pfac_match(const pfac_automaton *a, const uint8_t *d_text, uint64_t n, int32_t *d_out, void *stream) {
    return pfac_match_checked(a, d_text, n, d_out, nullptr, stream);
}

int pfac_pack(const uint8_t *d_text, uint64_t n, uint32_t *d_packed, uint64_t *first_bad, void *stream) {
    DeviceGuard guard;
    if (first_bad) *first_bad = ~0ull;
    if (n == 0) return PFAC_OK;
    if (!d_packed || !d_text) return fail(PFAC_E_ARG, "pfac_pack: null buffer");
    if (!aligned16(d_packed)) return fail(PFAC_E_ARG, "pfac_pack: d_packed must be 16-byte aligned");
    if (device_of(d_packed) < 0) return fail(PFAC_E_ARG, "pfac_pack: d_packed is not device memory");
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t *d_bad = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&d_bad), 8, st);
    if (e != cudaSuccess) return cuda_fail(e, "pfac_pack: scratch allocation");
    uint64_t bad = ~0ull;
    int ce = launch_pack(d_text, n, d_packed, pfac_packed_words(n), d_bad, nullptr, stream);
    if (!ce) ce = cudaMemcpyAsync(&bad, d_bad, 8, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(d_bad, st);
    if (!ce) ce = cudaStreamSynchronize(st);
    if (ce) return cuda_fail(ce, "pfac_pack");
    if (first_bad) *first_bad = bad;
    if (bad != ~0ull) {
        char msg[128];
        snprintf(msg, sizeof msg, "pfac_pack: byte %llu is not ACGTacgt", (unsigned long long)bad);
        return fail(PFAC_E_NON_ACGT, msg);
    }
    return PFAC_OK;
}

int pfac_match_packed(const pfac_automaton *a, const uint32_t *d_packed, uint64_t n_own, uint64_t n_avail,
                      int32_t *d_out, void *stream) {
    DeviceGuard guard;
    int rc = pfac_match_packed_async(a, d_packed, n_own, n_avail, d_out, stream);
    if (rc != PFAC_OK || n_own == 0) return rc;
    const cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    return e ? cuda_fail(e, "pfac_match_packed") : PFAC_OK;
}

int pfac_set_text_kernel(pfac_automaton *a, int mode) {
    if (!a) return fail(PFAC_E_ARG, "pfac_set_text_kernel: null automaton");
    if (mode < -1 || mode > 3) return fail(PFAC_E_ARG, "pfac_set_text_kernel: mode must be -1, 0, 1, 2 or 3");
    a->text_kernel.store(mode, std::memory_order_relaxed);
    return PFAC_OK;
}

int pfac_text_walk_stats(const pfac_automaton *a, const uint8_t *h_text, uint64_t n, uint64_t stride, uint32_t deep,
                         double *deep_frac, double *mean_steps) {
    return text_walk_stats(a, h_text, n, stride, deep, deep_frac, mean_steps);
}

constexpr uint32_t kDeepWalk = 16;       // pfac_plan_text: a walk of >= 16 transitions is "deep"
constexpr double kWalkHeavyShare = 0.01;  // ... and >= 1% deep walks make a text walk-heavy (cfg5: 21%, cfg2-4 < 0.04%)

int pfac_plan_text(pfac_automaton *a, const uint8_t *h_sample, uint64_t n, uint64_t stride, int *mode,
                   double *deep_frac) {
    double df = 0, ms = 0;
    const int rc = text_walk_stats(a, h_sample, n, stride, kDeepWalk, &df, &ms);
    if (rc != PFAC_OK) return rc;
    const int m = df >= kWalkHeavyShare ? 3 : -1;
    a->text_kernel.store(m, std::memory_order_relaxed);
    if (mode) *mode = m;
    if (deep_frac) *deep_frac = df;
    return PFAC_OK;
}

uint64_t pfac_compact_workspace_bytes(uint64_t n) { return compact_workspace_bytes(n); }

int pfac_match_compact_barriers_async(const pfac_automaton *a, const uint32_t *d_packed, const uint16_t *d_inv,
                                      uint64_t n_own, uint64_t n_avail, int32_t *d_out, uint64_t pos_base,
                                      uint64_t *d_pos, uint32_t *d_pid, uint64_t capacity, uint64_t *d_count,
                                      uint64_t *d_hist, void *d_workspace, void *stream) {
    DeviceGuard guard;
    if (d_inv && !aligned16(d_inv)) return fail(PFAC_E_ARG, "pfac_match_compact_barriers_async: misaligned d_inv");
    if (!a) return fail(PFAC_E_ARG, "pfac_match_compact_async: null automaton");
    if (n_avail < n_own) return fail(PFAC_E_ARG, "pfac_match_compact_async: n_avail < n_own");
    if (!d_count || !d_workspace) return fail(PFAC_E_ARG, "pfac_match_compact_async: null d_count / d_workspace");
    if (capacity > 0 && (!d_pos || !d_pid)) return fail(PFAC_E_ARG, "pfac_match_compact_async: null d_pos / d_pid");
    if (n_own > 0 && (!d_packed || !d_out)) return fail(PFAC_E_ARG, "pfac_match_compact_async: null buffer");
    if (n_own > 0 && (!aligned16(d_packed) || !aligned16(d_out)))
        return fail(PFAC_E_ARG, "pfac_match_compact_async: d_packed and d_out must be 16-byte aligned");
    const int dev = device_of(d_count);
    if (dev < 0) return fail(PFAC_E_ARG, "pfac_match_compact_async: d_count is not device memory");
    DeviceImage *im = nullptr;
    if (n_own > 0) {
        int rc = get_image(a, dev, &im);
        if (rc) return rc;
    }
    int e = n_own > 0 ? launch_match_compact(*im, a->k, d_packed, d_inv, n_own, n_avail, d_out, pos_base, d_pos, d_pid,
                                             capacity, d_count, d_hist, d_workspace, stream)
                      : cudaMemsetAsync(d_count, 0, 8, (cudaStream_t)stream);
    return e ? cuda_fail(e, "pfac_match_compact_async") : PFAC_OK;
}

uint64_t pfac_match_list_workspace_bytes(uint64_t n_own) { return compact_workspace_bytes(n_own) + n_own * 4 + 16; }

int pfac_match_list_async(const pfac_automaton *a, const uint32_t *d_packed, const uint16_t *d_inv, uint64_t n_own,
                          uint64_t n_avail, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid, uint64_t capacity,
                          uint64_t *d_count, uint64_t *d_hist, void *d_workspace, void *stream) {
    DeviceGuard guard;
    if (!a) return fail(PFAC_E_ARG, "pfac_match_list_async: null automaton");
    if (n_avail < n_own) return fail(PFAC_E_ARG, "pfac_match_list_async: n_avail < n_own");
    if (!d_count || !d_workspace) return fail(PFAC_E_ARG, "pfac_match_list_async: null d_count / d_workspace");
    if (capacity > 0 && (!d_pos || !d_pid)) return fail(PFAC_E_ARG, "pfac_match_list_async: null d_pos / d_pid");
    if (n_own > 0 && !d_packed) return fail(PFAC_E_ARG, "pfac_match_list_async: null d_packed");
    if (n_own > 0 && (!aligned16(d_packed) || !aligned16(d_workspace) || (d_inv && !aligned16(d_inv))))
        return fail(PFAC_E_ARG, "pfac_match_list_async: d_packed, d_inv and d_workspace must be 16-byte aligned");
    const int dev = device_of(d_count);
    if (dev < 0) return fail(PFAC_E_ARG, "pfac_match_list_async: d_count is not device memory");
    if (n_own == 0) {
        cudaError_t e = cudaMemsetAsync(d_count, 0, 8, (cudaStream_t)stream);
        return e ? cuda_fail(e, "pfac_match_list_async") : PFAC_OK;
    }
    DeviceImage *im = nullptr;
    int rc = get_image(a, dev, &im);
    if (rc) return rc;
    // the sparse out[] scratch sits after the compaction workspace: written only where a pattern
    // matches, read back only there
    int32_t *scratch = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(d_workspace) +
                                                   ((compact_workspace_bytes(n_own) + 15) & ~15ull));
    int e = launch_match_compact(*im, a->k, d_packed, d_inv, n_own, n_avail, scratch, pos_base, d_pos, d_pid, capacity,
                                 d_count, d_hist, d_workspace, stream, true);
    return e ? cuda_fail(e, "pfac_match_list_async") : PFAC_OK;
}

static uint64_t al16(uint64_t x) { return (x + 15) & ~15ull; }

// Which path pfac_match_text_async runs for this image: 0 = pack -> fused kernel, 1 = the text kernel,
// 2 = the text kernel with 1024-position slices, 3 = that kernel with slices claimed dynamically.
// The plan's measured preference (MatchPlan::txt_pref, txt1k_pref), unless pfac_set_text_kernel (or
// pfac_plan_text) forced 0 (never) / 1 (whenever one fits; 2048 slices first) / 2 or 3 (1024 slices
// whenever they fit).
static int text_kernel_for(const pfac_automaton *a, const DeviceImage &im) {
    const int force = a->text_kernel.load(std::memory_order_relaxed);
    const MatchPlan &pl = im.plan;
    if (!im.K2 || force == 0) return 0;
    if (force == 2 || force == 3) return pl.txt1k_ok ? force : 0;
    if (force == 1) return pl.txt_ok ? 1 : pl.txt1k_ok ? 2 : 0;
    return pl.txt_pref ? 1 : pl.txt1k_pref ? 2 : 0;
}

uint64_t pfac_match_text_workspace_bytes(uint64_t n_own, uint64_t n_avail, int list_only) {
    // [compaction workspace | list-only out[] scratch | two-kernel path: packed words | barrier words]
    return al16(compact_workspace_bytes(n_own)) + (list_only ? al16(n_own * 4) : 0) +
           al16(pfac_packed_words(n_avail) * 4) + al16(pfac_inv_words(n_avail) * 2) + 16;
}

static int match_text_impl(const pfac_automaton *a, DeviceImage &imr, const uint8_t *d_text, uint64_t n_own,
                           uint64_t n_avail, int32_t *d_out, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                           uint64_t capacity, uint64_t *d_count, uint64_t *d_hist, uint64_t *d_first_bad,
                           void *d_workspace, void *stream);

int pfac_match_text_async(const pfac_automaton *a, const uint8_t *d_text, uint64_t n_own, uint64_t n_avail,
                          int32_t *d_out, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid, uint64_t capacity,
                          uint64_t *d_count, uint64_t *d_hist, uint64_t *d_first_bad, void *d_workspace,
                          void *stream) {
    DeviceGuard guard;
    if (!a) return fail(PFAC_E_ARG, "pfac_match_text_async: null automaton");
    if (n_avail < n_own) return fail(PFAC_E_ARG, "pfac_match_text_async: n_avail < n_own");
    if (!d_count || !d_workspace) return fail(PFAC_E_ARG, "pfac_match_text_async: null d_count / d_workspace");
    if (capacity > 0 && (!d_pos || !d_pid)) return fail(PFAC_E_ARG, "pfac_match_text_async: null d_pos / d_pid");
    if (n_own > 0 && !d_text) return fail(PFAC_E_ARG, "pfac_match_text_async: null d_text");
    if (!aligned16(d_workspace) || (d_out && !aligned16(d_out)))
        return fail(PFAC_E_ARG, "pfac_match_text_async: d_out and d_workspace must be 16-byte aligned");
    const int dev = device_of(d_count);
    if (dev < 0) return fail(PFAC_E_ARG, "pfac_match_text_async: d_count is not device memory");
    cudaStream_t st = (cudaStream_t)stream;
    if (n_own == 0) {
        cudaError_t e = cudaMemsetAsync(d_count, 0, 8, st);
        if (e == cudaSuccess && d_first_bad) e = cudaMemsetAsync(d_first_bad, 0xFF, 8, st);
        return e ? cuda_fail(e, "pfac_match_text_async") : PFAC_OK;
    }
    DeviceImage *im = nullptr;
    int rc = get_image(a, dev, &im);
    if (rc) return rc;
    const int e = match_text_impl(a, *im, d_text, n_own, n_avail, d_out, pos_base, d_pos, d_pid, capacity, d_count,
                                  d_hist, d_first_bad, d_workspace, stream);
    return e ? cuda_fail(e, "pfac_match_text_async") : PFAC_OK;
}

// The text call's GPU work on one device image (pfac_match_text_async, pfac_scan_host's chunks):
// the text kernel when the plan takes it and the text is 16-byte aligned, else pack -> fused kernel
// through the workspace.  n_own > 0.  Returns a cudaError_t.
static int match_text_impl(const pfac_automaton *a, DeviceImage &imr, const uint8_t *d_text, uint64_t n_own,
                           uint64_t n_avail, int32_t *d_out, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                           uint64_t capacity, uint64_t *d_count, uint64_t *d_hist, uint64_t *d_first_bad,
                           void *d_workspace, void *stream) {
    DeviceImage *im = &imr;
    uint8_t *ws = reinterpret_cast<uint8_t *>(d_workspace);
    const bool list_only = d_out == nullptr;
    uint8_t *after = ws + al16(compact_workspace_bytes(n_own));
    int32_t *out = list_only ? reinterpret_cast<int32_t *>(after) : d_out;
    if (list_only) after += al16(n_own * 4);
    int e;
    const int tk = text_kernel_for(a, *im);
    if (tk && aligned16(d_text)) {
        e = launch_match_compact(*im, a->k, nullptr, nullptr, n_own, n_avail, out, pos_base, d_pos, d_pid, capacity,
                                 d_count, d_hist, d_workspace, stream, list_only, d_text, d_first_bad, nullptr,
                                 tk >= 2, tk == 3);
    } else {  // two kernels through the workspace (unaligned text, or a halo too long for the plan)
        // pack records the first bad index over the readable text; the fused kernel skips the barrier
        // bits when there is none and writes the owned part of it to d_first_bad
        uint32_t *packed = reinterpret_cast<uint32_t *>(after);
        uint16_t *inv = reinterpret_cast<uint16_t *>(after + al16(pfac_packed_words(n_avail) * 4));
        uint64_t *bad_all = reinterpret_cast<uint64_t *>(after + al16(pfac_packed_words(n_avail) * 4) +
                                                         al16(pfac_inv_words(n_avail) * 2));
        e = launch_pack(d_text, n_avail, packed, pfac_packed_words(n_avail), bad_all, inv, stream);
        if (!e)
            e = launch_match_compact(*im, a->k, packed, inv, n_own, n_avail, out, pos_base, d_pos, d_pid, capacity,
                                     d_count, d_hist, d_workspace, stream, list_only, nullptr, d_first_bad, bad_all);
    }
    return e;
}

int pfac_match_compact_async(const pfac_automaton *a, const uint32_t *d_packed, uint64_t n_own, uint64_t n_avail,
                             int32_t *d_out, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid, uint64_t capacity,
                             uint64_t *d_count, uint64_t *d_hist, void *d_workspace, void *stream) {
    return pfac_match_compact_barriers_async(a, d_packed, nullptr, n_own, n_avail, d_out, pos_base, d_pos, d_pid,
                                             capacity, d_count, d_hist, d_workspace, stream);
}

int pfac_compact_async(const int32_t *d_out, uint64_t n, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                       uint64_t capacity, uint64_t *d_count, uint32_t k, uint64_t *d_hist, void *d_workspace,
                       void *stream) {
    DeviceGuard guard;
    if (!d_count || !d_workspace) return fail(PFAC_E_ARG, "pfac_compact_async: null d_count / d_workspace");
    if (n > 0 && !d_out) return fail(PFAC_E_ARG, "pfac_compact_async: null d_out");
    if (capacity > 0 && (!d_pos || !d_pid)) return fail(PFAC_E_ARG, "pfac_compact_async: null d_pos / d_pid");
    if (n > 0 && !aligned16(d_out)) return fail(PFAC_E_ARG, "pfac_compact_async: d_out must be 16-byte aligned");
    if (device_of(d_count) < 0) return fail(PFAC_E_ARG, "pfac_compact_async: d_count is not device memory");
    int e = launch_compact(d_out, n, pos_base, d_pos, d_pid, capacity, d_count, k, d_hist, d_workspace, stream);
    return e ? cuda_fail(e, "pfac_compact_async") : PFAC_OK;
}

int pfac_compact(const int32_t *d_out, uint64_t n, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                 uint64_t capacity, uint64_t *count, uint32_t k, uint64_t *d_hist, void *stream) {
    DeviceGuard guard;
    if (!count) return fail(PFAC_E_ARG, "pfac_compact: null count");
    if (n > 0 && !d_out) return fail(PFAC_E_ARG, "pfac_compact: null d_out");
    const void *probe = n > 0 ? (const void *)d_out : (const void *)d_pos;
    if (!probe || device_of(probe) < 0) return fail(PFAC_E_ARG, "pfac_compact: d_out is not device memory");
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t wsb = compact_workspace_bytes(n);
    void *ws = nullptr;
    cudaError_t e = cudaMallocAsync(&ws, wsb + 8, st);
    if (e != cudaSuccess) return cuda_fail(e, "pfac_compact: workspace allocation");
    uint64_t *d_count = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(ws) + wsb);
    int rc = pfac_compact_async(d_out, n, pos_base, d_pos, d_pid, capacity, d_count, k, d_hist, ws, stream);
    uint64_t c = 0;
    int ce = 0;
    if (rc == PFAC_OK) {
        ce = cudaMemcpyAsync(&c, d_count, 8, cudaMemcpyDeviceToHost, st);
        if (!ce) ce = cudaStreamSynchronize(st);
    }
    cudaFreeAsync(ws, st);
    if (rc) return rc;
    if (ce) return cuda_fail(ce, "pfac_compact");
    *count = c;
    if (c > capacity) {
        char msg[128];
        snprintf(msg, sizeof msg, "pfac_compact: %llu matches > capacity %llu", (unsigned long long)c,
                 (unsigned long long)capacity);
        return fail(PFAC_E_CAPACITY, msg);
    }
    return PFAC_OK;
}

}  // extern "C"

namespace pfac {
// Device buffers of one pipeline slot of pfac_scan_host.
struct ScanSlot {
    uint8_t *text = nullptr;
    uint64_t *pos = nullptr, *cnt = nullptr, *bad = nullptr;
    uint32_t *pid = nullptr;
    void *ws = nullptr;  // pfac_match_text_workspace_bytes(chunk, chunk + halo, 1): list only, no dense out[]
    uint64_t cap = 0;
    cudaEvent_t h2d = nullptr, done = nullptr;
};
// pfac_scan_host's pipeline resources, kept with the device image and reused across calls.
struct ScanCtx {
    std::mutex mu;
    uint64_t chunk = 0, halo = 0;
    cudaStream_t cs = nullptr, xs = nullptr;  // compute, copy
    ScanSlot slot[2];
    uint64_t *h_cnt = nullptr;  // pinned: per-slot count and first-bad
    ~ScanCtx() {
        for (ScanSlot &sl : slot) {
            cudaFree(sl.text);
            cudaFree(sl.pos);
            cudaFree(sl.pid);
            cudaFree(sl.cnt);
            cudaFree(sl.ws);
            if (sl.h2d) cudaEventDestroy(sl.h2d);
            if (sl.done) cudaEventDestroy(sl.done);
        }
        if (h_cnt) cudaFreeHost(h_cnt);
        if (cs) cudaStreamDestroy(cs);
        if (xs) cudaStreamDestroy(xs);
    }
    cudaError_t init(uint64_t chunk_, uint64_t halo_) {
        chunk = chunk_;
        halo = halo_;
        cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaMallocHost(&h_cnt, 4 * sizeof(uint64_t));
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            ScanSlot &sl = slot[i];
            sl.cap = chunk / 8 + 65536;
            e = cudaMalloc(&sl.text, chunk + halo + 16);
            if (e == cudaSuccess) e = cudaMalloc(&sl.pos, sl.cap * 8);
            if (e == cudaSuccess) e = cudaMalloc(&sl.pid, sl.cap * 4);
            if (e == cudaSuccess) e = cudaMalloc(&sl.cnt, 16);
            if (e == cudaSuccess) e = cudaMalloc(&sl.ws, pfac_match_text_workspace_bytes(chunk, chunk + halo, 1));
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sl.h2d, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming);
            sl.bad = sl.cnt + 1;
        }
        return e;
    }
};
void free_scan_ctx(ScanCtx *c) { delete c; }
constexpr uint64_t kScanChunk = 1ull << 26;  // 64 Mbases per pipeline chunk
}  // namespace pfac

extern "C" {

int pfac_scan_host(const pfac_automaton *a, int device, const uint8_t *h_text, uint64_t n_own, uint64_t n_avail,
                   uint64_t pos_base, uint64_t *h_pos, uint32_t *h_pid, uint64_t capacity, uint64_t *count,
                   uint64_t *first_bad) {
    DeviceGuard guard;
    if (!a || !count) return fail(PFAC_E_ARG, "pfac_scan_host: null automaton / count");
    if (n_avail < n_own) return fail(PFAC_E_ARG, "pfac_scan_host: n_avail < n_own");
    const uint64_t n = n_own, N = n_avail;  // positions to match; bases readable
    if (n > 0 && !h_text) return fail(PFAC_E_ARG, "pfac_scan_host: null text");
    if (capacity > 0 && (!h_pos || !h_pid)) return fail(PFAC_E_ARG, "pfac_scan_host: null h_pos / h_pid");
    *count = 0;
    if (n == 0) return PFAC_OK;
    if (cudaSetDevice(device) != cudaSuccess) return fail(PFAC_E_ARG, "pfac_scan_host: bad device");
    DeviceImage *im = nullptr;
    int rc = get_image(a, device, &im);
    if (rc) return rc;
    const uint64_t halo = a->maxlen > 0 ? a->maxlen - 1 : 0;
    {
        std::lock_guard<std::mutex> lock(const_cast<pfac_automaton *>(a)->mu);
        if (!im->scan) {
            auto *ctx = new (std::nothrow) ScanCtx();
            if (!ctx) return fail(PFAC_E_OOM, "pfac_scan_host: host allocation failed");
            cudaError_t e = ctx->init(kScanChunk, halo);
            if (e != cudaSuccess) {
                delete ctx;
                return cuda_fail(e, "pfac_scan_host: pipeline allocation");
            }
            im->scan = ctx;
        }
    }
    ScanCtx &X = *im->scan;
    std::lock_guard<std::mutex> lock(X.mu);
    const uint64_t chunk = X.chunk;
    const uint64_t nchunks = (n + chunk - 1) / chunk;
    cudaStream_t cs = X.cs, xs = X.xs;
    ScanSlot *slot = X.slot;
    uint64_t *h_cnt = X.h_cnt;
    cudaError_t e = cudaSuccess;
    uint64_t total = 0, bad_at = ~0ull;
    // chunk c owns positions [c*chunk, c*chunk + own) and reads bases up to avail past its start
    auto own_of = [&](uint64_t c) { return (n - c * chunk) < chunk ? (n - c * chunk) : chunk; };
    auto avail_of = [&](uint64_t c) {
        const uint64_t own = own_of(c);
        return (N - c * chunk) < own + halo ? (N - c * chunk) : own + halo;
    };
    // enqueue chunk c (copy in, the text call in list-only form -- pack + match + compact in one kernel
    // where the plan takes it; barriers handled per slice --, count + first owned bad index back)
    auto enqueue = [&](uint64_t c) -> cudaError_t {
        ScanSlot &sl = slot[c & 1];
        const uint64_t s0 = c * chunk, own = own_of(c), avail = avail_of(c);
        cudaError_t r = cudaStreamWaitEvent(xs, sl.done, 0);  // the slot's previous chunk is finished
        if (r == cudaSuccess) r = cudaMemcpyAsync(sl.text, h_text + s0, avail, cudaMemcpyHostToDevice, xs);
        if (r == cudaSuccess) r = cudaEventRecord(sl.h2d, xs);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(cs, sl.h2d, 0);
        if (r == cudaSuccess)
            r = (cudaError_t)match_text_impl(a, *im, sl.text, own, avail, nullptr, pos_base + s0, sl.pos, sl.pid,
                                             sl.cap, sl.cnt, nullptr, sl.bad, sl.ws, cs);
        if (r == cudaSuccess) r = cudaMemcpyAsync(h_cnt + 2 * (c & 1), sl.cnt, 16, cudaMemcpyDeviceToHost, cs);
        if (r == cudaSuccess) r = cudaEventRecord(sl.done, cs);
        return r;
    };
    e = enqueue(0);
    for (uint64_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
        if (c + 1 < nchunks) e = enqueue(c + 1);  // next chunk's copy overlaps this chunk's kernels
        if (e != cudaSuccess) break;
        ScanSlot &sl = slot[c & 1];
        e = cudaEventSynchronize(sl.done);
        if (e != cudaSuccess) break;
        uint64_t m = h_cnt[2 * (c & 1)];
        const uint64_t b = h_cnt[2 * (c & 1) + 1];  // pos_base-relative, owned positions only
        if (b != ~0ull && bad_at == ~0ull) bad_at = b - pos_base;
        // Dense chunk: grow this slot's list (kept for later calls) and redo it, after the next
        // chunk's enqueue (which touches only the other slot).
        const uint64_t own = own_of(c), avail = avail_of(c);
        if (m > sl.cap && e == cudaSuccess) {
            e = cudaStreamSynchronize(cs);
            cudaFree(sl.pos);
            cudaFree(sl.pid);
            sl.cap = m + 1024;
            if (e == cudaSuccess) e = cudaMalloc(&sl.pos, sl.cap * 8);
            if (e == cudaSuccess) e = cudaMalloc(&sl.pid, sl.cap * 4);
            if (e == cudaSuccess)
                e = (cudaError_t)match_text_impl(a, *im, sl.text, own, avail, nullptr, pos_base + c * chunk, sl.pos,
                                                 sl.pid, sl.cap, sl.cnt, nullptr, sl.bad, sl.ws, cs);
            if (e == cudaSuccess) e = cudaMemcpyAsync(h_cnt + 2 * (c & 1), sl.cnt, 8, cudaMemcpyDeviceToHost, cs);
            if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
            m = h_cnt[2 * (c & 1)];
        }
        if (e != cudaSuccess) break;
        const uint64_t take = total >= capacity ? 0 : (capacity - total < m ? capacity - total : m);
        if (take) {
            e = cudaMemcpyAsync(h_pos + total, sl.pos, take * 8, cudaMemcpyDeviceToHost, cs);
            if (e == cudaSuccess) e = cudaMemcpyAsync(h_pid + total, sl.pid, take * 4, cudaMemcpyDeviceToHost, cs);
            if (e == cudaSuccess) e = cudaEventRecord(sl.done, cs);  // the slot is free after these copies
        }
        total += m;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(xs);
    if (e != cudaSuccess) return cuda_fail(e, "pfac_scan_host");
    *count = total;
    if (first_bad) *first_bad = bad_at;
    if (total > capacity) {
        char msg[128];
        snprintf(msg, sizeof msg, "pfac_scan_host: %llu matches > capacity %llu", (unsigned long long)total,
                 (unsigned long long)capacity);
        return fail(PFAC_E_CAPACITY, msg);
    }
    return PFAC_OK;
}

const uint32_t *pfac_prefix_chain(const pfac_automaton *a) { return a ? a->prefix.data() : nullptr; }

uint64_t pfac_expand_workspace_bytes(void) { return expand_workspace_bytes(); }

int pfac_expand_async(const pfac_automaton *a, const uint64_t *d_pos, const uint32_t *d_pid, const uint64_t *d_count,
                      uint64_t in_capacity, uint64_t *d_pos_all, uint32_t *d_pid_all, uint64_t capacity,
                      uint64_t *d_count_all, void *d_workspace, void *stream) {
    DeviceGuard guard;
    if (!a) return fail(PFAC_E_ARG, "pfac_expand_async: null automaton");
    if (!d_count || !d_count_all || !d_workspace)
        return fail(PFAC_E_ARG, "pfac_expand_async: null d_count / d_count_all / d_workspace");
    if (in_capacity > 0 && (!d_pos || !d_pid)) return fail(PFAC_E_ARG, "pfac_expand_async: null d_pos / d_pid");
    if (capacity > 0 && (!d_pos_all || !d_pid_all))
        return fail(PFAC_E_ARG, "pfac_expand_async: null d_pos_all / d_pid_all");
    const int dev = device_of(d_count_all);
    if (dev < 0) return fail(PFAC_E_ARG, "pfac_expand_async: d_count_all is not device memory");
    DeviceImage *im = nullptr;
    int rc = get_image(a, dev, &im);
    if (rc) return rc;
    int e = launch_expand(*im, a->k, d_pos, d_pid, d_count, in_capacity, d_pos_all, d_pid_all, capacity, d_count_all,
                          d_workspace, stream);
    return e ? cuda_fail(e, "pfac_expand_async") : PFAC_OK;
}

int pfac_expand(const pfac_automaton *a, const uint64_t *d_pos, const uint32_t *d_pid, uint64_t count,
                uint64_t *d_pos_all, uint32_t *d_pid_all, uint64_t capacity, uint64_t *count_all, void *stream) {
    DeviceGuard guard;
    if (!count_all) return fail(PFAC_E_ARG, "pfac_expand: null count_all");
    *count_all = 0;
    if (!a) return fail(PFAC_E_ARG, "pfac_expand: null automaton");
    if (capacity > 0 && !d_pos_all) return fail(PFAC_E_ARG, "pfac_expand: null d_pos_all");
    const void *probe = capacity > 0 ? (const void *)d_pos_all : (const void *)d_pos;
    if (!probe) return count == 0 ? PFAC_OK : fail(PFAC_E_ARG, "pfac_expand: null buffers");
    const int dev = device_of(probe);
    if (dev < 0) return fail(PFAC_E_ARG, "pfac_expand: buffers are not device memory");
    cudaStream_t st = (cudaStream_t)stream;
    void *scratch = nullptr;
    cudaError_t ce = cudaMallocAsync(&scratch, expand_workspace_bytes() + 16, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "pfac_expand: scratch allocation");
    uint64_t *d_counts = reinterpret_cast<uint64_t *>(scratch);  // [0] = count in, [1] = count out
    void *ws = d_counts + 2;
    uint64_t h[2] = {count, 0};
    int rc = PFAC_OK;
    ce = cudaMemcpyAsync(d_counts, h, 8, cudaMemcpyHostToDevice, st);
    if (!ce) {
        rc = pfac_expand_async(a, d_pos, d_pid, d_counts, count, d_pos_all, d_pid_all, capacity, d_counts + 1, ws,
                               stream);
        if (!rc) ce = cudaMemcpyAsync(&h[1], d_counts + 1, 8, cudaMemcpyDeviceToHost, st);
        if (!rc && !ce) ce = cudaStreamSynchronize(st);
    }
    cudaFreeAsync(scratch, st);
    if (ce) return cuda_fail(ce, "pfac_expand");
    if (rc) return rc;
    *count_all = h[1];
    if (h[1] > capacity) {
        char msg[128];
        snprintf(msg, sizeof msg, "pfac_expand: %llu occurrences > capacity %llu", (unsigned long long)h[1],
                 (unsigned long long)capacity);
        return fail(PFAC_E_CAPACITY, msg);
    }
    return PFAC_OK;
}

int pfac_image_info(const pfac_automaton *a, int device, pfac_image_info_t *out) {
    DeviceGuard guard;
    if (!a || !out) return fail(PFAC_E_ARG, "pfac_image_info: null argument");
    DeviceImage *im = nullptr;
    int rc = get_image(a, device, &im);
    if (rc) return rc;
    const HostImage &h = a->host_image;
    out->device = device;
    out->cell_bytes = im->plan.cell;
    out->K = (uint32_t)im->K;
    out->K2 = (uint32_t)im->K2;
    out->states = im->S;
    out->window_rows = im->plan.window;
    out->all_smem = im->plan.all_smem ? 1u : 0u;
    out->short_pat = im->short_pat;
    out->smem_bytes = im->plan.smem;
    out->l2_persist_bytes = im->l2_persist_bytes;
    out->image_bytes = h.J.size() + h.T.size() + h.F.size() + h.J2.size() * 4 + h.FB.size() * 4 + h.HR.size() * 4 +
                       a->prefix_dev.size() * 4 + a->prefix_flat.size() * 4;
    out->hr_rows = (uint32_t)(h.HR.size() / 4);
    out->hr_nb_rows = h.hr_nb;
    out->text_kernel = (uint32_t)text_kernel_for(a, *im);
    out->text_window_rows = out->text_kernel == 2 ? im->plan.window_txt1k : im->plan.window_txt;
    return PFAC_OK;
}

const char *pfac_last_error(void) { return g_err.c_str(); }

}  // extern "C"
