// Internal declarations shared by the host builder (builder.cpp), the C-ABI (api.cu) and the
// kernels (kernels.cu).  Not part of the public ABI (see include/pfac.h).
#pragma once

#include <array>
#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

namespace pfac {

// Device image constants.
#ifndef PFAC_K16
#define PFAC_K16 8
#endif
constexpr int kJumpK16 = PFAC_K16;  // K for uint16 images: J has 4^8 cells = 128 KiB
constexpr int kJumpK32 = 7;   // K for uint32 images: J has 4^7 cells = 64 KiB (edge use only)
#ifndef PFAC_FBK
#define PFAC_FBK 10
#endif
constexpr int kFilterK = PFAC_FBK;  // K1-mer filter bitmap, 4^10 bits = 128 KiB (A/B knob)
#ifndef PFAC_FB16
#define PFAC_FB16 1
#endif
constexpr bool kFilterSmall = PFAC_FB16;  // filter + J2 for uint16 images too (A/B knob)
#ifndef PFAC_K2MAX
#define PFAC_K2MAX 11
#endif
constexpr int kK2Max = PFAC_K2MAX;  // largest second-level jump length (4^11 cells = 16 MiB)
#ifndef PFAC_K2MIN
#define PFAC_K2MIN PFAC_FBK
#endif
constexpr int kK2Min = PFAC_K2MIN;  // smallest (>= kFilterK: the filter must not look further than J2)
constexpr int kChainMax = 16; // bases per uint16 chain row (2 bits each -> one 32-bit word)
// uint32 chain rows: up to 32 forced bases (cells 1 and 3), and the answer of a walk that consumes the
// whole span when the span's end state has no transitions (cell 0 bits 6-29: F(end) + 1, 0 = none)
#ifndef PFAC_CHAIN32
#define PFAC_CHAIN32 1  // A/B knob: 0 = 16 bases per uint32 chain row
#endif
constexpr int kChainMax32 = PFAC_CHAIN32 ? 32 : 16;
#ifndef PFAC_ENDDEAD
#define PFAC_ENDDEAD 1  // A/B knob: 0 = no end-state answers in uint32 chain rows
#endif
constexpr bool kEndDead = PFAC_ENDDEAD;
constexpr uint32_t kChainLenMask32 = 63u, kEndShift = 6, kEndMask = 0xFFFFFFu;
// uint16 chain rows: FSTEP (cell 0 bit 13) -- F(u + j) = F(u) + j for every j < L (nested prefix
// families with consecutive ids), so a walk ending inside the span answers without an F lookup
#ifndef PFAC_FSTEP
#define PFAC_FSTEP 1  // A/B knob
#endif
constexpr bool kFStep = PFAC_FSTEP;
constexpr uint32_t kFStep16 = 0x2000u;
// Ablation (the paper's "two arrays vs one merged array"): PFAC_MERGED_F=1
// stores F(s) in cell 4 of an 8-cell row next to the 4 transitions, so a walk that ends at a branch
// state reads its answer from the row it already holds (rows twice as wide).  Default: T rows of 4
// cells and the separate F array (chain rows carry F(s) in their spare cell either way).
#ifndef PFAC_MERGED_F
#define PFAC_MERGED_F 0
#endif
constexpr bool kMergedF = PFAC_MERGED_F;
constexpr uint32_t kRowCells = kMergedF ? 8 : 4;
// J2 entry encoding (uint32, the same for both cell widths): ALIVE | id of the depth-K2 state, or
// the answer of a walk that dies within K2 bases.  uint32 images with chain-head copies (HR):
//   ALIVE | HR | h                      -> the head's row is HR[h]   (h < 2^29)
//   ALIVE | HR | NB | b4 << 21 | h      -> the same, and the row is a NOFIN chain of L >= 4 bases
//                                          with F = 0 whose first 4 forced bases are b4 (h < 2^21)
constexpr uint32_t kJ2Alive = 0x80000000u, kJ2HR = 0x40000000u, kJ2NB = 0x20000000u;
constexpr uint32_t kHRBases = 4, kHRIndexBitsNB = 21;

// Host-side device image: everything the match kernel reads, already in its cell width.
//  * Device ids 1..S number the states deep-first and chain-major: first the states at depth >= K
//    (breadth-first over chain heads starting from the depth-K states that J hands out, each head
//    followed by its run of single-child descendants), then the states at depth < K the same way
//    from the root.  Every chain row spans consecutive ids (runs never cross depth K), and the
//    shared-memory window -- a prefix of the ids -- starts with the states walks resume from.
//  * T row of state s (4 cells): a BRANCH row holds the child id per base A,C,G,T (0 = none); a
//    CHAIN row (s has exactly one child) holds CHAIN|NOFIN|L in cell 0, the next L <= 16 bases of
//    the chain, 2 bits each (base i at bits 2i), in the following 32 bits, and F(s) in the last
//    cell used (cell 3 for uint16, cell 2 for uint32).  After m matching bases the walk is in state
//    s + m; NOFIN says no state strictly inside (s, s+L) is final, so F(s + m) = F(s) for m < L.
//  * F[s] = pattern id of the deepest final state on the root path of s (0 = none).
//  * J[x] for each K-mer x (base t at bits 2t): ALIVE|id of the depth-K state, or F of the deepest
//    state the K-mer reaches when the walk dies within K bases.
//  * uint32 images (large automata) replace J in shared memory by FB, a 4^10-bit filter: bit x says
//    whether the 10-mer x starts a walk that survives 10 bases or completes a pattern.  Unflagged
//    positions answer 0; flagged ones are resolved by J2, the jump table over K2-mers (K2 in
//    [10, 11]) kept in global memory under an L2-persisting access-policy window, and the rare
//    survivors walk on from the depth-K2 state; the device numbering then starts at depth K2.
struct HostImage {
    int K = kJumpK32;
    uint32_t cell = 4;                 // bytes per cell: 2 if S < 32768 and k < 32768, else 4
    uint32_t S = 0;                    // device ids 1..S, row 0 is an all-zero dummy
    uint32_t root = 0;                 // device id of the root (= 1)
    uint32_t rows = 0;                 // rows allocated (S + 1 padded to a multiple of 8)
    uint32_t short_pat = 0;            // a pattern shorter than K exists (dead J cells may be nonzero)
    std::vector<uint8_t> J, T, F;      // raw little-endian cells
    int K2 = 0;                        // uint32 images: second-level jump over K2-mers (0 = none)
    std::vector<uint32_t> J2;          // 4^K2 cells, same encoding as J (ALIVE = bit 31); L2-resident
    std::vector<uint32_t> FB;          // K2 > 0: 4^kFilterK-bit filter ("this K1-mer needs J2")
    std::vector<uint32_t> HR;          // uint32 images: copies of the depth-K2 chain-head T rows (4 cells,
                                       // cell 3 = the head's device id); J2 entry ALIVE|HRF|h points at row h
    uint32_t hr_nb = 0;                // HR rows whose J2 entries use the NB form (kJ2NB)
};

// Launch plan of the match kernel for one automaton on one device (match.cu).
struct MatchPlan {
    uint32_t cell = 4;         // bytes per J/T/F cell (HostImage::cell)
    bool all_smem = false;     // every T row / F entry fits in shared memory (no window check)
    uint32_t window = 0;       // device ids [0, window) staged in shared memory
    uint32_t slice_words = 0;  // packed words per warp slice (512 bases + halo)
    size_t smem = 0;           // dynamic shared memory per CTA
    bool all_smem_bar = false; // the same three for the barrier-mode variant (BAR)
    uint32_t window_bar = 0;
    size_t smem_bar = 0;
    bool txt_ok = false;       // the text-input variant (TXT) fits in shared memory
    bool txt_pref = false;     // ... and is the faster choice for this automaton (plan_match)
    bool txt1k_ok = false;     // the text kernel with 1024-position slices fits (uint32 images)
    bool txt1k_pref = false;   // ... and is the choice (automata over kTxtMaxRows rows)
    bool all_smem_txt1k = false;
    uint32_t window_txt1k = 0;
    uint32_t slice_words_1k = 0;
    size_t smem_txt1k = 0;
    bool all_smem_txt = false; // the same three for it
    uint32_t window_txt = 0;
    size_t smem_txt = 0;
    int sms = 0;
};

// The match kernel's filter lookups assume the dynamic shared memory starts right after the
// per-block reserved region (match.cu, kFBSmemBase); false if this device reserves another size.
bool fb_addressing_ok(int device);

struct ScanCtx;  // pfac_scan_host pipeline resources (api.cu)
void free_scan_ctx(ScanCtx *c);

// A device image resident on one GPU.
struct DeviceImage {
    int device = -1;
    int K = kJumpK32;
    uint32_t S = 0, root = 0;
    uint32_t maxlen = 0, minlen = 0;
    uint32_t short_pat = 0;
    int K2 = 0;
    MatchPlan plan;
    void *d_base = nullptr;                               // one allocation: [J2 | T | F | J | FB]
    void *d_J = nullptr, *d_T = nullptr, *d_F = nullptr;  // cells of plan.cell bytes
    uint32_t *d_J2 = nullptr;                             // K2 > 0: L2-persisting second-level jump
    uint32_t *d_FB = nullptr;                             // K2 > 0: K1-mer filter bitmap
    const uint32_t *d_HR = nullptr;                       // chain-head row copies, 4 cells each (or null)
    const uint32_t *d_prefix = nullptr;                   // prefix_dev (uint4 per pattern)
    const uint32_t *d_prefix_flat = nullptr;              // prefix_flat
    size_t l2_persist_bytes = 0;                          // access-policy window from d_base (0 = none)
    ScanCtx *scan = nullptr;                              // created by the first pfac_scan_host
};

}  // namespace pfac

struct pfac_automaton {
    uint32_t k = 0;       // patterns
    uint32_t S = 0;       // canonical states (incl. root)
    uint32_t maxlen = 0;
    uint32_t minlen = 0;
    std::vector<uint32_t> table;  // canonical S*4, columns A,C,G,T
    std::vector<uint32_t> depth;  // canonical depth of each state
    std::vector<uint32_t> F;      // canonical: deepest final on the root path (pattern id) or 0
    std::vector<uint32_t> prefix;      // 2*(k+1): [2p] = longest pattern that is a proper prefix of p
                                       // (0 = none), [2p+1] = patterns on p's prefix chain incl. p
    std::vector<uint32_t> prefix_dev;  // 4*(k+1): (chain length, parent, flat base lo, hi) per pattern
    std::vector<uint32_t> prefix_flat; // every pattern's chain, shortest first, at its flat base
    pfac::HostImage host_image;   // derived once at build
    std::atomic<int> text_kernel{-1};  // pfac_set_text_kernel: -1 = the plan's choice, else forced 0/1/2
    std::mutex mu;                // guards images
    std::vector<pfac::DeviceImage *> images;
};

namespace pfac {
// Thread-local error message plumbing (api.cu).
int fail(int code, const std::string &msg);

// builder.cpp
int build_automaton(const uint8_t *bytes, const uint64_t *offsets, uint32_t k, pfac_automaton **out);
void derive_host_image(pfac_automaton *a);
int text_walk_stats(const pfac_automaton *a, const uint8_t *h_text, uint64_t n, uint64_t stride, uint32_t deep,
                    double *deep_frac, double *mean_steps);

// kernels.cu launchers (all asynchronous on `stream`); return cudaError_t as int.
int launch_pack(const uint8_t *d_text, uint64_t n, uint32_t *d_packed, uint64_t nwords_padded,
                uint64_t *d_first_bad, uint16_t *d_inv, void *stream);
int launch_match(const DeviceImage &img, const uint32_t *d_packed, const uint16_t *d_inv, uint64_t n_own,
                 uint64_t n_avail, int32_t *d_out, void *stream);
int launch_compact(const int32_t *d_out, uint64_t n, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                   uint64_t capacity, uint64_t *d_count, uint32_t k, uint64_t *d_hist, void *d_workspace,
                   void *stream);
uint64_t compact_workspace_bytes(uint64_t n);
int launch_match_compact(const DeviceImage &img, uint32_t k, const uint32_t *d_packed, const uint16_t *d_inv,
                         uint64_t n_own, uint64_t n_avail, int32_t *d_out, uint64_t pos_base, uint64_t *d_pos,
                         uint32_t *d_pid, uint64_t capacity, uint64_t *d_count, uint64_t *d_hist, void *d_workspace,
                         void *stream, bool list_only = false, const uint8_t *d_text = nullptr,
                         uint64_t *d_first_bad = nullptr, const uint64_t *d_bad_all = nullptr,
                         bool small = false, bool dyn = false);
MatchPlan plan_match(int device, const HostImage &h, uint32_t maxlen);
int launch_expand(const DeviceImage &img, uint32_t k, const uint64_t *d_pos, const uint32_t *d_pid,
                  const uint64_t *d_count, uint64_t in_capacity, uint64_t *d_pos_all, uint32_t *d_pid_all,
                  uint64_t capacity, uint64_t *d_count_all, void *d_workspace, void *stream);
uint64_t expand_workspace_bytes();
}  // namespace pfac
