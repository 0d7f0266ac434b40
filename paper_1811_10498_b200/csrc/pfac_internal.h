// Internal declarations shared by the host builder (builder.cpp), the C-ABI (api.cu) and the
// kernels (kernels.cu).  Not part of the public ABI (see include/pfac.h).
#pragma once

#include <array>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

namespace pfac {

// Device numbering / jump table constants.
constexpr uint32_t kAlive = 0x80000000u;  // J entry flag: walk is still alive at depth K
constexpr int kJumpK = 7;                  // J has 4^K entries (64 KiB of uint32 in smem)

// Host-side device image: everything the match kernel reads, before upload.
struct HostImage {
    int K = kJumpK;
    uint32_t S = 0;          // device states, ids 1..S (row 0 is a dummy all-zero row)
    uint32_t deep = 0;       // ids 1..deep are the states at depth >= K, breadth-first order
    uint32_t root = 0;       // device id of the root (among the shallow ids deep+1..S)
    std::vector<uint32_t> J; // 4^K: kAlive|id of the depth-K state, or the answer (pattern id/0)
    std::vector<uint32_t> T; // (S+1)*4: child device id per code A,C,G,T; 0 = none
    std::vector<uint32_t> F; // S+1: id of the deepest final state on the root path (0 = none)
};

// Launch plan of the match kernel for one automaton on one device (match.cu).
struct MatchPlan {
    uint32_t cell = 4;         // bytes per J/T/F cell: 2 (uint16, S < 32768 and k < 32768) or 4
    bool all_smem = false;     // every T row / F entry fits in shared memory (no window check)
    uint32_t window = 0;       // device ids [0, window) staged in shared memory
    uint32_t slice_words = 0;  // packed words per warp slice (512 bases + halo)
    size_t smem = 0;           // dynamic shared memory per CTA
    int sms = 0;
};

// A device image resident on one GPU.
struct DeviceImage {
    int device = -1;
    int K = kJumpK;
    uint32_t S = 0, deep = 0, root = 0;
    uint32_t maxlen = 0;
    MatchPlan plan;
    void *d_J = nullptr, *d_T = nullptr, *d_F = nullptr;  // cells of plan.cell bytes
};

}  // namespace pfac

struct pfac_automaton {
    uint32_t k = 0;       // patterns
    uint32_t S = 0;       // canonical states (incl. root)
    uint32_t maxlen = 0;
    std::vector<uint32_t> table;  // canonical S*4, columns A,C,G,T
    std::vector<uint32_t> depth;  // canonical depth of each state
    std::vector<uint32_t> F;      // canonical: deepest final on the root path (pattern id) or 0
    pfac::HostImage host_image;   // derived once at build
    std::mutex mu;                // guards images
    std::vector<pfac::DeviceImage *> images;
};

namespace pfac {
// Thread-local error message plumbing (api.cu).
int fail(int code, const std::string &msg);

// builder.cpp
int build_automaton(const uint8_t *bytes, const uint64_t *offsets, uint32_t k, pfac_automaton **out);
void derive_host_image(pfac_automaton *a, int K);

// kernels.cu launchers (all asynchronous on `stream`); return cudaError_t as int.
int launch_pack(const uint8_t *d_text, uint64_t n, uint32_t *d_packed, uint64_t nwords_padded,
                uint64_t *d_first_bad, void *stream);
int launch_match(const DeviceImage &img, const uint32_t *d_packed, uint64_t n_own, uint64_t n_avail,
                 int32_t *d_out, void *stream);
int launch_compact(const int32_t *d_out, uint64_t n, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                   uint64_t capacity, uint64_t *d_count, uint32_t k, uint64_t *d_hist, void *d_workspace,
                   void *stream);
uint64_t compact_workspace_bytes(uint64_t n);
MatchPlan plan_match(int device, int K, uint32_t maxlen, uint32_t S, uint32_t k);
}  // namespace pfac
