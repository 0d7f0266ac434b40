// Host automaton builder: SURVEY.md §8(a) steps 1-2 (Build, Device image).
//
//  1. Validate the patterns (readings R2 duplicate, R3 empty, R4 case, R5 non-ACGT, R13 length).
//  2. Insert them one by one into a trie, a new state per new character (PAPER.md:147-149,
//     §V-A; Table 1) -- with a fresh state for every new node (reading R1).
//  3. Renumber canonically: root 0, the state completing pattern p gets p, every other state
//     k+1, k+2, ... in breadth-first order, children in column order A,C,G,T (the "BFS-ordered
//     automaton with final states numbered as pattern IDs" of BASELINE.json's north star; BFS
//     rearrangement for locality is Nishimura et al.).
//  4. Derive the device image: the same automaton renumbered chain-major, its
//     unary runs stored as "chain rows" (up to 16 forced bases compared at once), the per-state
//     answer F, and a jump table J over all K-mers that performs the first K steps of every walk.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "../../include/pfac.h"
#include "pfac_internal.h"

namespace pfac {

// 2-bit code of a base, A,C,G,T -> 0,1,2,3 (case-insensitive); -1 otherwise.
static inline int base_code(uint8_t b) {
    switch (b | 0x20) {
        case 'a': return 0;
        case 'c': return 1;
        case 'g': return 2;
        case 't': return 3;
        default: return -1;
    }
}

int build_automaton(const uint8_t *bytes, const uint64_t *offsets, uint32_t k, pfac_automaton **out) {
    if (!out) return fail(PFAC_E_ARG, "pfac_build: out is null");
    *out = nullptr;
    if (k > 0 && (!bytes || !offsets)) return fail(PFAC_E_ARG, "pfac_build: null patterns with k > 0");
    if (k >= 0x7fffffffu) return fail(PFAC_E_TOO_MANY_STATES, "pfac_build: too many patterns");
    char msg[256];
    uint64_t total = 0;
    uint32_t maxlen = 0, minlen = 0xFFFFFFFFu;
    // ---- 1. validation, before any allocation that depends on the content
    for (uint32_t j = 0; j < k; ++j) {
        if (offsets[j + 1] < offsets[j]) {
            snprintf(msg, sizeof msg, "pfac_build: offsets decrease at pattern id %u", j + 1);
            return fail(PFAC_E_ARG, msg);
        }
        uint64_t len = offsets[j + 1] - offsets[j];
        if (len == 0) {
            snprintf(msg, sizeof msg, "pfac_build: pattern id %u is empty", j + 1);
            return fail(PFAC_E_EMPTY_PATTERN, msg);
        }
        if (len > PFAC_MAX_LEN) {
            snprintf(msg, sizeof msg, "pfac_build: pattern id %u has length %llu > PFAC_MAX_LEN=%u", j + 1,
                     (unsigned long long)len, PFAC_MAX_LEN);
            return fail(PFAC_E_TOO_LONG, msg);
        }
        for (uint64_t x = offsets[j]; x < offsets[j + 1]; ++x) {
            if (base_code(bytes[x]) < 0) {
                snprintf(msg, sizeof msg, "pfac_build: pattern id %u has non-ACGT byte 0x%02x at offset %llu",
                         j + 1, bytes[x], (unsigned long long)(x - offsets[j]));
                return fail(PFAC_E_NON_ACGT, msg);
            }
        }
        total += len;
        if (len > maxlen) maxlen = (uint32_t)len;
        if (len < minlen) minlen = (uint32_t)len;
    }
    // ---- 2. insertion-order trie (a new state per new character)
    std::vector<std::array<uint32_t, 4>> child;
    std::vector<uint32_t> fin;  // pattern id completed in this state, 0 = none
    try {
        child.reserve((size_t)std::min<uint64_t>(total + 1, 1ull << 28));
        fin.reserve(child.capacity());
    } catch (...) {
        return fail(PFAC_E_OOM, "pfac_build: host allocation failed");
    }
    child.push_back({0, 0, 0, 0});
    fin.push_back(0);
    for (uint32_t j = 0; j < k; ++j) {
        uint32_t s = 0;
        for (uint64_t x = offsets[j]; x < offsets[j + 1]; ++x) {
            int c = base_code(bytes[x]);
            if (child[s][c] == 0) {
                if (child.size() >= 0x7fffffffu)
                    return fail(PFAC_E_TOO_MANY_STATES, "pfac_build: automaton needs >= 2^31 states");
                child[s][c] = (uint32_t)child.size();
                child.push_back({0, 0, 0, 0});
                fin.push_back(0);
            }
            s = child[s][c];
        }
        if (fin[s] != 0) {
            snprintf(msg, sizeof msg, "pfac_build: pattern id %u duplicates pattern id %u", j + 1, fin[s]);
            return fail(PFAC_E_DUPLICATE, msg);
        }
        fin[s] = j + 1;
    }
    // ---- 3. canonical renumbering (BFS, finals = pattern ids)
    auto *a = new (std::nothrow) pfac_automaton();
    if (!a) return fail(PFAC_E_OOM, "pfac_build: host allocation failed");
    const uint32_t S = (uint32_t)child.size();
    a->k = k;
    a->S = S;
    a->maxlen = maxlen;
    a->minlen = k ? minlen : 0;
    try {
        a->table.assign((size_t)S * 4, 0);
        a->depth.assign(S, 0);
        a->F.assign(S, 0);
        a->prefix.assign(2 * ((size_t)k + 1), 0);
        std::vector<uint32_t> newid(S, 0);
        std::vector<uint32_t> fin_order;  // pattern ids in BFS (non-decreasing length) order
        fin_order.reserve(k);
        std::vector<uint32_t> order;  // insertion ids in BFS order
        order.reserve(S);
        order.push_back(0);
        uint32_t next = k + 1;
        for (size_t h = 0; h < order.size(); ++h) {
            uint32_t u = order[h];
            for (int c = 0; c < 4; ++c) {
                uint32_t v = child[u][c];
                if (!v) continue;
                uint32_t id = fin[v] ? fin[v] : next++;
                newid[v] = id;
                a->table[(size_t)newid[u] * 4 + c] = id;
                a->depth[id] = a->depth[newid[u]] + 1;
                a->F[id] = fin[v] ? fin[v] : a->F[newid[u]];
                if (fin[v]) {  // prefix chain: the longest pattern that is a proper prefix of this one
                    const uint32_t q = a->F[newid[u]];  // shallower, so its chain length is known
                    a->prefix[2 * (size_t)id] = q;
                    a->prefix[2 * (size_t)id + 1] = 1 + a->prefix[2 * (size_t)q + 1];
                    fin_order.push_back(id);
                }
                order.push_back(v);
            }
        }
        // Flattened prefix chains for the expand kernel: pattern p's chain, shortest first, at
        // prefix_flat[base(p) .. base(p) + len(p)); len(p) <= |p|, so the array is at most the total
        // pattern length.  Filled in BFS order so that a prefix's chain is ready before it is copied.
        a->prefix_dev.assign(4 * ((size_t)k + 1), 0);
        uint64_t flat = 0;
        for (uint32_t p = 1; p <= k; ++p) {
            const uint32_t len = a->prefix[2 * (size_t)p + 1];
            a->prefix_dev[4 * (size_t)p + 0] = len;
            a->prefix_dev[4 * (size_t)p + 1] = a->prefix[2 * (size_t)p];
            a->prefix_dev[4 * (size_t)p + 2] = (uint32_t)flat;
            a->prefix_dev[4 * (size_t)p + 3] = (uint32_t)(flat >> 32);
            flat += len;
        }
        a->prefix_flat.assign(flat ? flat : 1, 0);
        for (uint32_t p : fin_order) {
            const size_t b = a->prefix_dev[4 * (size_t)p + 2] | ((uint64_t)a->prefix_dev[4 * (size_t)p + 3] << 32);
            const uint32_t len = a->prefix_dev[4 * (size_t)p], q = a->prefix[2 * (size_t)p];
            if (q) {
                const size_t bq = a->prefix_dev[4 * (size_t)q + 2] | ((uint64_t)a->prefix_dev[4 * (size_t)q + 3] << 32);
                std::copy(a->prefix_flat.begin() + bq, a->prefix_flat.begin() + bq + (len - 1),
                          a->prefix_flat.begin() + b);
            }
            a->prefix_flat[b + len - 1] = p;
        }
    } catch (...) {
        delete a;
        return fail(PFAC_E_OOM, "pfac_build: host allocation failed");
    }
    try {
        derive_host_image(a);
    } catch (...) {
        delete a;
        return fail(PFAC_E_OOM, "pfac_build: host allocation failed (device image)");
    }
    *out = a;
    return PFAC_OK;
}

// Device image.  Layout documented on HostImage (pfac_internal.h) and in
// chain-major ids, branch/chain rows, F, and the K-mer jump table J.
template <typename C>
static void put(std::vector<uint8_t> &v, size_t i, uint32_t x) {
    reinterpret_cast<C *>(v.data())[i] = (C)x;
}

void derive_host_image(pfac_automaton *a) {
    HostImage &im = a->host_image;
    const uint32_t S = a->S;
    im.cell = (S < 32768u && a->k < 32768u) ? 2 : 4;
    const int K = im.cell == 2 ? kJumpK16 : kJumpK32;
    im.K = K;
    im.short_pat = 0;  // set below, once K2 is known
    const uint32_t *tab = a->table.data();
    auto nchild = [&](uint32_t u) {
        return (uint32_t)(tab[(size_t)u * 4] != 0) + (tab[(size_t)u * 4 + 1] != 0) + (tab[(size_t)u * 4 + 2] != 0) +
               (tab[(size_t)u * 4 + 3] != 0);
    };
    auto only_child = [&](uint32_t u, uint32_t &c) {
        for (c = 0; c < 4; ++c)
            if (tab[(size_t)u * 4 + c]) return tab[(size_t)u * 4 + c];
        return 0u;
    };
    // depth of every canonical state (BFS over the canonical table)
    std::vector<uint32_t> depth(S, 0);
    {
        std::vector<uint32_t> q;
        q.reserve(S);
        q.push_back(0);
        for (size_t h = 0; h < q.size(); ++h)
            for (int c = 0; c < 4; ++c)
                if (uint32_t v = tab[(size_t)q[h] * 4 + c]) {
                    depth[v] = depth[q[h]] + 1;
                    q.push_back(v);
                }
    }
    // uint32 images (large automata): a K1-mer filter bitmap (K1 = 10, 128 KiB, in shared memory)
    // plus a second-level jump table J2 over K2-mers, K2 in [10, 11] (J2 <= 16 MiB, L2-resident next
    // to the out[] stream): the smallest K2 whose depth-K2 states cover <= 3% of all K2-mers.
    im.K2 = 0;
    if (im.cell == 4 || kFilterSmall) {
        std::vector<uint64_t> per_depth(a->maxlen + 2, 0);
        for (uint32_t u = 0; u < S; ++u) per_depth[depth[u]]++;
        im.K2 = kK2Max;
        for (int k2 = kK2Min; k2 <= kK2Max; ++k2) {
            const uint64_t D = (uint32_t)k2 < per_depth.size() ? per_depth[k2] : 0;
            if (D * 100 <= 3 * (1ull << (2 * k2))) {
                im.K2 = k2;
                break;
            }
        }
    }
    im.short_pat = a->k > 0 && a->minlen < (uint32_t)(im.K2 ? im.K2 : K);
    // Deep-first, chain-major numbering.  Part A: the states at depth >= K, breadth-first over chain
    // heads starting from the depth-K states (the states J hands to the kernel), each head followed
    // by its unary run.  Part B: the states at depth < K, the same way from the root, with runs cut
    // at depth K-1.  Runs never cross the boundary, so every chain row spans consecutive ids.
    const uint32_t Kd = (uint32_t)(im.K2 ? im.K2 : K);  // walks resume at depth K2 when J2 exists
    auto unary_next = [&](uint32_t u, uint32_t &v) {  // the only child of u, if u is unary and in u's part
        uint32_t c;
        if (nchild(u) != 1) return false;
        v = only_child(u, c);
        return (depth[u] + 1 >= Kd) == (depth[u] >= Kd);
    };
    // The unary run from u: its next L <= maxL forced bases (base i at bits 2i), whether a final state
    // lies strictly inside (u, u+L), and the state the span ends in.
    struct Chain {
        uint64_t bits = 0;
        uint32_t L = 0, end = 0;
        bool inner_final = false;
    };
    auto chain_of = [&](uint32_t u, uint32_t maxL) {
        Chain ch;
        uint32_t v = u, c, w;
        while (ch.L < maxL && unary_next(v, w)) {
            if (ch.L > 0 && v >= 1 && v <= a->k) ch.inner_final = true;
            only_child(v, c);
            v = w;
            ch.bits |= (uint64_t)c << (2 * ch.L);
            ++ch.L;
        }
        ch.end = v;
        return ch;
    };
    // uint32 rows: a walk that consumes a span whose end state has no transitions stops there, so
    // the row can carry that answer (F(end) + 1 in 24 bits; 0 = the end state continues)
    auto end_answer = [&](const Chain &ch) -> uint32_t {
        return kEndDead && nchild(ch.end) == 0 && a->F[ch.end] < kEndMask ? a->F[ch.end] + 1 : 0u;
    };
    std::vector<uint32_t> dev(S, 0);
    uint32_t id = 1;
    auto number_from = [&](std::vector<uint32_t> heads, bool deep) {
        for (size_t h = 0; h < heads.size(); ++h) {
            uint32_t u = heads[h];
            while (true) {
                dev[u] = id++;
                uint32_t v;
                if (unary_next(u, v)) {
                    u = v;
                    continue;
                }
                for (int cc = 0; cc < 4; ++cc)
                    if (uint32_t w = tab[(size_t)u * 4 + cc])
                        if ((depth[w] >= Kd) == deep) heads.push_back(w);
                break;
            }
        }
    };
    {
        std::vector<uint32_t> q, atK;
        q.push_back(0);
        for (size_t h = 0; h < q.size(); ++h) {
            const uint32_t u = q[h];
            if (depth[u] == Kd) {
                atK.push_back(u);
                continue;
            }
            for (int c = 0; c < 4; ++c)
                if (uint32_t v = tab[(size_t)u * 4 + c]) q.push_back(v);
        }
        number_from(atK, true);
        number_from({0u}, false);
    }
    im.S = S;
    im.root = dev[0];
    im.rows = ((S + 1) + 7) & ~7u;
    const uint32_t cell = im.cell;
    const uint32_t chain_flag = cell == 2 ? 0x8000u : 0x80000000u;
    im.T.assign((size_t)im.rows * kRowCells * cell, 0);
    im.F.assign((size_t)im.rows * cell, 0);
    auto putc = [&](std::vector<uint8_t> &v, size_t i, uint32_t x) {
        if (cell == 2) put<uint16_t>(v, i, x);
        else put<uint32_t>(v, i, x);
    };
    for (uint32_t u = 0; u < S; ++u) {
        const uint32_t d = dev[u];
        putc(im.F, d, a->F[u]);
        if (kMergedF) putc(im.T, (size_t)d * kRowCells + 4, a->F[u]);  // ablation: F inside the row
        uint32_t v0;
        if (unary_next(u, v0)) {  // chain row: the next L forced bases within u's part
            const Chain ch = chain_of(u, cell == 2 ? (uint32_t)kChainMax : (uint32_t)kChainMax32);
            const uint32_t nofin = ch.inner_final ? 0u : (cell == 2 ? 0x4000u : 0x40000000u);
            if (cell == 2) {
                // FSTEP: every state inside the span answers F(u) + its offset (nested prefix families
                // with consecutive ids), so a walk that ends inside needs no F lookup
                bool fstep = kFStep && ch.inner_final;  // (NOFIN rows answer F(u) anyway)
                for (uint32_t j = 1, v = u, w2; fstep && j < ch.L; ++j) {
                    unary_next(v, w2);
                    v = w2;
                    fstep = a->F[v] == a->F[u] + j;
                }
                putc(im.T, (size_t)d * kRowCells + 0, chain_flag | nofin | (fstep ? kFStep16 : 0u) | ch.L);
                putc(im.T, (size_t)d * kRowCells + 1, (uint32_t)ch.bits & 0xFFFFu);
                putc(im.T, (size_t)d * kRowCells + 2, (uint32_t)ch.bits >> 16);
                putc(im.T, (size_t)d * kRowCells + 3, a->F[u]);
            } else {
                putc(im.T, (size_t)d * kRowCells + 0, chain_flag | nofin | (end_answer(ch) << kEndShift) | ch.L);
                putc(im.T, (size_t)d * kRowCells + 1, (uint32_t)ch.bits);
                putc(im.T, (size_t)d * kRowCells + 2, a->F[u]);
                putc(im.T, (size_t)d * kRowCells + 3, (uint32_t)(ch.bits >> 32));
            }
        } else {
            for (int c = 0; c < 4; ++c)
                if (uint32_t v = tab[(size_t)u * 4 + c]) putc(im.T, (size_t)d * kRowCells + c, dev[v]);
        }
    }
    const uint32_t nk = 1u << (2 * K);
    const uint32_t alive = cell == 2 ? 0x8000u : 0x80000000u;
    im.J.assign((size_t)nk * cell, 0);
    for (uint32_t x = 0; x < nk; ++x) {
        uint32_t s = 0;
        int d = 0;
        for (; d < K; ++d) {
            uint32_t t = tab[(size_t)s * 4 + ((x >> (2 * d)) & 3)];
            if (!t) break;
            s = t;
        }
        putc(im.J, x, (d == K) ? (alive | dev[s]) : a->F[s]);
    }
    if (im.K2) {
        const uint32_t K2 = (uint32_t)im.K2;
        const uint64_t n2 = 1ull << (2 * K2);
        im.J2.assign(n2, 0);
        for (uint64_t x = 0; x < n2; ++x) {
            uint32_t s2 = 0, d = 0;
            for (; d < K2; ++d) {
                const uint32_t t = tab[(size_t)s2 * 4 + ((x >> (2 * d)) & 3)];
                if (!t) break;
                s2 = t;
            }
            im.J2[x] = (d == K2) ? (0x80000000u | dev[s2]) : a->F[s2];
        }
        // uint32 images: a live walk's first row is its depth-K2 state's, and chain-major numbering
        // scatters those rows over T (each head is followed by its run), so most are DRAM misses.
        // Chain-head rows are copied into a compact array HR that sits next to J2 inside the
        // L2-persisting window; cell 3 (unused in chain rows) holds the head's device id, and the
        // J2 entry becomes ALIVE | HRF | index.  Branch heads keep pointing into T.
        im.HR.clear();
        im.hr_nb = 0;
        std::vector<uint32_t> canon(cell == 4 ? (size_t)S + 1 : 0, 0);  // device id -> canonical id
        for (uint32_t u = 0; cell == 4 && u < S; ++u) canon[dev[u]] = u;
        if (cell == 4 && im.S < (1u << 30)) {
            uint64_t heads = 0;
            for (uint64_t x = 0; x < n2; ++x)
                if (im.J2[x] & 0x80000000u) ++heads;
            if (heads * 16 <= (8ull << 20)) {  // at most 8 MiB of copies
                for (uint64_t x = 0; x < n2; ++x) {
                    if (!(im.J2[x] & 0x80000000u)) continue;
                    const uint32_t s = im.J2[x] & 0x7FFFFFFFu;
                    uint32_t row[4];
                    memcpy(row, im.T.data() + (size_t)s * kRowCells * 4, 16);
                    if (!(row[0] & 0x80000000u)) continue;  // a branch row: stays in T
                    // the copy spans at most 16 bases (cell 3 holds the head's device id)
                    const Chain ch = chain_of(canon[s], (uint32_t)kChainMax);
                    row[0] = 0x80000000u | (ch.inner_final ? 0u : 0x40000000u) | (end_answer(ch) << kEndShift) | ch.L;
                    row[1] = (uint32_t)ch.bits;
                    row[3] = s;
                    const uint32_t h = (uint32_t)(im.HR.size() / 4);
                    im.HR.insert(im.HR.end(), row, row + 4);
                    // NB form: a NOFIN chain of L >= 4 forced bases whose head answers 0 (F = 0, so
                    // every state strictly inside the span answers 0 too).  The entry carries the
                    // first 4 forced bases; a walk whose next 4 bases differ (or that has fewer than
                    // 4 left) ends inside the span and answers 0 without loading the row (all but
                    // ~1/256 of the live walks on random text).
                    const bool nb = (row[0] & 0x40000000u) && (row[0] & kChainLenMask32) >= kHRBases && row[2] == 0 &&
                                    h < (1u << kHRIndexBitsNB);
                    im.hr_nb += nb ? 1u : 0u;
                    im.J2[x] = nb ? kJ2Alive | kJ2HR | kJ2NB | ((row[1] & 0xFFu) << kHRIndexBitsNB) | h
                                  : kJ2Alive | kJ2HR | h;
                }
            }
        }
        // FB[x] = 1 iff the K1-mer x starts a walk that survives K1 bases or completes a pattern on the
        // way: every other position's answer is 0 without touching J2.
        const uint32_t K1 = (uint32_t)kFilterK;
        const uint64_t n1 = 1ull << (2 * K1);
        im.FB.assign(n1 / 32, 0);
        for (uint64_t x = 0; x < n1; ++x) {
            uint32_t s1 = 0, d = 0;
            for (; d < K1; ++d) {
                const uint32_t t = tab[(size_t)s1 * 4 + ((x >> (2 * d)) & 3)];
                if (!t) break;
                s1 = t;
            }
            if (d == K1 || a->F[s1] != 0) im.FB[x >> 5] |= 1u << (x & 31);
        }
    }
}

// Walk statistics of a host text sample (pfac_text_walk_stats): the PFAC walk from
// positions 0, stride, 2*stride, ... over the canonical table, counting transitions; a byte outside
// ACGTacgt has no transition (reading R5).  Host code only.
int text_walk_stats(const pfac_automaton *a, const uint8_t *h_text, uint64_t n, uint64_t stride, uint32_t deep,
                    double *deep_frac, double *mean_steps) {
    if (!a || (!h_text && n) || !stride || !deep_frac || !mean_steps)
        return fail(PFAC_E_ARG, "pfac_text_walk_stats: null argument or zero stride");
    uint64_t walks = 0, deep_walks = 0, steps = 0;
    for (uint64_t i = 0; i < n; i += stride) {
        uint32_t s = 0, d = 0;
        for (uint64_t j = i; j < n; ++j) {
            const int c = base_code(h_text[j]);
            if (c < 0) break;
            const uint32_t t = a->table[(size_t)s * 4 + c];
            if (!t) break;
            s = t;
            ++d;
        }
        ++walks;
        steps += d;
        deep_walks += d >= deep;
    }
    *deep_frac = walks ? (double)deep_walks / (double)walks : 0.0;
    *mean_steps = walks ? (double)steps / (double)walks : 0.0;
    return PFAC_OK;
}

}  // namespace pfac
