/*
 * pfac_oracle.c -- O2, the bit-exactness reference for the PFAC hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library.  It shares no code, header, table or constant
 * generator with paper_1811_10498_b200/ (the product), and the product never calls it.
 *
 * What it computes (a plain, slow, single-threaded transcription of the paper):
 *
 *  1. Transition table, PAPER.md:120 (§V-A) and Table 1: a 4 x N array whose
 *     columns are the letters A, T, C, G in the paper's header order and whose
 *     cells hold the pair (next state, matched pattern id); "0,0" is an empty cell.
 *  2. Loading: "Input patterns are loaded into this transition table one by
 *     one. Next state ... is decided by current letter of the pattern and the previous state ...
 *     When the program find new state (new character) then it adds a new state."  The cell that
 *     completes pattern number p (1-based, Table 1 cell "6,1") gets matched id p.  A brand-new
 *     state number is allocated for every new trie node (reading R1: the printed
 *     Table 1 reuses states 6 and 11, which would produce false matches).
 *  3. Matching, PAPER.md:91-93 (§IV) and :204 (§V-B): every text position i gets its own walk
 *     ("each character of the input has it's own thread"); the walk starts in state 0, follows
 *     the goto function only (no failure links), stops at the first missing transition, and the
 *     result is the id of the last pattern completed on the way -- "PFAC can detect only the
 *     longest patterns".  A byte outside ACGTacgt has no transition (reading R5,
 *     the barrier); a walk also stops at the end of the text (reading R6).
 *
 * The result out[i] therefore equals the plain definition "id of the longest pattern p with
 * text[i .. i+|p|) = p, else 0"; tests/test_oracle_pins.py checks that against brute force.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_E_EMPTY_PATTERN (-2)
#define ORACLE_E_NON_ACGT (-3)
#define ORACLE_E_DUPLICATE (-4)
#define ORACLE_E_OOM (-9)

/* One cell of the 4 x N table (Table 1): (next state, matched pattern id). */
typedef struct {
    uint32_t next;
    uint32_t pid;
} cell_t;

typedef struct {
    cell_t *rows;      /* rows[4*s + col], col order A,T,C,G */
    uint32_t nstates;  /* states 0 .. nstates-1, state 0 = start */
    uint32_t cap;
    uint32_t npatterns;
    uint32_t maxlen;
} oracle_trie;

/* Column of a letter in the paper's table: A,T,C,G -> 0,1,2,3; anything else -> -1. */
static int column_of(uint8_t ch) {
    switch (ch) {
        case 'A': case 'a': return 0;
        case 'T': case 't': return 1;
        case 'C': case 'c': return 2;
        case 'G': case 'g': return 3;
        default: return -1;
    }
}

static int grow(oracle_trie *t) {
    uint32_t ncap = t->cap ? t->cap * 2 : 64;
    cell_t *r = (cell_t *)realloc(t->rows, (size_t)ncap * 4 * sizeof(cell_t));
    if (!r) return ORACLE_E_OOM;
    memset(r + (size_t)t->cap * 4, 0, (size_t)(ncap - t->cap) * 4 * sizeof(cell_t));
    t->rows = r;
    t->cap = ncap;
    return ORACLE_OK;
}

void oracle_free(oracle_trie *t) {
    if (!t) return;
    free(t->rows);
    free(t);
}

/* Build the table by loading patterns one by one.
 * Pattern j (id j+1) is bytes[offsets[j] .. offsets[j+1]).
 * On error returns a negative code and sets *bad_id (1-based id of the offending pattern;
 * for a duplicate, *other_id is the earlier pattern it repeats). */
int oracle_build(const uint8_t *bytes, const uint64_t *offsets, uint32_t k, oracle_trie **out,
                 uint32_t *bad_id, uint32_t *other_id) {
    oracle_trie *t = (oracle_trie *)calloc(1, sizeof(oracle_trie));
    if (!t) return ORACLE_E_OOM;
    if (grow(t)) { oracle_free(t); return ORACLE_E_OOM; }
    t->nstates = 1; /* state 0 */
    t->npatterns = k;
    for (uint32_t j = 0; j < k; ++j) {
        uint64_t a = offsets[j], b = offsets[j + 1];
        uint32_t pid = j + 1;
        if (b <= a) { *bad_id = pid; oracle_free(t); return ORACLE_E_EMPTY_PATTERN; }
        if (b - a > t->maxlen) t->maxlen = (uint32_t)(b - a);
        uint32_t s = 0;
        for (uint64_t x = a; x < b; ++x) {
            int col = column_of(bytes[x]);
            if (col < 0) { *bad_id = pid; oracle_free(t); return ORACLE_E_NON_ACGT; }
            cell_t *c = &t->rows[(size_t)s * 4 + col];
            if (c->next == 0) {                 /* new character -> add a new state */
                if (t->nstates == t->cap && grow(t)) { oracle_free(t); return ORACLE_E_OOM; }
                c = &t->rows[(size_t)s * 4 + col];
                c->next = t->nstates++;
            }
            if (x + 1 == b) {                   /* last letter: record the matched pattern id */
                if (c->pid != 0) {
                    *bad_id = pid; *other_id = c->pid; oracle_free(t); return ORACLE_E_DUPLICATE;
                }
                c->pid = pid;
            }
            s = c->next;
        }
    }
    *out = t;
    return ORACLE_OK;
}

uint32_t oracle_num_states(const oracle_trie *t) { return t->nstates; }
uint32_t oracle_max_len(const oracle_trie *t) { return t->maxlen; }

/* Cell (state s, column col in A,T,C,G order). */
void oracle_cell(const oracle_trie *t, uint32_t s, uint32_t col, uint32_t *next, uint32_t *pid) {
    cell_t c = t->rows[(size_t)s * 4 + col];
    *next = c.next;
    *pid = c.pid;
}

/* The walk of one position. */
static int32_t walk(const oracle_trie *t, const uint8_t *text, uint64_t n, uint64_t i) {
    uint32_t s = 0;
    int32_t last = 0;
    for (uint64_t j = i; j < n; ++j) {
        int col = column_of(text[j]);
        if (col < 0) break;                     /* no transition on a non-ACGT byte */
        cell_t c = t->rows[(size_t)s * 4 + col];
        if (c.next == 0) break;                 /* first missing transition ends the walk */
        if (c.pid != 0) last = (int32_t)c.pid;  /* a pattern completes on this edge */
        s = c.next;
    }
    return last;
}

/* out[i - a] for every position i in [a, b); walks may read text up to n (exclusive). */
void oracle_match(const oracle_trie *t, const uint8_t *text, uint64_t n, uint64_t a, uint64_t b,
                  int32_t *out) {
    for (uint64_t i = a; i < b; ++i) out[i - a] = walk(t, text, n, i);
}

/* The match list [(i, out[i]) : out[i] != 0] for i in [a, b), ascending i.  Writes at most cap
 * entries; returns the total count (which may exceed cap). */
uint64_t oracle_match_list(const oracle_trie *t, const uint8_t *text, uint64_t n, uint64_t a,
                           uint64_t b, uint64_t *pos, uint32_t *pid, uint64_t cap) {
    uint64_t m = 0;
    for (uint64_t i = a; i < b; ++i) {
        int32_t r = walk(t, text, n, i);
        if (r != 0) {
            if (m < cap) { pos[m] = i; pid[m] = (uint32_t)r; }
            ++m;
        }
    }
    return m;
}

/* Every occurrence: the walk of position i passes the final state of
 * every pattern that occurs at i, since each such pattern's bases are the first bases of the walk
 * (PAPER.md:91-93); emitting each completed id as the walk goes gives the occurrences at i in
 * ascending length.  For i in [a, b), ascending i; writes at most cap entries, returns the total. */
uint64_t oracle_match_all(const oracle_trie *t, const uint8_t *text, uint64_t n, uint64_t a,
                          uint64_t b, uint64_t *pos, uint32_t *pid, uint64_t cap) {
    uint64_t m = 0;
    for (uint64_t i = a; i < b; ++i) {
        uint32_t s = 0;
        for (uint64_t j = i; j < n; ++j) {
            int col = column_of(text[j]);
            if (col < 0) break;
            cell_t c = t->rows[(size_t)s * 4 + col];
            if (c.next == 0) break;
            if (c.pid != 0) {
                if (m < cap) { pos[m] = i; pid[m] = c.pid; }
                ++m;
            }
            s = c.next;
        }
    }
    return m;
}
