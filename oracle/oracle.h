/*
 * oracle.h — CPU ORACLE for the Genome-on-Diet hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load
 * or call this.  The product path (paper_2211_08157_b200/, include/god.h) never does, and shares
 * no code, header, table or helper with it.
 *
 * Plain, slow, single-threaded C.  Each function restates a definition of arXiv 2211.08157
 * (PAPER.md, "P:n" = line n) in the order the paper states it; where the paper is silent or
 * garbled the reading of SURVEY.md §8(c) (O1-O9) is taken and listed in DESIGN.md §2.
 *
 * Parity status: every function is pinned by tests/test_oracle_*.py against
 * something other than itself — worked examples (tests/golden/), closed forms, brute force on
 * tiny inputs and invariants.  The hash for k >= 8 is pinned only by bijectivity, the k <= 7
 * closed form of the same formula and an independent big-integer implementation (the paper
 * prints no known-answer hash values for k >= 8; "parity unpinned" against the paper there).
 */
#ifndef GOD_ORACLE_H
#define GOD_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define OR_N 4  /* code of an ambiguous base */

typedef struct {
    uint32_t p;          /* pattern length, 1..64 */
    uint32_t x;          /* weight = number of ones */
    uint8_t bit[64];     /* P[0..p-1] */
} or_pattern;

typedef struct { uint64_t hash; uint64_t pos; uint8_t strand; } or_mz;

typedef struct { uint32_t read_id; uint32_t ref_pos; uint32_t read_pos; uint32_t strand; } or_anchor;

/* one adjusted location (P:314 step (1)) and one voted location */
typedef struct { uint64_t hash; int64_t diag; uint32_t strand; uint32_t ref_pos, read_pos; } or_hit;
typedef struct {
    uint32_t read_id, strand;
    int64_t diag;                 /* Delta0 */
    uint32_t votes, rescued;
    uint32_t ref_lo, ref_hi, read_lo, read_hi;   /* member spans */
} or_vote;

typedef struct {
    uint64_t n_entries_all, n_distinct_all, m, tau;
    uint64_t kept_entries, dropped_entries, kept_distinct, dropped_distinct;
} or_index_stats;

typedef struct or_index or_index;

/* O1: A/a->0 C/c->1 G/g->2 T/t->3, anything else -> OR_N. */
int or_code(uint8_t b);
/* O2 (P:282, P:286(1)): parse a 0/1 pattern; returns 0 ok, -1 invalid (empty, >64, non-binary, all-zero). */
int or_parse_pattern(const char* text, or_pattern* out);
/* O3: PQ_s.  J = <i in [0,L): i >= s and P[(i-s) mod p] = 1>.
 * codes[j] = code(S[J[j]]), orig[j] = J[j].  Returns |J| (or -1 if s >= p). Either output may be NULL. */
int64_t or_sparsify(const uint8_t* seq, uint64_t L, const or_pattern* P, uint32_t s, uint8_t* codes, uint64_t* orig);
/* O5 (ref. 120): Thomas Wang's 64-bit integer mix with every step reduced mod 4^k. */
uint64_t or_hash(uint64_t x, int k);
/* O4+O6 (P:294, P:286(3)): double-strand (w,k)-minimizers of Sparsify(seq, P, s),
 * all ties kept, positions = pos_base + orig (start of the k-mer in original coordinates).
 * Writes up to `cap` records in position order; returns the total count. */
int64_t or_minimizers(const uint8_t* seq, uint64_t L, const or_pattern* P, uint32_t s, int k, int w,
                      uint64_t pos_base, or_mz* out, uint64_t cap);
/* Batch over CSR sequences; phases may be NULL (all 0).  out_offsets[n+1].  Returns total or -1 if cap too small. */
int64_t or_minimizers_batch(const uint8_t* seq, const uint64_t* offsets, uint32_t n, const uint8_t* phases,
                            const char* pattern, int k, int w, int global_pos, or_mz* out, uint64_t cap,
                            uint64_t* out_offsets);

/* O7: tau from the distinct-hash counts; m = floor(n*num/den), tau = a_{n-m-1} of the sorted counts. */
uint64_t or_cutoff_tau(const uint64_t* counts, uint64_t n, uint32_t num, uint32_t den, uint64_t* m_out);
/* O7 (P:286(3)): collect -> sort -> count -> cutoff -> table.
 * max_occ < 0: fraction rule (num/den of distinct hashes); max_occ >= 0: keep iff count <= max_occ. */
or_index* or_build_index(const uint8_t* ref, const uint64_t* offsets, uint32_t n, const char* pattern, int k, int w,
                         uint32_t frac_num, uint32_t frac_den, int64_t max_occ);
/* batch hash for exhaustive tests */
void or_hash_batch(const uint64_t* x, uint64_t n, int k, uint64_t* out);
void or_index_free(or_index* ix);
void or_index_stats_get(const or_index* ix, or_index_stats* st);
/* kept entries in (hash, pos) order */
uint64_t or_index_dump(const or_index* ix, uint64_t* hash, uint64_t* pos, uint8_t* strand, uint64_t cap);
/* occ(h): number of kept entries with hash h (0 if absent or dropped) — P:300 "occurrence frequency" */
uint32_t or_index_occ(const or_index* ix, uint64_t h);

/* O8: pattern alignment; returns a, writes score_s for s<p into scores (may be NULL). */
int or_select_phase(const or_index* ix, const uint8_t* read, uint64_t L, uint32_t t, uint64_t* scores);
/* O9: compressed seeding with phase a.  Anchors (read_id, ref_pos, read_pos, strand) sorted
 * canonically.  Returns total (writes up to cap). */
int64_t or_seed_read(const or_index* ix, const uint8_t* read, uint64_t L, uint32_t a, uint32_t read_id,
                     or_anchor* out, uint64_t cap);
/* Batch: mode 0 = SELECT (phases is output), 1 = GIVEN (phases is input).  anchor_offsets[n+1]. */
int64_t or_seed_reads_batch(const or_index* ix, const uint8_t* reads, const uint64_t* offsets, uint32_t n,
                            int mode, uint8_t* phases, uint32_t t, or_anchor* out, uint64_t cap,
                            uint64_t* anchor_offsets);

/* Location voting (readings V1-V6 in oracle.c / DESIGN.md §2).
 * or_vote_hits: steps (2)-(4) + rescue on a given hit list (sorted in place).  D = max distance,
 * V = vote threshold, max_pairs = cap on winners (0 = none).  Returns the number of voted
 * locations (writes up to cap). */
int64_t or_vote_hits(or_hit* hits, uint64_t n, uint64_t D, uint32_t V, uint32_t max_pairs, uint32_t read_id,
                     or_vote* out, uint64_t cap);
/* Step (1) from the read: minimizers of PQ_a matched against the index, then or_vote_hits with
 * D (0 = read length). */
int64_t or_vote_read(const or_index* ix, const uint8_t* read, uint64_t L, uint32_t a, uint32_t read_id,
                     uint32_t D, uint32_t V, uint32_t max_pairs, or_vote* out, uint64_t cap);
/* Batch over CSR reads with given phases (NULL = all 0); vote_offsets[n+1]. */
int64_t or_vote_reads_batch(const or_index* ix, const uint8_t* reads, const uint64_t* offsets, uint32_t n,
                            const uint8_t* phases, uint32_t D, uint32_t V, uint32_t max_pairs, or_vote* out,
                            uint64_t cap, uint64_t* vote_offsets);

/* Containment search (readings C1-C4 in oracle.c): per reference sequence
 * the number of mapped reads, their total length, and the accept decision.  Returns 0 (-1 on
 * invalid parameters). */
int or_contain(const uint8_t* refs, const uint64_t* ref_offsets, uint32_t n_refs, const char* pattern, int k, int w,
               uint32_t frac_num, uint32_t frac_den, int64_t max_occ, const uint8_t* reads,
               const uint64_t* read_offsets, uint32_t n_reads, uint32_t t, uint32_t D, uint32_t V,
               uint32_t max_pairs, uint64_t batch_bases, uint32_t min_reads, uint32_t cov_num, uint32_t cov_den,
               uint64_t* mapped_reads, uint64_t* mapped_bases, uint8_t* accepted);

/* Seed-comparison harness (readings S1-S4 in oracle.c).  algo 0 all k-mers, 1 minimizers,
 * 2 spaced seeds, 3 Genome-on-Diet (phase s).  Seeds = hashes, in extraction order. */
int64_t or_harness_seeds(const uint8_t* seq, uint64_t L, int algo, int k, int w, const char* pattern, uint32_t s,
                         uint64_t* out, uint64_t cap);
int64_t or_levenshtein(const uint8_t* a, uint64_t la, const uint8_t* b, uint64_t lb);
int64_t or_harness_pair(const uint8_t* a, const uint8_t* b, uint64_t L, int k, int w, const char* pattern,
                        uint64_t* out_m, uint64_t* out_t, uint32_t* god_phase);

#ifdef __cplusplus
}
#endif
#endif
