/*
 * god.h — C ABI of the B200-native Genome-on-Diet hot path (libgod.so).
 *
 * Implements the data-parallel hot path of arXiv 2211.08157 ("Genome-on-Diet", PAPER.md; P:n =
 * line n): (1) pattern sparsification, (2) double-strand (w,k)-minimizer extraction, (3) seed
 * index build with an occurrence cutoff, (4) pattern alignment (phase selection) and compressed
 * seeding into anchors.  Every step runs in hand-written CUDA kernels for sm_100a; there is no
 * CPU fallback.  Readings of the paper (tie rule, position convention, cutoff quantile, phase
 * rules) are DESIGN.md §2 (= SURVEY.md §8(c) O1-O9).
 *
 * CONVENTIONS (all entry points)
 *  - Pointers may be DEVICE or HOST memory: each pointer is classified with
 *    cudaPointerGetAttributes; host inputs are staged to the device inside the call and host
 *    outputs are copied back before it returns (such calls synchronize `stream`).  Device-only
 *    calls are asynchronous on `stream` except where a host-visible size is returned
 *    (`*_needed` out-params, god_build_index, god_index_get_stats): those synchronize `stream`.
 *  - Sequences are CSR: `seq` holds the concatenated ASCII bases of n sequences, `offsets[n+1]`
 *    (u64) delimits them.  Bytes A/C/G/T (either case) are bases; every other byte is an
 *    ambiguous base N (reading O1).
 *  - Inputs are caller-owned and read-only; outputs are caller-allocated with an explicit
 *    capacity.  If the capacity is too small the call returns GOD_ETRUNC, writes the required
 *    size to `*needed` (host u64) and writes nothing else.
 *  - Index memory is library-owned (stream-ordered allocations) and released by god_index_free.
 *    An index is immutable after build; concurrent god_seed_reads calls on one index are safe.
 *  - Errors: GOD_EINVAL is detected on the host before any device work; god_last_error() returns
 *    a thread-local message for the last failing call.  The library never exits or throws.
 *  - Limits: pattern length 1..64 with at least one '1'; 1 <= k <= 28; 1 <= w <= 255;
 *    total reference length < 2^32 (positions are u32); each read < 2^32 bases; phases < p.
 */
#ifndef GOD_H
#define GOD_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GOD_API __attribute__((visibility("default")))
#else
#define GOD_API
#endif

typedef int32_t god_status;
#define GOD_OK 0
#define GOD_EINVAL 1  /* contract violation, detected on the host before any launch */
#define GOD_ENOMEM 2  /* device allocation failed */
#define GOD_ECUDA 3   /* CUDA runtime / launch error */
#define GOD_ETRUNC 4  /* output capacity too small; required size in *needed */

typedef void* god_stream;   /* a cudaStream_t (0 = legacy default stream) */

/* The user's diet pattern P ("a binary pattern sequence P[0..p-1] ... weight x"),
 * the k-mer length k and minimizer window w ("(w,k)-minimizer"). */
typedef struct {
    const char* pattern;   /* NUL-terminated '0'/'1' string, 1 <= p <= 64, >= one '1' */
    int32_t k;             /* 1..28 */
    int32_t w;             /* 1..255 */
} god_params;

/* Occurrence cutoff ("we discard the most frequently (>= a user-defined threshold)
 * occurring minimizers").  mode 0: drop the top frac_num/frac_den of distinct hashes by count
 * (reading O7: m = floor(n*num/den), tau = a_{n-m-1} of the ascending counts, keep count <= tau;
 * BASELINE "top 0.02%" = 1/5000).  mode 1: absolute, keep iff count <= max_occ. */
typedef struct {
    uint32_t mode;
    uint32_t frac_num, frac_den;
    uint32_t max_occ;
} god_cutoff;

typedef struct {
    uint64_t n_entries_all;    /* |E|: minimizer occurrences collected from the reference */
    uint64_t n_distinct_all;   /* n: distinct hashes */
    uint64_t m;                /* floor(n * frac) (0 in mode 1) */
    uint64_t tau;              /* keep iff count <= tau */
    uint64_t kept_entries, dropped_entries, kept_distinct, dropped_distinct;
    uint32_t k, w, p, x;       /* parameters the index was built with */
    uint32_t dir_bits;         /* mode 0: B, directory = top B bits of the 2k-bit hash; mode 1: floor(log2 slots) */
    uint32_t dir_mode;         /* 0: top-bit directory; 1: data-sized slot map over the top 12 hash bits */
} god_index_stats;

/* One seed match ("finds exact matches of minimizers in the reference genome by querying
 * the seed index"; P:312 anchors): reference start position (global, original coordinates),
 * read start position (original read coordinates, read as supplied), read index, and
 * strand = reference-minimizer strand XOR read-minimizer strand. */
typedef struct {
    uint32_t ref_pos;
    uint32_t read_pos;
    uint32_t read_id;
    uint32_t strand;
} god_anchor;

typedef enum { GOD_PHASE_SELECT = 0, GOD_PHASE_GIVEN = 1 } god_phase_mode;

typedef struct god_index god_index;

GOD_API const char* god_last_error(void);
GOD_API const char* god_version(void);

/* ---- stage 1: sparsification (P:282 PR/PQ; P:286 steps (1)-(2); P:300 PQ_s) ----
 * For sequence i with phase s_i (phases == NULL: all 0, the reference convention of P:286) keep
 * original base j iff j >= s_i and P[(j - s_i) mod p] = 1, in order (reading O3).
 * Output per sequence, starting on a fresh word: `packed` 2 bits per kept base, 32 bases per u64
 * word, LSB-first (kept base q -> word q>>5, bits 2(q&31)..+1; A0 C1 G2 T3; N stored as 0);
 * `nmask` parallel to `packed` (same word index), bit (q&31) set iff kept base q is N.  Pad bits 0.
 * out_offsets[n+1]: word offsets per sequence; counts[n]: kept bases per sequence.
 * Needs packed_cap_words >= out_offsets[n]; else GOD_ETRUNC with *packed_needed.  Synchronizes. */
GOD_API god_status god_sparsify(const god_params* prm, const uint8_t* seq, const uint64_t* offsets, uint32_t n_seqs,
                                const uint8_t* phases, uint64_t* packed, uint64_t* nmask, uint64_t* out_offsets,
                                uint64_t* counts, uint64_t packed_cap_words, uint64_t* packed_needed,
                                god_stream stream);

/* ---- stage 2: (w,k)-minimizers (P:286 (3); P:370 N handling) ----
 * Canonical k-mers over each N-free run of the sparsified sequence, Thomas Wang's hash masked to
 * 2k bits (ref. 120), every position attaining a window minimum (all ties; windows of w
 * consecutive k-mers, or the whole run if shorter; palindromes never selected).
 * Records per sequence in position order: hash[], pos[] (u32 start in original coordinates;
 * + the sequence's global offset if global_pos != 0), strand[] (1 = reverse is canonical).
 * out_offsets[n+1].  cap = record capacity; GOD_ETRUNC + *needed if too small.  Synchronizes. */
GOD_API god_status god_minimizers(const god_params* prm, const uint8_t* seq, const uint64_t* offsets, uint32_t n_seqs,
                                  const uint8_t* phases, int32_t global_pos, uint64_t* hash, uint32_t* pos,
                                  uint8_t* strand, uint64_t* out_offsets, uint64_t cap, uint64_t* needed,
                                  god_stream stream);

/* ---- stage 3: the seed index (P:286 (3), P:294 collect-then-sort, P:302 cutoff) ----
 * Minimizers of every reference sequence (phase 0, global positions), sorted by (hash, pos),
 * counted per distinct hash, filtered by the cutoff, stored as a bucketed table: a directory over
 * the top B bits of the hash and, per kept entry, the remaining hash bits + strand and the
 * position.  *out receives a library-owned handle.  Synchronizes `stream`.
 * A host reference of >= 64 MB (pinned memory for the overlap to be real) is streamed: it goes up in
 * chunks on a copy stream while stage 1+2 runs on the parts that are in; the result is the same. */
GOD_API god_status god_build_index(const god_params* prm, const uint8_t* ref, const uint64_t* ref_offsets,
                                   uint32_t n_refs, const god_cutoff* cutoff, god_index** out, god_stream stream);
GOD_API god_status god_index_get_stats(const god_index* idx, god_index_stats* out_host);
/* Kept entries in (hash, pos) order.  cap = entry capacity (>= kept_entries else GOD_ETRUNC). */
GOD_API god_status god_index_dump(const god_index* idx, uint64_t* hash, uint32_t* pos, uint8_t* strand, uint64_t cap,
                                  uint64_t* needed, god_stream stream);
/* occ(h) for n query hashes ("their sum of occurrence frequencies"): kept count, 0 if absent/dropped. */
GOD_API god_status god_index_count(const god_index* idx, const uint64_t* hashes, uint64_t n, uint32_t* counts,
                                   god_stream stream);
GOD_API void god_index_free(god_index* idx);

/* ---- stage 4: pattern alignment + compressed seeding ----
 * mode GOD_PHASE_SELECT: for each read and s = 0..p-1 take the minimizers of PQ_s, c = min(t,
 * min_s |M_s|), score_s = sum of occ over the first c, a = argmax (smallest s on ties; p = 1 ->
 * 0); phases[n] (u8) receives a.  mode GOD_PHASE_GIVEN: phases[n] is an input (each < p).
 * Then every minimizer of PQ_a is looked up and every kept entry with the same hash yields one
 * anchor (no deduplication).  Anchors of read r occupy [anchor_offsets[r], anchor_offsets[r+1]),
 * ordered by read minimizer position then reference position.  t >= 1 (default 16).
 * cap = anchor capacity; GOD_ETRUNC + *needed (phases are still written).  Synchronizes. */
GOD_API god_status god_seed_reads(const god_index* idx, const uint8_t* reads, const uint64_t* read_offsets,
                                  uint32_t n_reads, god_phase_mode mode, uint8_t* phases, uint32_t t,
                                  god_anchor* anchors, uint64_t* anchor_offsets, uint64_t cap, uint64_t* needed,
                                  god_stream stream);

/* The same seeding with 8-byte anchors for transfers: the read id is implied by anchor_offsets
 * (anchors of read r occupy [anchor_offsets[r], anchor_offsets[r+1])), and the strand is bit 31 of
 * read_pos_strand (read positions must be < 2^31, else GOD_EINVAL after the call's device work).
 * Same order, conventions and errors as god_seed_reads. */
typedef struct {
    uint32_t ref_pos;
    uint32_t read_pos_strand;   /* read_pos | strand << 31 */
} god_anchor_compact;

GOD_API god_status god_seed_reads_compact(const god_index* idx, const uint8_t* reads, const uint64_t* read_offsets,
                                          uint32_t n_reads, god_phase_mode mode, uint8_t* phases, uint32_t t,
                                          god_anchor_compact* anchors, uint64_t* anchor_offsets, uint64_t cap,
                                          uint64_t* needed, god_stream stream);

/* Index build and seeding in one call (the mapper's flow: P:286 (1)-(3) then P:298-308 on one reference
 * and one read set), with the transfers overlapped across the two stages.  Same results as
 * god_build_index(prm, ref, ref_offsets, n_refs, cutoff, out_index, stream) followed by god_seed_reads
 * (compact == 0: anchors is god_anchor[cap]) or god_seed_reads_compact (compact != 0: anchors is
 * god_anchor_compact[cap]) on *out_index; every argument as documented there.  With host buffers and
 * >= 2^21 reads the first read batches are queued on the copy stream right behind the reference, so the
 * host link stays busy while the index is sorted; otherwise it is exactly the two calls in sequence.
 * *out_index is set as soon as the index is built, also when the seeding part then fails (GOD_ETRUNC
 * with *needed, or an error): the caller owns it (god_index_free).  Synchronizes. */
GOD_API god_status god_build_index_and_seed(const god_params* prm, const uint8_t* ref, const uint64_t* ref_offsets,
                                            uint32_t n_refs, const god_cutoff* cutoff, god_index** out_index,
                                            const uint8_t* reads, const uint64_t* read_offsets, uint32_t n_reads,
                                            god_phase_mode mode, uint8_t* phases, uint32_t t, int compact,
                                            void* anchors, uint64_t* anchor_offsets, uint64_t cap, uint64_t* needed,
                                            god_stream stream);

/* ---- location voting (section 3.4, Fig. 8; rescue P:398) ----
 * Consumes the anchors of god_seed_reads (same reads, same phases).  Readings (DESIGN.md §2,
 * V1-V6):
 *  (1) adjusted location of each anchor: forward (strand 0) diag = ref_pos - read_pos;
 *      reverse (strand 1) diag = ref_pos + read_end, read_end = original read coordinate of the
 *      read k-mer's last included base under the read's phase (colinear reverse anchors share
 *      it).  Anchors with equal (hash, strand, diag) are one vote ("consider both repeated
 *      seeds ... and repeated mapping locations only once").
 *  (2)-(3) one sorted list per read; sweep per strand: Delta0 = the first diag, the
 *      cluster takes the following anchors with diag - Delta0 <= D, the first beyond D is the next
 *      Delta0.  D = 0 means D = the read's length.
 *  (4) winners: votes >= V, sorted by votes descending (ties: strand, then Delta0 ascending),
 *      at most max_pairs (0 = no limit).  No winner and >= 1 anchor: the single
 *      best cluster, rescued = 1.  No anchor: no location.
 * Each location reports the [min, max] ref_pos and read_pos of its member anchors (Fig. 8B's
 * subsequence pairs).  Output CSR: locations of read r in [out_offsets[r], out_offsets[r+1]);
 * read_id = r.  anchors: 16-B god_anchor records (the full form of god_seed_reads; the 8-B
 * god_anchor_compact form is NOT accepted), at least anchor_offsets[n_reads] of them; any
 * alignment.  cap = location capacity (GOD_ETRUNC + *needed).  GOD_EINVAL if an anchor's
 * read_pos is not an included position of its read under phases[r] (anchors and phases from
 * different calls), or a read has >= 2^29 anchors.  Synchronizes. */
typedef struct {
    uint32_t D;           /* maximum allowed distance; 0 = read length */
    uint32_t V;           /* voting threshold */
    uint32_t max_pairs;   /* cap on winning locations per read; 0 = no limit */
} god_vote_params;

typedef struct {
    uint32_t read_id;
    uint32_t strand;      /* 0 forward, 1 reverse complement */
    int64_t diag;         /* Delta0 (forward: ref - read; reverse: ref + read_end) */
    uint32_t votes;
    uint32_t rescued;     /* 1: the read's rescue location (votes < V) */
    uint32_t ref_lo, ref_hi, read_lo, read_hi;
} god_vote;

GOD_API god_status god_vote_reads(const god_index* idx, const uint8_t* reads, const uint64_t* read_offsets,
                                  uint32_t n_reads, const uint8_t* phases, const god_anchor* anchors,
                                  const uint64_t* anchor_offsets, const god_vote_params* vp, god_vote* out,
                                  uint64_t* out_offsets, uint64_t cap, uint64_t* needed, god_stream stream);

/* ---- containment search, desk scale ----
 * The reference sequences are processed in batches of consecutive sequences holding at most
 * batch_bases bases ("-I"; a longer sequence is a batch of its own; 0 = one batch), each
 * batch's index built on the fly with `cutoff` applied within the batch (C1).  Every read is
 * phase-selected (SELECT, cap t), seeded and voted (vp) against each batch; "mapped read ... the
 * read that receives a mapping location using the location voting step": a read maps to
 * sequence i if one of its voted locations (winning or rescue) has ref_lo inside i (C2).
 * Outputs per reference sequence (n_refs each): mapped_reads = distinct reads mapped to it,
 * mapped_bases = the sum of their lengths (coverage = mapped_bases / length, C3), accepted = 1 iff
 * mapped_reads >= min_reads and mapped_bases * cov_den >= cov_num * length ("at least
 * 100,000 mapped reads with a genome coverage of at least 1"; C4).  Each batch < 2^32 bases.
 * Synchronizes. */
typedef struct {
    uint64_t batch_bases;   /* I: bases per reference batch (0 = all at once) */
    uint32_t min_reads;     /* accept: mapped reads >= min_reads */
    uint32_t cov_num, cov_den;  /* accept: coverage >= cov_num / cov_den (cov_den >= 1) */
} god_contain_params;

GOD_API god_status god_contain(const god_params* prm, const uint8_t* refs, const uint64_t* ref_offsets,
                               uint32_t n_refs, const god_cutoff* cutoff, const uint8_t* reads,
                               const uint64_t* read_offsets, uint32_t n_reads, uint32_t t,
                               const god_vote_params* vp, const god_contain_params* cp, uint64_t* mapped_reads,
                               uint64_t* mapped_bases, uint8_t* accepted, god_stream stream);

/* ---- seed-comparison harness (section 2.1.1-2.1.2, Fig. 4) ----
 * For pair i, sequences orig[offsets[i] .. offsets[i+1]) and mut[same range] (equal lengths,
 * <= 4096 bases), with prm's pattern P, k and w:
 *  matches[4i + a], totals[4i + a]: the seed matching rate matches/totals of extractor a (P:87:
 *    "the ratio of the number of matching seeds ... to the total number of extracted seeds"):
 *    totals = seed occurrences of the mutated sequence, matches = those whose hash is among the
 *    original's seeds.  a = 0 "All Seeds": every N-free k-mer, H_k(canonical); 1 "Minimizers":
 *    (w,k)-minimizers (pattern '1'); 2 "Spaced": per window start the bases at offsets j < k with
 *    P[j mod p] = 1, H over the included bases (canonical); 3 "Genome-on-Diet": minimizers of the
 *    patterned sequence, the original in phase 0, the mutated one in the phase s < p with the best
 *    rate (god_phase[i]; a phase without seeds has no rate; ties -> smaller s).
 *  edit[i]: Levenshtein distance of the pair, unit costs, bytes compared exactly.
 * Readings S1-S5: DESIGN.md §2.  GOD_EINVAL: a pair longer than 4096 bases, or a spaced mask of
 * weight > 28.  Synchronizes. */
GOD_API god_status god_seed_harness(const god_params* prm, const uint8_t* orig, const uint8_t* mut,
                                    const uint64_t* offsets, uint32_t n_pairs, uint64_t* edit, uint64_t* matches,
                                    uint64_t* totals, uint32_t* god_phase, god_stream stream);

/* Accepted pairs (reading S5) for n_thresholds edit-distance thresholds E[e]: the rate
 * threshold is the minimum rate matches/totals over the pairs with edit <= E[e]; accepted[4e + a] =
 * pairs of extractor a whose rate >= that threshold (pairs with totals 0 have no rate; no rated pair
 * within E -> 0).  Inputs as written by god_seed_harness.  Synchronizes. */
GOD_API god_status god_harness_accepted(const uint64_t* edit, const uint64_t* matches, const uint64_t* totals,
                                        uint32_t n_pairs, const uint64_t* thresholds, uint32_t n_thresholds,
                                        uint64_t* accepted, god_stream stream);

/* ---- tracing: per-kernel device time by CUDA events on the launching stream ----
 * Off by default.  When on, every kernel launch is bracketed by two events; god_profile_query
 * synchronizes on the pending events and returns, per kernel name (in first-launch order), the
 * accumulated milliseconds and launch count: names are written NUL-separated into `names`
 * (capacity names_len bytes), ms[i] and launches[i] for i < return value (<= max_entries).
 * god_launch_count() counts every kernel launch of the library since load (always on).
 * god_profile_units(name) returns the work units recorded for the launches named `name` while
 * profiling was on: for the extraction launches ("extract_ref", "extract_phase", "extract_seed")
 * the number of k-mer start positions processed (sum of n_k over the jobs); 0 for other names. */
GOD_API void god_profile_enable(int on);
GOD_API void god_profile_reset(void);
GOD_API int god_profile_query(char* names, size_t names_len, double* ms, uint64_t* launches, int max_entries);
GOD_API uint64_t god_launch_count(void);
GOD_API uint64_t god_profile_units(const char* name);

#ifdef __cplusplus
}
#endif
#endif /* GOD_H */
