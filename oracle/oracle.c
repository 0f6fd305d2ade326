/*
 * oracle.c — CPU ORACLE (test infrastructure only; see oracle.h for who may call it).
 *
 * A plain, slow, obviously-correct, single-threaded restatement of the Genome-on-Diet hot path
 * (arXiv 2211.08157, PAPER.md).  No blocking, no fusion, no rolling state: every k-mer value is
 * recomputed from its bases, every window minimum is recomputed by a scan of the window, the index
 * is qsort + a linear scan, lookups are binary searches.  Readings where the paper is silent or
 * garbled are SURVEY.md §8(c) O1-O9 (listed in DESIGN.md §2).
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------ */
/* O1 — alphabet and 2-bit encoding.  P:282 (alphabet ACGT + N), P:368/P:370 (2-bit encoding).  */
int or_code(uint8_t b) {
    switch (b) {
        case 'A': case 'a': return 0;
        case 'C': case 'c': return 1;
        case 'G': case 'g': return 2;
        case 'T': case 't': return 3;
        default: return OR_N;
    }
}

/* O2 — the diet pattern P[0..p-1] over {0,1}, weight x = #ones, beta = p/x.  P:282, P:286 (1). */
int or_parse_pattern(const char* text, or_pattern* out) {
    if (!text || !out) return -1;
    size_t p = strlen(text);
    if (p == 0 || p > 64) return -1;
    uint32_t x = 0;
    for (size_t i = 0; i < p; i++) {
        if (text[i] == '1') { out->bit[i] = 1; x++; }
        else if (text[i] == '0') out->bit[i] = 0;
        else return -1;
    }
    if (x == 0) return -1;
    out->p = (uint32_t)p;
    out->x = x;
    return 0;
}

/* O3 — patterned sequence PQ_s (PQ_s ⊆ {Q[i+s]·P[i mod p]}; P:308 with s = a; P:282 PR
 * with s = 0).  Keep original position i iff i >= s and P[(i - s) mod p] = 1, in increasing i. */
int64_t or_sparsify(const uint8_t* seq, uint64_t L, const or_pattern* P, uint32_t s, uint8_t* codes, uint64_t* orig) {
    if (s >= P->p) return -1;
    int64_t n = 0;
    for (uint64_t i = 0; i < L; i++) {
        if (i < s) continue;
        if (P->bit[(i - s) % P->p] != 1) continue;
        if (codes) codes[n] = (uint8_t)or_code(seq[i]);
        if (orig) orig[n] = i;
        n++;
    }
    return n;
}

/* O5 — Thomas Wang's invertible 64-bit integer hash (ref. 120), each step mod m = 4^k.  */
uint64_t or_hash(uint64_t key, int k) {
    uint64_t m = (k >= 32) ? ~0ull : ((1ull << (2 * k)) - 1);   /* mask = m - 1 */
    key = (~key + (key << 21)) & m;      /* x1 = 2^21 x - x - 1 */
    key = key ^ (key >> 24);             /* x2 */
    key = (key + (key << 3) + (key << 8)) & m;  /* x3 = 265 x2 */
    key = key ^ (key >> 14);             /* x4 */
    key = (key + (key << 2) + (key << 4)) & m;  /* x5 = 21 x4 */
    key = key ^ (key >> 28);             /* x6 */
    key = (key + (key << 31)) & m;       /* H = (2^31 + 1) x6 */
    return key;
}

void or_hash_batch(const uint64_t* x, uint64_t n, int k, uint64_t* out) {
    for (uint64_t i = 0; i < n; i++) out[i] = or_hash(x[i], k);
}

/* ------------------------------------------------------------------------------------------ */
/* O4 + O6 — double-strand (w,k)-minimizers of the patterned sequence.
 *  P:286 (3): "computes minimizers of the patterned genome sequence ... the start location of each
 *             minimizer in the original unpatterned reference genome".
 *  P:294:     "the double-strand (w,k)-minimizer of a string is the smallest k-mer in a surrounding
 *             window of w consecutive k-mers".
 *  P:370:     an N terminates the current computation; restart after it.
 * Step 1: t = Sparsify(seq, P, s) with orig[].
 * Step 2: for each k-mer start j with t[j..j+k-1] free of N: fwd, rev, canonical, strand, hash;
 *         palindromes (fwd == rev) are marked and never take part in a window minimum.
 * Step 3: runs of consecutive valid starts (N-free segments).  Windows: every w consecutive
 *         starts of a run, or the whole run if it has fewer than w starts.
 * Step 4: in every window, every non-palindromic start whose hash equals the window minimum is
 *         selected (all ties kept).  Output selected starts in increasing j.                  */
int64_t or_minimizers(const uint8_t* seq, uint64_t L, const or_pattern* P, uint32_t s, int k, int w,
                      uint64_t pos_base, or_mz* out, uint64_t cap) {
    if (s >= P->p || k < 1 || k > 28 || w < 1) return -1;
    int64_t n = or_sparsify(seq, L, P, s, NULL, NULL);
    if (n < k) return 0;
    uint8_t* t = (uint8_t*)malloc((size_t)n);
    uint64_t* orig = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
    or_sparsify(seq, L, P, s, t, orig);
    int64_t nk = n - k + 1;                       /* k-mer start positions 0..nk-1 */
    uint8_t* valid = (uint8_t*)calloc((size_t)nk, 1);
    uint8_t* pal = (uint8_t*)calloc((size_t)nk, 1);
    uint8_t* z = (uint8_t*)calloc((size_t)nk, 1);
    uint64_t* h = (uint64_t*)calloc((size_t)nk, sizeof(uint64_t));
    uint8_t* sel = (uint8_t*)calloc((size_t)nk, 1);
    /* step 2 */
    for (int64_t j = 0; j < nk; j++) {
        int ok = 1;
        for (int i = 0; i < k; i++) if (t[j + i] == OR_N) { ok = 0; break; }
        if (!ok) continue;
        uint64_t fwd = 0, rev = 0;
        for (int i = 0; i < k; i++) fwd = fwd * 4 + t[j + i];                     /* first base most significant */
        for (int i = 0; i < k; i++) rev = rev * 4 + (uint64_t)(3 - t[j + k - 1 - i]); /* reverse complement */
        valid[j] = 1;
        if (fwd == rev) { pal[j] = 1; continue; }
        uint64_t canon = fwd < rev ? fwd : rev;
        z[j] = fwd > rev;
        h[j] = or_hash(canon, k);
    }
    /* steps 3-4 */
    int64_t j = 0;
    while (j < nk) {
        if (!valid[j]) { j++; continue; }
        int64_t rs = j;
        while (j < nk && valid[j]) j++;
        int64_t re = j;                          /* run [rs, re) */
        int64_t nrun = re - rs;
        int64_t win = nrun >= w ? w : nrun;
        for (int64_t a = rs; a + win <= re; a++) {
            int have = 0; uint64_t mn = 0;
            for (int64_t i = a; i < a + win; i++) {
                if (pal[i]) continue;
                if (!have || h[i] < mn) { mn = h[i]; have = 1; }
            }
            if (!have) continue;
            for (int64_t i = a; i < a + win; i++) if (!pal[i] && h[i] == mn) sel[i] = 1;
        }
    }
    int64_t cnt = 0;
    for (int64_t q = 0; q < nk; q++) {
        if (!sel[q]) continue;
        if ((uint64_t)cnt < cap && out) { out[cnt].hash = h[q]; out[cnt].pos = pos_base + orig[q]; out[cnt].strand = z[q]; }
        cnt++;
    }
    free(t); free(orig); free(valid); free(pal); free(z); free(h); free(sel);
    return cnt;
}

int64_t or_minimizers_batch(const uint8_t* seq, const uint64_t* offsets, uint32_t n, const uint8_t* phases,
                            const char* pattern, int k, int w, int global_pos, or_mz* out, uint64_t cap,
                            uint64_t* out_offsets) {
    or_pattern P;
    if (or_parse_pattern(pattern, &P)) return -1;
    uint64_t tot = 0;
    for (uint32_t r = 0; r < n; r++) {
        uint32_t s = phases ? phases[r] : 0;
        if (out_offsets) out_offsets[r] = tot;
        uint64_t room = tot < cap ? cap - tot : 0;
        int64_t c = or_minimizers(seq + offsets[r], offsets[r + 1] - offsets[r], &P, s, k, w,
                                  global_pos ? offsets[r] : 0, out ? out + (tot < cap ? tot : cap) : NULL, room);
        if (c < 0) return -1;
        tot += (uint64_t)c;
    }
    if (out_offsets) out_offsets[n] = tot;
    return tot > cap && out ? -1 : (int64_t)tot;
}

/* ------------------------------------------------------------------------------------------ */
/* O7 — the seed index.  P:286 (3) key = hash, value = list of start locations (original coords);
 * P:294 "append the minimizer information to an array and sort the array after collecting ...
 * then add it to the hash table"; P:302 discard minimizers occurring >= a user threshold.
 * Cutoff (reading O7): n distinct hashes with counts a_0 <= ... <= a_{n-1}, m = floor(n*num/den),
 * tau = a_{n-m-1}; keep h iff c(h) <= tau.  max_occ >= 0 overrides: keep iff c(h) <= max_occ.   */
struct or_index {
    or_pattern P; int k, w;
    uint64_t n_kept;
    uint64_t* hash; uint64_t* pos; uint8_t* strand;     /* kept entries, (hash,pos) order */
    uint64_t n_keys; uint64_t* key; uint64_t* key_first; uint32_t* key_count;  /* distinct kept hashes */
    or_index_stats st;
};

static int cmp_mz(const void* a, const void* b) {
    const or_mz* x = (const or_mz*)a; const or_mz* y = (const or_mz*)b;
    if (x->hash != y->hash) return x->hash < y->hash ? -1 : 1;
    if (x->pos != y->pos) return x->pos < y->pos ? -1 : 1;
    return 0;
}
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

/* Cutoff (reading O7 of SURVEY §8(c); "discard the most frequently (>= a user-defined
 * threshold) occurring minimizers"): sort the n distinct-hash counts ascending a_0..a_{n-1},
 * m = floor(n*num/den); tau = a_{n-m-1} (m = 0 gives tau = max count: keep all). */
uint64_t or_cutoff_tau(const uint64_t* counts, uint64_t n, uint32_t num, uint32_t den, uint64_t* m_out) {
    uint64_t m = den ? (uint64_t)(((unsigned __int128)n * num) / den) : 0;
    if (m_out) *m_out = m;
    if (n == 0 || m >= n) return 0;
    uint64_t* a = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
    memcpy(a, counts, sizeof(uint64_t) * (size_t)n);
    qsort(a, (size_t)n, sizeof(uint64_t), cmp_u64);
    uint64_t tau = a[n - m - 1];
    free(a);
    return tau;
}

or_index* or_build_index(const uint8_t* ref, const uint64_t* offsets, uint32_t n, const char* pattern, int k, int w,
                         uint32_t frac_num, uint32_t frac_den, int64_t max_occ) {
    or_pattern P;
    if (or_parse_pattern(pattern, &P) || k < 1 || k > 28 || w < 1 || (max_occ < 0 && frac_den == 0)) return NULL;
    /* collect: E = multiset of (h, global pos, z) over every reference sequence, phase 0 */
    int64_t tot = or_minimizers_batch(ref, offsets, n, NULL, pattern, k, w, 1, NULL, 0, NULL);
    if (tot < 0) return NULL;
    or_mz* E = (or_mz*)malloc(sizeof(or_mz) * (size_t)(tot ? tot : 1));
    or_minimizers_batch(ref, offsets, n, NULL, pattern, k, w, 1, E, (uint64_t)tot, NULL);
    /* sort */
    qsort(E, (size_t)tot, sizeof(or_mz), cmp_mz);
    /* count per distinct hash */
    uint64_t nd = 0;
    for (int64_t i = 0; i < tot; i++) if (i == 0 || E[i].hash != E[i - 1].hash) nd++;
    uint64_t* cnt = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nd ? nd : 1));
    uint64_t d = 0;
    for (int64_t i = 0; i < tot; ) {
        int64_t j = i;
        while (j < tot && E[j].hash == E[i].hash) j++;
        cnt[d++] = (uint64_t)(j - i);
        i = j;
    }
    /* cutoff: fraction rule, or the absolute override (keep iff count <= max_occ) */
    uint64_t m = 0, tau;
    if (max_occ >= 0) tau = (uint64_t)max_occ;
    else tau = or_cutoff_tau(cnt, nd, frac_num, frac_den, &m);
    or_index* ix = (or_index*)calloc(1, sizeof(or_index));
    ix->P = P; ix->k = k; ix->w = w;
    ix->st.n_entries_all = (uint64_t)tot; ix->st.n_distinct_all = nd; ix->st.m = m; ix->st.tau = tau;
    /* table: keep hashes with count <= tau */
    ix->hash = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(tot ? tot : 1));
    ix->pos = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(tot ? tot : 1));
    ix->strand = (uint8_t*)malloc((size_t)(tot ? tot : 1));
    ix->key = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nd ? nd : 1));
    ix->key_first = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nd ? nd : 1));
    ix->key_count = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(nd ? nd : 1));
    d = 0;
    for (int64_t i = 0; i < tot; ) {
        uint64_t c = cnt[d++];
        if (c <= tau) {
            ix->key[ix->n_keys] = E[i].hash;
            ix->key_first[ix->n_keys] = ix->n_kept;
            ix->key_count[ix->n_keys] = (uint32_t)c;
            ix->n_keys++;
            for (uint64_t q = 0; q < c; q++) {
                ix->hash[ix->n_kept] = E[i + q].hash;
                ix->pos[ix->n_kept] = E[i + q].pos;
                ix->strand[ix->n_kept] = E[i + q].strand;
                ix->n_kept++;
            }
            ix->st.kept_distinct++;
            ix->st.kept_entries += c;
        } else {
            ix->st.dropped_distinct++;
            ix->st.dropped_entries += c;
        }
        i += (int64_t)c;
    }
    free(cnt); free(E);
    return ix;
}

void or_index_free(or_index* ix) {
    if (!ix) return;
    free(ix->hash); free(ix->pos); free(ix->strand); free(ix->key); free(ix->key_first); free(ix->key_count);
    free(ix);
}

void or_index_stats_get(const or_index* ix, or_index_stats* st) { *st = ix->st; }

uint64_t or_index_dump(const or_index* ix, uint64_t* hash, uint64_t* pos, uint8_t* strand, uint64_t cap) {
    for (uint64_t i = 0; i < ix->n_kept && i < cap; i++) {
        if (hash) hash[i] = ix->hash[i];
        if (pos) pos[i] = ix->pos[i];
        if (strand) strand[i] = ix->strand[i];
    }
    return ix->n_kept;
}

/* binary search over the sorted distinct kept keys; returns key index or -1 */
static int64_t find_key(const or_index* ix, uint64_t h) {
    int64_t lo = 0, hi = (int64_t)ix->n_keys - 1;
    while (lo <= hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (ix->key[mid] == h) return mid;
        if (ix->key[mid] < h) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

uint32_t or_index_occ(const or_index* ix, uint64_t h) {
    int64_t q = find_key(ix, h);
    return q < 0 ? 0 : ix->key_count[q];
}

/* ------------------------------------------------------------------------------------------ */
/* O8 — pattern alignment.  For s = 0..p-1: M_s = minimizers of PQ_s (position order).
 * "the same number of minimizer seeds from each PQ_s" and "limit the number of calculated
 * minimizers in each PQ_s to a user-defined threshold" t  =>  c = min(t, min_s |M_s|);
 * score_s = sum over the first c records of M_s of occ(hash);  a = argmax_s score_s, ties -> smallest s. */
int or_select_phase(const or_index* ix, const uint8_t* read, uint64_t L, uint32_t t, uint64_t* scores) {
    uint32_t p = ix->P.p;
    if (p == 1) { if (scores) scores[0] = 0; return 0; }
    or_mz* M[64]; int64_t cntM[64];
    int64_t cmin = -1;
    for (uint32_t s = 0; s < p; s++) {
        int64_t c = or_minimizers(read, L, &ix->P, s, ix->k, ix->w, 0, NULL, 0);
        M[s] = (or_mz*)malloc(sizeof(or_mz) * (size_t)(c ? c : 1));
        or_minimizers(read, L, &ix->P, s, ix->k, ix->w, 0, M[s], (uint64_t)c);
        cntM[s] = c;
        if (cmin < 0 || c < cmin) cmin = c;
    }
    int64_t c = cmin < (int64_t)t ? cmin : (int64_t)t;
    int best = 0; uint64_t best_score = 0;
    for (uint32_t s = 0; s < p; s++) {
        uint64_t sc = 0;
        for (int64_t i = 0; i < c; i++) sc += or_index_occ(ix, M[s][i].hash);
        if (scores) scores[s] = sc;
        if (s == 0 || sc > best_score) { best_score = sc; best = (int)s; }
        free(M[s]);
    }
    (void)cntM;
    return best;
}

static int cmp_anchor(const void* a, const void* b) {
    const or_anchor* x = (const or_anchor*)a; const or_anchor* y = (const or_anchor*)b;
    if (x->read_id != y->read_id) return x->read_id < y->read_id ? -1 : 1;
    if (x->ref_pos != y->ref_pos) return x->ref_pos < y->ref_pos ? -1 : 1;
    if (x->read_pos != y->read_pos) return x->read_pos < y->read_pos ? -1 : 1;
    if (x->strand != y->strand) return x->strand < y->strand ? -1 : 1;
    return 0;
}

/* O9 — compressed seeding: minimizers of PQ_a, every kept index entry with the same
 * hash is a match -> anchor (read_id, ref_pos, read_pos, ref strand XOR read strand). */
int64_t or_seed_read(const or_index* ix, const uint8_t* read, uint64_t L, uint32_t a, uint32_t read_id,
                     or_anchor* out, uint64_t cap) {
    int64_t c = or_minimizers(read, L, &ix->P, a, ix->k, ix->w, 0, NULL, 0);
    if (c < 0) return -1;
    or_mz* M = (or_mz*)malloc(sizeof(or_mz) * (size_t)(c ? c : 1));
    or_minimizers(read, L, &ix->P, a, ix->k, ix->w, 0, M, (uint64_t)c);
    uint64_t tot = 0;
    for (int64_t i = 0; i < c; i++) {
        int64_t q = find_key(ix, M[i].hash);
        if (q < 0) continue;
        for (uint64_t e = ix->key_first[q]; e < ix->key_first[q] + ix->key_count[q]; e++) {
            if (out && tot < cap) {
                out[tot].read_id = read_id;
                out[tot].ref_pos = (uint32_t)ix->pos[e];
                out[tot].read_pos = (uint32_t)M[i].pos;
                out[tot].strand = (uint32_t)(ix->strand[e] ^ M[i].strand);
            }
            tot++;
        }
    }
    if (out) qsort(out, (size_t)(tot < cap ? tot : cap), sizeof(or_anchor), cmp_anchor);
    free(M);
    return (int64_t)tot;
}

int64_t or_seed_reads_batch(const or_index* ix, const uint8_t* reads, const uint64_t* offsets, uint32_t n,
                            int mode, uint8_t* phases, uint32_t t, or_anchor* out, uint64_t cap,
                            uint64_t* anchor_offsets) {
    uint64_t tot = 0;
    for (uint32_t r = 0; r < n; r++) {
        const uint8_t* q = reads + offsets[r];
        uint64_t L = offsets[r + 1] - offsets[r];
        uint32_t a;
        if (mode == 0) { a = (uint32_t)or_select_phase(ix, q, L, t, NULL); if (phases) phases[r] = (uint8_t)a; }
        else { a = phases ? phases[r] : 0; if (a >= ix->P.p) return -1; }
        if (anchor_offsets) anchor_offsets[r] = tot;
        uint64_t room = tot < cap ? cap - tot : 0;
        int64_t c = or_seed_read(ix, q, L, a, r, out ? out + (tot < cap ? tot : cap) : NULL, room);
        if (c < 0) return -1;
        tot += (uint64_t)c;
    }
    if (anchor_offsets) anchor_offsets[n] = tot;
    return tot > cap && out ? -1 : (int64_t)tot;
}

/* ------------------------------------------------------------------------------------------ */
/* Location voting (P:312-324 steps (1)-(4), Fig. 8) and the rescue location.
 * Readings (V1-V6):
 *  V1 adjusted location ("subtract the location of each seed extracted from the read sequence
 *     from that of its corresponding matching seed"): forward hit (strand 0)
 *     diag = ref_pos - read_pos; reverse hit (strand 1) diag = ref_pos + read_end, read_end = the
 *     original read coordinate of the read k-mer's LAST included base (O9's reverse invariant:
 *     colinear reverse hits share ref_pos + read_end = g + L - 1).
 *  V2 "consider both repeated seeds (e.g., having the same hash value) ... and repeated mapping
 *     locations only once": hits with equal (hash, strand, diag) are one vote.
 *  V3 the sweep runs over the hits sorted by (strand, diag); each strand is its own
 *     coordinate system: Delta0 = first diag, members = following hits of the same strand with
 *     diag - Delta0 <= D, the first hit beyond D (or of the other strand) is the next Delta0.
 *  V4 a cluster wins iff votes >= V; winners are sorted by votes (descending; ties by
 *     strand, then Delta0, ascending) and truncated to max_pairs ("we limit the size of the list
 *     ... to a user-defined number"; 0 = no limit).
 *  V5 rescue: if no cluster wins and the read has hits, the output is the single cluster
 *     with the most votes (same tie order), flagged rescued.
 *  V6 each cluster reports the ref / read spans [min, max] of its member hits (Fig. 8B's
 *     subsequence pairs); D = 0 means D = read length (SPEC's short-read default). */
static int cmp_hit(const void* a, const void* b) {
    const or_hit* x = (const or_hit*)a; const or_hit* y = (const or_hit*)b;
    if (x->strand != y->strand) return x->strand < y->strand ? -1 : 1;
    if (x->diag != y->diag) return x->diag < y->diag ? -1 : 1;
    if (x->hash != y->hash) return x->hash < y->hash ? -1 : 1;
    if (x->ref_pos != y->ref_pos) return x->ref_pos < y->ref_pos ? -1 : 1;
    if (x->read_pos != y->read_pos) return x->read_pos < y->read_pos ? -1 : 1;
    return 0;
}

/* V4 order: more votes first, then smaller strand, then smaller Delta0 */
static int vote_before(const or_vote* x, const or_vote* y) {
    if (x->votes != y->votes) return x->votes > y->votes;
    if (x->strand != y->strand) return x->strand < y->strand;
    return x->diag < y->diag;
}
static int cmp_vote(const void* a, const void* b) {
    const or_vote* x = (const or_vote*)a; const or_vote* y = (const or_vote*)b;
    return vote_before(x, y) ? -1 : (vote_before(y, x) ? 1 : 0);
}

int64_t or_vote_hits(or_hit* hits, uint64_t n, uint64_t D, uint32_t V, uint32_t max_pairs, uint32_t read_id,
                     or_vote* out, uint64_t cap) {
    if (n == 0) return 0;
    /* step (2): a single sorted list (the paper merges the per-seed sorted lists; qsort here) */
    qsort(hits, (size_t)n, sizeof(or_hit), cmp_hit);
    /* step (3): sweep */
    or_vote* cl = (or_vote*)malloc(sizeof(or_vote) * (size_t)n);
    uint64_t ncl = 0, i = 0;
    while (i < n) {
        or_vote c;
        memset(&c, 0, sizeof c);
        c.read_id = read_id; c.strand = hits[i].strand; c.diag = hits[i].diag;
        c.ref_lo = c.ref_hi = hits[i].ref_pos; c.read_lo = c.read_hi = hits[i].read_pos;
        uint64_t j = i;
        while (j < n && hits[j].strand == c.strand && (uint64_t)(hits[j].diag - c.diag) <= D) {
            /* V2: one vote per distinct (hash, strand, diag) — duplicates are adjacent after the sort */
            int dup = j > i && hits[j].diag == hits[j - 1].diag && hits[j].hash == hits[j - 1].hash;
            if (!dup) c.votes++;
            if (hits[j].ref_pos < c.ref_lo) c.ref_lo = hits[j].ref_pos;
            if (hits[j].ref_pos > c.ref_hi) c.ref_hi = hits[j].ref_pos;
            if (hits[j].read_pos < c.read_lo) c.read_lo = hits[j].read_pos;
            if (hits[j].read_pos > c.read_hi) c.read_hi = hits[j].read_pos;
            j++;
        }
        cl[ncl++] = c;
        i = j;                       /* the first location beyond D is the next Delta0 */
    }
    /* step (4): winners (votes >= V), sorted by votes, capped; else the rescue location */
    or_vote* win = (or_vote*)malloc(sizeof(or_vote) * (size_t)ncl);
    uint64_t nw = 0;
    for (uint64_t q = 0; q < ncl; q++) if (cl[q].votes >= V) win[nw++] = cl[q];
    int64_t res;
    if (nw > 0) {
        qsort(win, (size_t)nw, sizeof(or_vote), cmp_vote);
        if (max_pairs && nw > max_pairs) nw = max_pairs;
        for (uint64_t q = 0; q < nw && q < cap; q++) if (out) out[q] = win[q];
        res = (int64_t)nw;
    } else {
        uint64_t b = 0;
        for (uint64_t q = 1; q < ncl; q++) if (vote_before(&cl[q], &cl[b])) b = q;
        cl[b].rescued = 1;
        if (out && cap) out[0] = cl[b];
        res = 1;
    }
    free(win);
    free(cl);
    return res;
}

/* Step (1) for one read: the minimizers of PQ_a (O6 on Sparsify(read, P, a)) matched against the
 * index (O9), each match turned into an adjusted location (V1). */
int64_t or_vote_read(const or_index* ix, const uint8_t* read, uint64_t L, uint32_t a, uint32_t read_id,
                     uint32_t D, uint32_t V, uint32_t max_pairs, or_vote* out, uint64_t cap) {
    if (a >= ix->P.p) return -1;
    int64_t c = or_minimizers(read, L, &ix->P, a, ix->k, ix->w, 0, NULL, 0);
    if (c <= 0) return c;
    or_mz* M = (or_mz*)malloc(sizeof(or_mz) * (size_t)c);
    or_minimizers(read, L, &ix->P, a, ix->k, ix->w, 0, M, (uint64_t)c);
    int64_t nj = or_sparsify(read, L, &ix->P, a, NULL, NULL);
    uint64_t* orig = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nj ? nj : 1));
    or_sparsify(read, L, &ix->P, a, NULL, orig);
    uint64_t nh = 0;
    for (int64_t i = 0; i < c; i++) { int64_t q = find_key(ix, M[i].hash); if (q >= 0) nh += ix->key_count[q]; }
    or_hit* H = (or_hit*)malloc(sizeof(or_hit) * (size_t)(nh ? nh : 1));
    uint64_t h = 0;
    for (int64_t i = 0; i < c; i++) {
        int64_t q = find_key(ix, M[i].hash);
        if (q < 0) continue;
        /* the read k-mer starting at orig[j] = pos ends at orig[j + k - 1] */
        int64_t j = 0;
        while ((uint64_t)orig[j] != M[i].pos) j++;
        uint64_t read_end = orig[j + ix->k - 1];
        for (uint64_t e = ix->key_first[q]; e < ix->key_first[q] + ix->key_count[q]; e++) {
            or_hit* t = &H[h++];
            t->hash = M[i].hash;
            t->strand = (uint32_t)(ix->strand[e] ^ M[i].strand);
            t->ref_pos = (uint32_t)ix->pos[e];
            t->read_pos = (uint32_t)M[i].pos;
            t->diag = t->strand == 0 ? (int64_t)ix->pos[e] - (int64_t)M[i].pos
                                     : (int64_t)ix->pos[e] + (int64_t)read_end;
        }
    }
    int64_t r = or_vote_hits(H, nh, D ? D : L, V, max_pairs, read_id, out, cap);
    free(M); free(orig); free(H);
    return r;
}

int64_t or_vote_reads_batch(const or_index* ix, const uint8_t* reads, const uint64_t* offsets, uint32_t n,
                            const uint8_t* phases, uint32_t D, uint32_t V, uint32_t max_pairs, or_vote* out,
                            uint64_t cap, uint64_t* vote_offsets) {
    uint64_t tot = 0;
    for (uint32_t r = 0; r < n; r++) {
        uint32_t a = phases ? phases[r] : 0;
        if (vote_offsets) vote_offsets[r] = tot;
        uint64_t room = tot < cap ? cap - tot : 0;
        int64_t c = or_vote_read(ix, reads + offsets[r], offsets[r + 1] - offsets[r], a, r,
                                 D, V, max_pairs, out ? out + (tot < cap ? tot : cap) : NULL, room);
        if (c < 0) return -1;
        tot += (uint64_t)c;
    }
    if (vote_offsets) vote_offsets[n] = tot;
    return tot > cap && out ? -1 : (int64_t)tot;
}

/* ------------------------------------------------------------------------------------------ */
/* Containment search at desk scale (SPEC contain module).  Readings
 * (C1-C4):
 *  C1 the references are processed in batches of consecutive sequences of at most batch_bases
 *     bases ("-I", "limit the loaded number of bases at once"; a longer sequence is a batch
 *     of its own; 0 = one batch); each batch's index is built on the fly, with the cutoff
 *     computed within the batch.
 *  C2 every read is phase-selected (O8), seeded (O9) and voted (V1-V6) against each batch's index;
 *     "mapped read ... the read that receives a mapping location using the location voting step"
 *     (P:184): a read maps to reference t if one of its voted locations (winning or rescue) has
 *     its ref_lo inside t.
 *  C3 per reference: mapped_reads = number of distinct reads mapped to it; mapped_bases = the sum
 *     of their lengths; genome coverage = mapped_bases / len(t) (read depth; "a genome
 *     coverage of at least 1").
 *  C4 accepted iff mapped_reads >= min_reads and mapped_bases * cov_den >= cov_num * len(t)
 *     (100,000 reads and coverage 1 at RefSeq scale; both are parameters here). */
int or_contain(const uint8_t* refs, const uint64_t* ref_offsets, uint32_t n_refs, const char* pattern, int k, int w,
               uint32_t frac_num, uint32_t frac_den, int64_t max_occ, const uint8_t* reads,
               const uint64_t* read_offsets, uint32_t n_reads, uint32_t t, uint32_t D, uint32_t V,
               uint32_t max_pairs, uint64_t batch_bases, uint32_t min_reads, uint32_t cov_num, uint32_t cov_den,
               uint64_t* mapped_reads, uint64_t* mapped_bases, uint8_t* accepted) {
    for (uint32_t i = 0; i < n_refs; i++) { mapped_reads[i] = 0; mapped_bases[i] = 0; }
    uint32_t b0 = 0;
    while (b0 < n_refs) {
        /* C1: the batch [b0, b1) */
        uint32_t b1 = b0 + 1;
        while (b1 < n_refs && batch_bases && ref_offsets[b1 + 1] - ref_offsets[b0] <= batch_bases) b1++;
        if (!batch_bases) b1 = n_refs;
        uint32_t nb = b1 - b0;
        uint64_t* off = (uint64_t*)malloc(sizeof(uint64_t) * (nb + 1));
        for (uint32_t i = 0; i <= nb; i++) off[i] = ref_offsets[b0 + i] - ref_offsets[b0];
        or_index* ix = or_build_index(refs + ref_offsets[b0], off, nb, pattern, k, w, frac_num, frac_den, max_occ);
        if (!ix) { free(off); return -1; }
        /* C2 */
        for (uint32_t r = 0; r < n_reads; r++) {
            const uint8_t* q = reads + read_offsets[r];
            uint64_t L = read_offsets[r + 1] - read_offsets[r];
            uint32_t a = (uint32_t)or_select_phase(ix, q, L, t, NULL);
            int64_t nv = or_vote_read(ix, q, L, a, r, D, V, max_pairs, NULL, 0);
            if (nv <= 0) continue;
            or_vote* v = (or_vote*)malloc(sizeof(or_vote) * (size_t)nv);
            or_vote_read(ix, q, L, a, r, D, V, max_pairs, v, (uint64_t)nv);
            uint32_t* hit = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nv);
            int64_t nh = 0;
            for (int64_t j = 0; j < nv; j++) {
                uint32_t ti = 0;                     /* the batch sequence containing ref_lo */
                while (ti + 1 < nb && off[ti + 1] <= v[j].ref_lo) ti++;
                int seen = 0;
                for (int64_t u = 0; u < nh; u++) if (hit[u] == ti) seen = 1;
                if (!seen) hit[nh++] = ti;
            }
            for (int64_t u = 0; u < nh; u++) {    /* C3 */
                mapped_reads[b0 + hit[u]] += 1;
                mapped_bases[b0 + hit[u]] += L;
            }
            free(v); free(hit);
        }
        or_index_free(ix);
        free(off);
        b0 = b1;
    }
    for (uint32_t i = 0; i < n_refs; i++) {       /* C4 */
        unsigned __int128 lhs = (unsigned __int128)mapped_bases[i] * cov_den;
        unsigned __int128 rhs = (unsigned __int128)cov_num * (ref_offsets[i + 1] - ref_offsets[i]);
        accepted[i] = (uint8_t)(mapped_reads[i] >= min_reads && lhs >= rhs);
    }
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Seed-comparison harness (section 2.1.1-2.1.2).  Readings (DESIGN.md §2,
 * S1-S5):
 *  S2 a seed is the hash H of a canonical (multi-)k-mer; four extractors over a sequence:
 *     algo 0 "All Seeds": every k-mer start without N: H_k(canon);
 *     algo 1 "Minimizers": O6 with pattern '1', phase 0;
 *     algo 2 "Spaced": per window start i, the bases i + j for the ones of the mask
 *            M[j] = P[j mod p], j < k (span k, weight x_k = ones of M: "spaced seeds", the
 *            literature patterns are given with span = seed length); canonical over the included
 *            bases, hash H_{x_k};
 *     algo 3 "Genome-on-Diet": O6 on Sparsify(seq, P, s) (the original with s = 0).
 *  S3 rate = matches / total: total = seeds (occurrences) of the mutated sequence, matches = those
 *     whose hash is among the original's seeds ("ratio of the number of matching seeds ... to
 *     the total number of extracted seeds").  Genome-on-Diet scores the mutated sequence in every
 *     phase s < p against the original's phase 0 and keeps the best rate (smallest s on ties).
 *  S4 edit distance = Levenshtein, unit costs ("outputs the Levenshtein distance").  */
int64_t or_harness_seeds(const uint8_t* seq, uint64_t L, int algo, int k, int w, const char* pattern, uint32_t s,
                         uint64_t* out, uint64_t cap) {
    or_pattern P;
    if (or_parse_pattern(pattern, &P)) return -1;
    if (k < 1 || k > 28 || w < 1) return -1;
    int64_t n = 0;
    if (algo == 0) {
        for (uint64_t i = 0; i + (uint64_t)k <= L; i++) {
            uint64_t fwd = 0, rev = 0; int ok = 1;
            for (int j = 0; j < k; j++) {
                int c = or_code(seq[i + j]);
                if (c == OR_N) { ok = 0; break; }
                fwd = fwd * 4 + (uint64_t)c;
            }
            if (!ok) continue;
            for (int j = 0; j < k; j++) rev = rev * 4 + (uint64_t)(3 - or_code(seq[i + k - 1 - j]));
            uint64_t h = or_hash(fwd < rev ? fwd : rev, k);
            if (out && (uint64_t)n < cap) out[n] = h;
            n++;
        }
    } else if (algo == 1 || algo == 3) {
        or_pattern Q;
        if (algo == 1) or_parse_pattern("1", &Q); else Q = P;
        if (s >= Q.p) return -1;
        int64_t c = or_minimizers(seq, L, &Q, s, k, w, 0, NULL, 0);
        or_mz* M = (or_mz*)malloc(sizeof(or_mz) * (size_t)(c ? c : 1));
        or_minimizers(seq, L, &Q, s, k, w, 0, M, (uint64_t)c);
        for (int64_t i = 0; i < c; i++) { if (out && (uint64_t)n < cap) out[n] = M[i].hash; n++; }
        free(M);
    } else if (algo == 2) {
        int x = 0;
        for (int j = 0; j < k; j++) x += P.bit[j % P.p];
        if (x == 0 || x > 28) return x == 0 ? 0 : -1;
        for (uint64_t i = 0; i + (uint64_t)k <= L; i++) {
            uint8_t inc[28]; int ni = 0, ok = 1;
            for (int j = 0; j < k; j++) {
                if (!P.bit[j % P.p]) continue;
                int c = or_code(seq[i + j]);
                if (c == OR_N) { ok = 0; break; }
                inc[ni++] = (uint8_t)c;
            }
            if (!ok) continue;
            uint64_t fwd = 0, rev = 0;
            for (int j = 0; j < x; j++) fwd = fwd * 4 + inc[j];
            for (int j = 0; j < x; j++) rev = rev * 4 + (uint64_t)(3 - inc[x - 1 - j]);
            uint64_t h = or_hash(fwd < rev ? fwd : rev, x);
            if (out && (uint64_t)n < cap) out[n] = h;
            n++;
        }
    } else {
        return -1;
    }
    return n;
}

/* S3: matches of b's seeds among a's (set membership by linear scan of a's sorted seeds) */
static void rate_of(const uint64_t* sa, int64_t na, const uint64_t* sb, int64_t nb, uint64_t* m, uint64_t* t) {
    uint64_t mm = 0;
    for (int64_t i = 0; i < nb; i++) {
        int found = 0;
        for (int64_t j = 0; j < na && !found; j++) found = sa[j] == sb[i];
        mm += (uint64_t)found;
    }
    *m = mm; *t = (uint64_t)nb;
}

/* S4: textbook dynamic programming, unit costs */
int64_t or_levenshtein(const uint8_t* a, uint64_t la, const uint8_t* b, uint64_t lb) {
    uint64_t* prev = (uint64_t*)malloc(sizeof(uint64_t) * (lb + 1));
    uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * (lb + 1));
    for (uint64_t j = 0; j <= lb; j++) prev[j] = j;
    for (uint64_t i = 1; i <= la; i++) {
        cur[0] = i;
        for (uint64_t j = 1; j <= lb; j++) {
            uint64_t del = prev[j] + 1, ins = cur[j - 1] + 1, sub = prev[j - 1] + (a[i - 1] != b[j - 1]);
            uint64_t v = del < ins ? del : ins;
            cur[j] = v < sub ? v : sub;
        }
        uint64_t* t = prev; prev = cur; cur = t;
    }
    int64_t d = (int64_t)prev[lb];
    free(prev); free(cur);
    return d;
}

/* One pair: edit distance and (matches, total) for the four extractors (out_m[4], out_t[4]); the
 * Genome-on-Diet phase kept is written to *god_phase.  Returns the edit distance (-1 on error). */
int64_t or_harness_pair(const uint8_t* a, const uint8_t* b, uint64_t L, int k, int w, const char* pattern,
                        uint64_t* out_m, uint64_t* out_t, uint32_t* god_phase) {
    or_pattern P;
    if (or_parse_pattern(pattern, &P)) return -1;
    uint64_t* sa = (uint64_t*)malloc(sizeof(uint64_t) * (L + 1));
    uint64_t* sb = (uint64_t*)malloc(sizeof(uint64_t) * (L + 1));
    for (int algo = 0; algo < 4; algo++) {
        int64_t na = or_harness_seeds(a, L, algo, k, w, pattern, 0, sa, L + 1);
        if (na < 0) { free(sa); free(sb); return -1; }
        if (algo < 3) {
            int64_t nb = or_harness_seeds(b, L, algo, k, w, pattern, 0, sb, L + 1);
            rate_of(sa, na, sb, nb, &out_m[algo], &out_t[algo]);
        } else {
            /* the best rate m/t over the phases; a phase without seeds has no rate; ties -> smaller s */
            uint64_t bm = 0, bt = 0; uint32_t bs = 0;
            for (uint32_t s = 0; s < P.p; s++) {
                int64_t nb = or_harness_seeds(b, L, 3, k, w, pattern, s, sb, L + 1);
                uint64_t m, t;
                rate_of(sa, na, sb, nb, &m, &t);
                if (t > 0 && (bt == 0 || (unsigned __int128)m * bt > (unsigned __int128)bm * t)) {
                    bm = m; bt = t; bs = s;
                }
            }
            out_m[3] = bm; out_t[3] = bt;
            if (god_phase) *god_phase = bs;
        }
    }
    free(sa); free(sb);
    return or_levenshtein(a, L, b, L);
}
