/*
 * synth.c — seeded synthetic genomes and reads for the Genome-on-Diet hot path.
 *
 * This module is INPUT GENERATION ONLY.  It holds none of the method's arithmetic (no pattern,
 * no k-mer, no hash, no minimizer, no index): it produces ASCII sequences and read-simulation
 * truth (origin, strand, error counts).  Both the CPU oracle (oracle/) and the CUDA path
 * (paper_2211_08157_b200/) consume its output; neither imports the other.
 *
 * Workload recipes follow SURVEY.md §8(d) (which shapes them after the paper's data: human
 * genome ~50% repeats; GIAB Illumina/HiFi/ONT read statistics, Supp. Table 1)
 * and BASELINE.json `configs`.  The paper's real data (GRCh38, HG002) is not in the container;
 * these stand in for it.
 *
 * RNG: splitmix64.  Bulk i.i.d. bases are counter-based (block b of 32 bases = mix(key + b)),
 * so they are generated in parallel (OpenMP) and are identical for any thread count.  Sequential
 * procedures (duplication, repeat placement, read simulation) use a stateful splitmix64 stream
 * seeded per config; reads are simulated per read from a counter-derived sub-stream so that the
 * result does not depend on thread count either.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

static const uint8_t ACGT[4] = {'A', 'C', 'G', 'T'};

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

typedef struct { uint64_t s; } rng_t;
static inline uint64_t rng_next(rng_t* r) { r->s += 0x9E3779B97F4A7C15ull; uint64_t z = r->s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }
static inline double rng_unif(rng_t* r) { return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline uint64_t rng_below(rng_t* r, uint64_t n) { return n ? (uint64_t)(rng_unif(r) * (double)n) % n : 0; }
static inline double rng_normal(rng_t* r) {
    double u1 = rng_unif(r), u2 = rng_unif(r);
    if (u1 < 1e-300) u1 = 1e-300;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
static inline rng_t rng_make(uint64_t seed, uint64_t stream) { rng_t r; r.s = mix64(seed * 0x100000001B3ull ^ mix64(stream + 0x51ED)); return r; }

/* ---- i.i.d. uniform ACGT (counter-based, parallel) ---- */
void synth_iid(uint64_t seed, uint8_t* out, uint64_t L) {
    uint64_t key = mix64(seed ^ 0xA5A5A5A5DEADBEEFull);
    int64_t nblk = (int64_t)((L + 31) / 32);
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < nblk; b++) {
        uint64_t v = mix64(key + (uint64_t)b);
        uint64_t i0 = (uint64_t)b * 32;
        uint64_t n = L - i0 < 32 ? L - i0 : 32;
        for (uint64_t t = 0; t < n; t++) out[i0 + t] = ACGT[(v >> (2 * t)) & 3];
    }
}

static inline uint8_t other_base(rng_t* r, uint8_t b) {
    uint8_t c;
    do { c = ACGT[rng_next(r) & 3]; } while (c == b);
    return c;
}

/* ---- config 2-4 reference: i.i.d. + duplicated segments ----
 * Until the total copied length reaches dup_total: l ~ U{lmin..lmax}, src, dst ~ U; copy from the
 * i.i.d. snapshot with per-base substitution at rate d ~ U[dmin, dmax], overwriting dst. */
void synth_dup_segments(uint64_t seed, uint8_t* seq, uint64_t L, uint64_t dup_total,
                        uint32_t lmin, uint32_t lmax, double dmin, double dmax) {
    if (L <= lmax + 1) return;
    uint8_t* snap = (uint8_t*)malloc(L);
    memcpy(snap, seq, L);
    rng_t r = rng_make(seed, 7);
    uint64_t done = 0;
    while (done < dup_total) {
        uint64_t l = lmin + rng_below(&r, (uint64_t)(lmax - lmin + 1));
        uint64_t src = rng_below(&r, L - l);
        uint64_t dst = rng_below(&r, L - l);
        double d = dmin + (dmax - dmin) * rng_unif(&r);
        for (uint64_t t = 0; t < l; t++) {
            uint8_t b = snap[src + t];
            if (rng_unif(&r) < d) b = other_base(&r, b);
            seq[dst + t] = b;
        }
        done += l;
    }
    free(snap);
}

/* ---- config 5 reference: interspersed repeat families (a proposal) ----
 * n_fam consensus sequences, length log-uniform on [cmin, cmax]; family weight ∝ 1/rank (Zipf).
 * Copies: divergence d ~ U[dmin, dmax] applied as sub 0.9d, del 0.05d, ins 0.05d; placed at
 * uniform positions, overwriting, until >= cover_frac of the bases are covered by some copy. */
void synth_repeats(uint64_t seed, uint8_t* seq, uint64_t L, uint32_t n_fam, uint32_t cmin, uint32_t cmax,
                   double dmin, double dmax, double cover_frac) {
    if (L < 4ull * cmax) return;
    rng_t r = rng_make(seed, 11);
    uint32_t* clen = (uint32_t*)malloc(sizeof(uint32_t) * n_fam);
    uint8_t** cons = (uint8_t**)malloc(sizeof(uint8_t*) * n_fam);
    double* cdf = (double*)malloc(sizeof(double) * n_fam);
    double tot = 0;
    for (uint32_t f = 0; f < n_fam; f++) {
        double u = rng_unif(&r);
        clen[f] = (uint32_t)llround(exp(log((double)cmin) + u * (log((double)cmax) - log((double)cmin))));
        cons[f] = (uint8_t*)malloc(clen[f]);
        for (uint32_t t = 0; t < clen[f]; t++) cons[f][t] = ACGT[rng_next(&r) & 3];
        tot += 1.0 / (double)(f + 1);
        cdf[f] = tot;
    }
    uint64_t nwords = (L + 63) / 64;
    uint64_t* cov = (uint64_t*)calloc(nwords, sizeof(uint64_t));
    uint64_t covered = 0, target = (uint64_t)(cover_frac * (double)L);
    uint8_t* buf = (uint8_t*)malloc(2ull * cmax + 64);
    while (covered < target) {
        double u = rng_unif(&r) * tot;
        uint32_t lo = 0, hi = n_fam - 1;
        while (lo < hi) { uint32_t mid = (lo + hi) / 2; if (cdf[mid] < u) lo = mid + 1; else hi = mid; }
        uint32_t f = lo;
        double d = dmin + (dmax - dmin) * rng_unif(&r);
        double ps = 0.9 * d, pd = 0.05 * d, pi = 0.05 * d;
        uint64_t n = 0;
        for (uint32_t t = 0; t < clen[f] && n < 2ull * cmax; ) {
            double e = rng_unif(&r);
            if (e < pd) { t++; continue; }                                  /* deletion */
            if (e < pd + pi) { buf[n++] = ACGT[rng_next(&r) & 3]; continue; } /* insertion */
            uint8_t b = cons[f][t++];
            if (e < pd + pi + ps) b = other_base(&r, b);                    /* substitution */
            buf[n++] = b;
        }
        uint64_t dst = rng_below(&r, L - n);
        for (uint64_t t = 0; t < n; t++) {
            uint64_t i = dst + t;
            seq[i] = buf[t];
            uint64_t m = 1ull << (i & 63);
            if (!(cov[i >> 6] & m)) { cov[i >> 6] |= m; covered++; }
        }
    }
    free(buf); free(cov); free(cdf);
    for (uint32_t f = 0; f < n_fam; f++) free(cons[f]);
    free(cons); free(clen);
}

/* Fraction of bases lying in homopolymer runs of length >= 3 (used to rescale ONT indel rates). */
double synth_homopolymer_frac(const uint8_t* seq, uint64_t L) {
    uint64_t in = 0, i = 0;
    while (i < L) {
        uint64_t j = i + 1;
        while (j < L && seq[j] == seq[i]) j++;
        if (j - i >= 3) in += j - i;
        i = j;
    }
    return L ? (double)in / (double)L : 0.0;
}

static inline uint8_t comp(uint8_t b) {
    switch (b) { case 'A': return 'T'; case 'C': return 'G'; case 'G': return 'C'; case 'T': return 'A'; default: return 'N'; }
}

/*
 * Read simulation (SURVEY §8(d) "Read simulation").  For read r (sub-stream r of `seed`):
 *   length: fixed `len_fixed` if > 0, else round(lognormal(mu, sigma)) clamped to [lmin, lmax];
 *   start g ~ U[0, L - span_reserve) where span_reserve = ceil(1.3*len)+64 (fixed-length reads:
 *   g ~ U[0, L - start_margin]); strand ~ Bernoulli(1/2).
 *   Walk the reference from g: per emitted base draw one event: deletion (skip a reference base),
 *   insertion (emit a random base), substitution (emit another base) or match.  With hp_factor > 0
 *   indel probabilities are multiplied by hp_factor inside homopolymer runs >= 3 and by
 *   hp_rescale elsewhere (so genome-average rates hold).  Reverse reads are reverse-complemented
 *   after errors are applied.
 * Outputs: reads (concatenated ASCII), offsets[n+1], truth arrays (g, span, strand, nsub, nins, ndel).
 * Returns total bases written, or -1 if `cap` is too small (call with reads=NULL to size).
 */
int64_t synth_reads(uint64_t seed, const uint8_t* ref, uint64_t L, uint64_t n_reads,
                    uint32_t len_fixed, double mu, double sigma, uint32_t lmin, uint32_t lmax, uint32_t start_margin,
                    double p_sub, double p_ins, double p_del, double hp_factor, double hp_rescale,
                    uint8_t* reads, uint64_t cap, uint64_t* offsets,
                    uint64_t* t_g, uint32_t* t_span, uint8_t* t_strand, uint32_t* t_nsub, uint32_t* t_nins, uint32_t* t_ndel) {
    /* pass 1: lengths (counter-based per read) */
    uint64_t total = 0;
    for (uint64_t r = 0; r < n_reads; r++) {
        rng_t g = rng_make(seed, 1000003ull + r * 2);
        uint32_t len = len_fixed;
        if (!len) {
            double v = exp(mu + sigma * rng_normal(&g));
            long long lv = llround(v);
            if (lv < (long long)lmin) lv = lmin;
            if (lv > (long long)lmax) lv = lmax;
            len = (uint32_t)lv;
        }
        if (offsets) offsets[r] = total;
        total += len;
    }
    if (offsets) offsets[n_reads] = total;
    if (!reads) return (int64_t)total;
    if (total > cap) return -1;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t rr = 0; rr < (int64_t)n_reads; rr++) {
        uint64_t r = (uint64_t)rr;
        uint32_t len = (uint32_t)(offsets[r + 1] - offsets[r]);
        rng_t g = rng_make(seed, 1000003ull + r * 2 + 1);
        uint64_t reserve = len_fixed ? (uint64_t)start_margin : (uint64_t)(1.3 * len) + 64;
        if (reserve >= L) reserve = L - 1;
        uint64_t g0 = rng_below(&g, L - reserve);
        uint8_t strand = (uint8_t)(rng_next(&g) & 1);
        uint8_t* out = reads + offsets[r];
        uint64_t i = g0, n = 0;
        uint32_t ns = 0, ni = 0, nd = 0;
        while (n < len) {
            if (i >= L) { out[n++] = ACGT[rng_next(&g) & 3]; ni++; continue; } /* ran off the end: pad */
            double pi = p_ins, pd = p_del;
            if (hp_factor > 0) {
                int hp = 0;
                uint8_t b = ref[i];
                uint64_t a = i, z = i;
                while (a > 0 && ref[a - 1] == b && i - a < 3) a--;
                while (z + 1 < L && ref[z + 1] == b && z - i < 3) z++;
                hp = (z - a + 1) >= 3;
                double f = hp ? hp_factor : hp_rescale;
                pi *= f; pd *= f;
            }
            double e = rng_unif(&g);
            if (e < pd) { i++; nd++; continue; }
            if (e < pd + pi) { out[n++] = ACGT[rng_next(&g) & 3]; ni++; continue; }
            uint8_t b = ref[i++];
            if (e < pd + pi + p_sub) { b = other_base(&g, b); ns++; }
            out[n++] = b;
        }
        if (strand && len) {
            for (uint32_t a = 0, z = len - 1; a < z; a++, z--) { uint8_t t = out[a]; out[a] = comp(out[z]); out[z] = comp(t); }
            if (len & 1) out[len / 2] = comp(out[len / 2]);
        }
        t_g[r] = g0; t_span[r] = (uint32_t)(i - g0); t_strand[r] = strand;
        t_nsub[r] = ns; t_nins[r] = ni; t_ndel[r] = nd;
    }
    return (int64_t)total;
}

/* Sprinkle N runs (for edge-case inputs): n_runs runs of length U{1..max_run} at uniform positions. */
void synth_sprinkle_n(uint64_t seed, uint8_t* seq, uint64_t L, uint64_t n_runs, uint32_t max_run) {
    rng_t r = rng_make(seed, 13);
    for (uint64_t q = 0; q < n_runs && L; q++) {
        uint64_t at = rng_below(&r, L);
        uint64_t len = 1 + rng_below(&r, max_run);
        for (uint64_t t = 0; t < len && at + t < L; t++) seq[at + t] = 'N';
    }
}
