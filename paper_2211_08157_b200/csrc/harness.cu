// harness.cu — the seed-comparison harness of P:83-103 (section 2.1.1-2.1.2, Fig. 4; SURVEY §8(f)
// f4) on the GPU: for every (original, mutated) pair, the seed matching rate of four seed extractors
// and the Levenshtein distance.  Readings S1-S5: DESIGN.md §2 / include/god.h.
//
// k_harness_seeds: one CTA per pair.  Each extractor's seeds of the original are built in shared
// memory and sorted (bitonic); the mutated sequence's seeds are then looked up by binary search and
// counted (block reduction).  Minimizer selection (O6) is evaluated per k-mer start by scanning the
// windows that contain it (w <= 255, runs split at N, one partial window for a short run).
// k_levenshtein: one thread per pair, Myers' bit-parallel algorithm over 64-bit words (Hyyro's
// multi-word form, global distance: the top row's horizontal delta is +1).
#include <algorithm>

#include "internal.cuh"

namespace god {
namespace {

constexpr int HN_NT = 256;
constexpr uint32_t HN_MAXL = 4096;      // bases per sequence of a pair
constexpr uint64_t H_INVALID = ~0ull;   // start without a k-mer (N inside, or past a run)
constexpr uint64_t H_PAL = ~0ull - 1;   // palindromic k-mer: never in a window minimum (O6)

struct HArgs {
  const uint8_t* a;   // originals
  const uint8_t* b;   // mutated copies
  const uint64_t* off;
  Pattern pat;
  int32_t k, w;
  uint64_t* matches;  // [n][4]
  uint64_t* totals;   // [n][4]
  uint32_t* god_phase;
};

__device__ __forceinline__ uint64_t mask2(int k) { return k >= 32 ? ~0ull : ((1ull << (2 * k)) - 1); }

// H(canonical k-mer) of the k bases at seq[pos[0..k)] given by an index function
template <class F>
__device__ __forceinline__ uint64_t seed_hash(const uint8_t* seq, int x, F at) {
  uint64_t fwd = 0, rev = 0;
  for (int j = 0; j < x; j++) {
    const uint32_t c = base_code(seq[at(j)]);
    if (c > 3) return H_INVALID;
    fwd = (fwd << 2) | c;
    rev |= (uint64_t)(3u - c) << (2 * j);
  }
  if (fwd == rev) return H_PAL;
  return wang_hash(fwd < rev ? fwd : rev, mask2(x));
}

// Extract the seeds of one sequence into out[] (count in *cnt).  algo 0 all k-mers, 1 minimizers
// ('1', phase 0), 2 spaced (mask P[j mod p], span k), 3 Genome-on-Diet (pattern P, phase s).
// hbuf: scratch of L entries (per-start hashes for the minimizer extractors).
__device__ void extract_seeds(const HArgs& A, const uint8_t* seq, uint32_t L, int algo, uint32_t s, uint64_t* out,
                              uint32_t* cnt, uint64_t* hbuf) {
  const int k = A.k, w = A.w;
  if (threadIdx.x == 0) *cnt = 0;
  __syncthreads();
  if (algo == 0 || algo == 2) {
    int x = k;
    if (algo == 2) {
      x = 0;
      for (int j = 0; j < k; j++) x += (int)((A.pat.bits >> (j % A.pat.p)) & 1ull);
    }
    if (x > 0 && x <= 28 && L >= (uint32_t)k)
      for (uint32_t i = threadIdx.x; i + k <= L; i += HN_NT) {
        uint64_t h;
        if (algo == 0) {
          h = seed_hash(seq, k, [&](int j) { return i + j; });
          if (h == H_PAL) {  // a palindrome is still a k-mer seed: its canonical value is fwd
            uint64_t f = 0;
            for (int j = 0; j < k; j++) f = (f << 2) | base_code(seq[i + j]);
            h = wang_hash(f, mask2(k));
          }
        } else {
          // the included bases of window i: offsets j < k with P[j mod p] = 1
          uint64_t fwd = 0, rev = 0;
          int q = 0;
          bool ok = true;
          for (int j = 0; j < k && ok; j++) {
            if (!((A.pat.bits >> (j % A.pat.p)) & 1ull)) continue;
            const uint32_t c = base_code(seq[i + j]);
            if (c > 3) { ok = false; break; }
            fwd = (fwd << 2) | c;
            rev |= (uint64_t)(3u - c) << (2 * q);
            ++q;
          }
          h = ok ? wang_hash(fwd < rev ? fwd : rev, mask2(x)) : H_INVALID;
        }
        if (h != H_INVALID) out[atomicAdd(cnt, 1u)] = h;
      }
    __syncthreads();
    return;
  }
  // minimizer extractors: the patterned sequence (pattern '1' for algo 1)
  Pattern P = A.pat;
  if (algo == 1) {
    P.p = 1; P.x = 1; P.bits = 1; P.one[0] = 0;
  }
  const uint32_t nq = (uint32_t)included_count(P, L, s);
  const uint32_t nk = nq >= (uint32_t)k ? nq - k + 1 : 0;
  for (uint32_t q = threadIdx.x; q < nk; q += HN_NT)
    hbuf[q] = seed_hash(seq, k, [&](int j) { return (uint32_t)orig_of(P, q + j, s); });
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < nk; q += HN_NT) {
    const uint64_t hq = hbuf[q];
    if (hq >= H_PAL) continue;  // invalid or palindrome: never selected
    // run bounds around q, walked up to w - 1 starts each way
    uint32_t lo = q, hi = q;
    while (lo > 0 && q - lo < (uint32_t)(w - 1) && hbuf[lo - 1] != H_INVALID) --lo;
    while (hi + 1 < nk && hi - q < (uint32_t)(w - 1) && hbuf[hi + 1] != H_INVALID) ++hi;
    const bool lo_end = lo == 0 || hbuf[lo - 1] == H_INVALID;
    const bool hi_end = hi + 1 >= nk || hbuf[hi + 1] == H_INVALID;
    bool sel = false;
    if (lo_end && hi_end && hi - lo + 1 < (uint32_t)w) {  // a run shorter than w: one partial window
      uint64_t mn = H_PAL;
      for (uint32_t r = lo; r <= hi; r++) mn = min(mn, hbuf[r]);
      sel = hq == mn;
    } else {
      const uint32_t a0 = max(lo, q >= (uint32_t)(w - 1) ? q - (w - 1) : 0u);
      for (uint32_t a = a0; a <= q && a + w - 1 <= hi && !sel; a++) {
        uint64_t mn = H_PAL;
        for (uint32_t r = a; r < a + w; r++) mn = min(mn, hbuf[r]);
        sel = hq == mn;
      }
    }
    if (sel) out[atomicAdd(cnt, 1u)] = hq;
  }
  __syncthreads();
}

// ascending bitonic sort of v[0..n) (virtual +inf padding), n <= HN_MAXL
__device__ void block_sort(uint64_t* v, uint32_t n) {
  uint32_t lg = 0;
  while ((1u << lg) < n) ++lg;
  const uint32_t N2 = 1u << lg;
  for (uint32_t ls = 1; ls <= lg; ++ls) {
    const uint32_t lh = ls - 1, half = 1u << lh;
    for (uint32_t q = threadIdx.x; q < N2 / 2; q += HN_NT) {
      const uint32_t base = (q >> lh) << ls, off = q & (half - 1);
      const uint32_t i = base + off, j = base + 2 * half - 1 - off;
      if (j < n && v[j] < v[i]) { const uint64_t t = v[i]; v[i] = v[j]; v[j] = t; }
    }
    __syncthreads();
    for (int l = (int)lh - 1; l >= 0; --l) {
      const uint32_t st = 1u << l;
      for (uint32_t q = threadIdx.x; q < N2 / 2; q += HN_NT) {
        const uint32_t i = ((q >> l) << (l + 1)) | (q & (st - 1)), j = i + st;
        if (j < n && v[j] < v[i]) { const uint64_t t = v[i]; v[i] = v[j]; v[j] = t; }
      }
      __syncthreads();
    }
  }
}

// matches of m[0..nm) in the sorted sa[0..na) (block-wide count)
__device__ uint32_t count_matches(const uint64_t* sa, uint32_t na, const uint64_t* m, uint32_t nm, uint32_t* red) {
  uint32_t c = 0;
  for (uint32_t i = threadIdx.x; i < nm; i += HN_NT) {
    const uint64_t x = m[i];
    uint32_t lo = 0, hi = na;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (sa[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    c += lo < na && sa[lo] == x;
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (threadIdx.x == 0) *red = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(red, c);
  __syncthreads();
  return *red;
}

__global__ void __launch_bounds__(HN_NT) k_harness_seeds(HArgs A) {
  extern __shared__ __align__(16) unsigned char hsm[];
  uint64_t* sa = reinterpret_cast<uint64_t*>(hsm);  // original's seeds, sorted
  uint64_t* sb = sa + HN_MAXL;                      // mutated's seeds
  uint64_t* hb = sb + HN_MAXL;                      // per-start hashes
  __shared__ uint32_t na, nb, red;
  const uint32_t pr = blockIdx.x;
  const uint64_t o = A.off[pr];
  const uint32_t L = (uint32_t)(A.off[pr + 1] - o);
  const uint8_t* a = A.a + o;
  const uint8_t* b = A.b + o;
  for (int algo = 0; algo < 4; algo++) {
    extract_seeds(A, a, L, algo, 0, sa, &na, hb);
    block_sort(sa, na);
    const uint32_t nphase = algo == 3 ? A.pat.p : 1u;
    uint64_t bm = 0, bt = 0;
    uint32_t bs = 0;
    for (uint32_t s = 0; s < nphase; s++) {
      extract_seeds(A, b, L, algo, s, sb, &nb, hb);
      const uint32_t m = count_matches(sa, na, sb, nb, &red);
      const uint64_t t = nb;
      // S3: the best phase (a phase without seeds has no rate; ties -> smaller s)
      if (t > 0 && (bt == 0 || (unsigned __int128)m * bt > (unsigned __int128)bm * t)) { bm = m; bt = t; bs = s; }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      A.matches[4ull * pr + algo] = bm;
      A.totals[4ull * pr + algo] = bt;
      if (algo == 3) A.god_phase[pr] = bs;
    }
    __syncthreads();
  }
}

// S4: Levenshtein distance of (a, b), Myers' bit-vector algorithm, pattern = a in 64-bit words
constexpr int LV_WORDS = HN_MAXL / 64;
__global__ void k_levenshtein(const uint8_t* __restrict__ A, const uint8_t* __restrict__ B,
                              const uint64_t* __restrict__ off, uint32_t n, uint64_t* __restrict__ ed) {
  const uint32_t pr = blockIdx.x * blockDim.x + threadIdx.x;
  if (pr >= n) return;
  const uint64_t o = off[pr];
  const uint32_t m = (uint32_t)(off[pr + 1] - o);
  const uint8_t* a = A + o;
  const uint8_t* b = B + o;
  if (m == 0) { ed[pr] = 0; return; }
  const int nw = (int)((m + 63) / 64);
  // Peq[c]: positions of a equal to the byte "ACGT"[c] (bytes compare exactly, as in S4); a text
  // byte outside ACGT gets its match vector by a scan of a (rare: the harness inputs are ACGT)
  uint64_t Peq[4][LV_WORDS];
  uint64_t Pv[LV_WORDS], Mv[LV_WORDS];
  for (int c = 0; c < 4; c++)
    for (int q = 0; q < nw; q++) Peq[c][q] = 0;
  for (uint32_t i = 0; i < m; i++) {
    const uint8_t x = a[i];
    const int c = x == 'A' ? 0 : x == 'C' ? 1 : x == 'G' ? 2 : x == 'T' ? 3 : -1;
    if (c >= 0) Peq[c][i >> 6] |= 1ull << (i & 63);
  }
  for (int q = 0; q < nw; q++) { Pv[q] = ~0ull; Mv[q] = 0; }
  const int last = nw - 1;
  const uint64_t hbit = 1ull << ((m - 1) & 63);
  uint32_t score = m;
  for (uint32_t j = 0; j < m; j++) {
    const uint8_t y = b[j];
    const int c = y == 'A' ? 0 : y == 'C' ? 1 : y == 'G' ? 2 : y == 'T' ? 3 : -1;
    uint64_t add_c = 0, ph_c = 1, mh_c = 0;  // global distance: top-row horizontal delta +1
    for (int q = 0; q < nw; q++) {
      uint64_t eq;
      if (c >= 0) {
        eq = Peq[c][q];
      } else {
        eq = 0;
        for (uint32_t i = (uint32_t)q * 64; i < m && i < (uint32_t)q * 64 + 64; i++)
          eq |= (uint64_t)(a[i] == y) << (i & 63);
      }
      const uint64_t pv = Pv[q], mv = Mv[q];
      const uint64_t xv = eq | mv;
      const uint64_t x = eq & pv;
      const uint64_t s1 = x + pv;
      const uint64_t s2 = s1 + add_c;
      add_c = (uint64_t)(s1 < x) | (uint64_t)(s2 < s1);
      const uint64_t xh = (s2 ^ pv) | eq;
      const uint64_t ph = mv | ~(xh | pv);
      const uint64_t mh = pv & xh;
      if (q == last) {
        if (ph & hbit) ++score;
        if (mh & hbit) --score;
      }
      const uint64_t nph = (ph << 1) | ph_c, nmh = (mh << 1) | mh_c;
      ph_c = ph >> 63;
      mh_c = mh >> 63;
      Pv[q] = nmh | ~(xv | nph);
      Mv[q] = nph & xv;
    }
  }
  ed[pr] = score;
}

// P:87-89 (reading S5): the rate threshold of edit threshold E is the minimum rate over the pairs with
// edit distance <= E; accepted = pairs whose rate >= it (pairs without seeds have no rate).  One CTA
// per (E, extractor): a block minimum of the fractions m/t (exact, by cross-multiplication), then a
// block count.
__global__ void __launch_bounds__(HN_NT) k_harness_accept(const uint64_t* __restrict__ ed,
                                                          const uint64_t* __restrict__ mm,
                                                          const uint64_t* __restrict__ tt, uint32_t n,
                                                          const uint64_t* __restrict__ E, uint64_t* __restrict__ acc) {
  __shared__ uint64_t s_m[HN_NT / 32], s_t[HN_NT / 32];
  __shared__ unsigned long long s_cnt;
  const uint32_t e = blockIdx.x >> 2, a = blockIdx.x & 3u;
  const uint64_t th = E[e];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto less = [](uint64_t m1, uint64_t t1, uint64_t m2, uint64_t t2) {  // m1/t1 < m2/t2 (t2 = 0: +inf)
    if (t2 == 0) return t1 != 0;
    if (t1 == 0) return false;
    return (unsigned __int128)m1 * t2 < (unsigned __int128)m2 * t1;
  };
  uint64_t bm = 0, bt = 0;  // running minimum (bt = 0: none yet)
  for (uint32_t i = threadIdx.x; i < n; i += HN_NT) {
    const uint64_t t = tt[4ull * i + a], m = mm[4ull * i + a];
    if (t && ed[i] <= th && less(m, t, bm, bt)) { bm = m; bt = t; }
  }
  for (int o = 16; o; o >>= 1) {
    const uint64_t om = __shfl_xor_sync(0xffffffffu, bm, o), ot = __shfl_xor_sync(0xffffffffu, bt, o);
    if (less(om, ot, bm, bt)) { bm = om; bt = ot; }
  }
  if (lane == 0) { s_m[wid] = bm; s_t[wid] = bt; }
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  bm = s_m[0]; bt = s_t[0];
  for (int q = 1; q < HN_NT / 32; q++)
    if (less(s_m[q], s_t[q], bm, bt)) { bm = s_m[q]; bt = s_t[q]; }
  unsigned long long c = 0;
  if (bt)
    for (uint32_t i = threadIdx.x; i < n; i += HN_NT) {
      const uint64_t t = tt[4ull * i + a], m = mm[4ull * i + a];
      c += t && !less(m, t, bm, bt);
    }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) atomicAdd(&s_cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) acc[4ull * e + a] = s_cnt;
}

}  // namespace

void harness_accepted(const uint64_t* ed, const uint64_t* mm, const uint64_t* tt, uint32_t n, const uint64_t* E,
                      uint32_t nE, uint64_t* acc, cudaStream_t st) {
  if (!nE) return;
  GOD_LAUNCH("k_harness_accept", k_harness_accept, 4u * nE, HN_NT, 0, st, ed, mm, tt, n, E, acc);
}

void seed_harness(const Params& P, const uint8_t* a, const uint8_t* b, const uint64_t* off, uint32_t n,
                  uint64_t* ed, uint64_t* matches, uint64_t* totals, uint32_t* god_phase, cudaStream_t st) {
  if (!n) return;
  HArgs A;
  A.a = a;
  A.b = b;
  A.off = off;
  A.pat = P.pat;
  A.k = P.k;
  A.w = P.w;
  A.matches = matches;
  A.totals = totals;
  A.god_phase = god_phase;
  const size_t sm = 3 * HN_MAXL * sizeof(uint64_t);
  static DeviceOnce attr_once;
  attr_once.run([&] { GOD_CUDA(cudaFuncSetAttribute(k_harness_seeds, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); });
  GOD_LAUNCH("k_harness_seeds", k_harness_seeds, n, HN_NT, sm, st, A);
  GOD_LAUNCH("k_levenshtein", k_levenshtein, grid_for(n, 64), 64, 0, st, a, b, off, n, ed);
}

uint32_t harness_max_len() { return HN_MAXL; }

}  // namespace god
