// index.cu — stage 3: the seed index (P:286 (3)).
//
// "We do not directly insert minimizer information ... Instead, we append the minimizer
// information to an array and sort the array after collecting information on all minimizers and
// then add it to the hash table".  B200 version:
//   K1  fused sparsify+minimizer extraction of the reference (extract2.cu / extract.cu) -> records
//       (hash | strand << 63, pos) in position order
//   K2  sort to (hash, pos) order.  2k >= 36: data-sized monotone bins over the top 12 hash bits
//       (k_seg_hist / k_seg_table / k_seg_assign), two stable 9-bit LSD passes over the bin number
//       (k_rs_hist, scan, k_rs_scatter2), then a per-bin SMEM sort on (low hash, pos) (k_bin_sort;
//       oversized bins: k_bucket_sort_big).  Otherwise a stable 8-bit LSD over all 2k hash bits.
//   K3  runs of equal hashes = distinct hashes: fused into the bin sorts (run lengths in the key's
//       free bits + count histogram); k_runs on the full-LSD path
//   K4  cutoff tau on device (reading O7): count histogram (small counts) + radix select
//       over the rare large counts; tau = (m+1)-th largest count, m = floor(n*num/den)
//   K5  kept entries in one ordered pass (k_keep_write: ballots + decoupled look-back), which also
//       marks the first entry of every non-empty directory slot (K6a)
//   K6  directory: data-sized slot map (or top-B-bit prefix); one right-to-left suffix-min pass
//       fills the empty slots and writes the 32-B slot records (k_dir_suffix_min, K6b + K6c)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>
#include "internal.cuh"

namespace god {

namespace {
constexpr int RS_NT = 256;
#ifndef RS_IPT_DEF
#define RS_IPT_DEF 16
#endif
constexpr int RS_IPT = RS_IPT_DEF;
constexpr int RS_TILE = RS_NT * RS_IPT;
constexpr int RS_BITS = 8;
constexpr int RS_BINS = 1 << RS_BITS;
constexpr uint64_t HASH_BITS_MASK = (1ull << 63) - 1;
#ifndef RS2_NT_DEF
#define RS2_NT_DEF 512
#endif
constexpr int RS2_NT = RS2_NT_DEF, RS2_IPT = RS_TILE / RS2_NT;  // scatter: 8 items per thread
// dynamic SMEM of the scatter: the staged tile (keys, values) + the digit counter rows
constexpr int rs_dyn_smem(int rb, bool stable) {
  return RS_TILE * (int)(sizeof(uint64_t) + sizeof(uint32_t)) + (stable ? RS2_NT / 32 : 1) * (1 << rb) * 4;
}
// tiles per histogram column of the bin-sort passes: one CTA can scatter RS_GROUP consecutive tiles,
// carrying its digit offsets from tile to tile, so that the tile histograms and their scan are
// RS_GROUP times smaller.  Measured (human, both passes): the scan falls 0.49 -> 0.27 / 0.15 / 0.09 ms
// at 2 / 4 / 8 but the scatter itself slows 4.61 -> 5.03 / 6.07 / 6.41 ms (a digit's 128-B output
// line is then completed by one CTA over several tiles instead of by neighbouring CTAs at once), so 1.
#ifndef RS_GROUP_DEF
#define RS_GROUP_DEF 1
#endif
constexpr int RS_GROUP = RS_GROUP_DEF;

// Lanes of the warp holding the same digit as this lane (digit < 2^NBITS; invalid lanes carry
// d = 2^NBITS and only match each other): one ballot per digit bit.  Measured much cheaper than
// __match_any_sync, whose long latency stalled the ranking loops.
template <int NBITS>
__device__ __forceinline__ uint32_t warp_peers(uint32_t d) {
  uint32_t peers = 0xFFFFFFFFu;
#pragma unroll
  for (int b = 0; b <= NBITS; b++) {
    const bool bit = (d >> b) & 1u;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

// bulk L2 prefetch of [p, p + bytes) (16-B aligned, whole 16-B units)
__device__ __forceinline__ void l2_prefetch_range(const void* p, uint64_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~(uintptr_t)15;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a)) : "memory");
}

template <int RB, int G = 1>
__global__ void __launch_bounds__(RS_NT) k_rs_hist(const uint64_t* __restrict__ keys, uint64_t n, int shift,
                                                   uint32_t dmask, uint32_t* hist, uint32_t ntiles) {
  __shared__ uint32_t h[(1 << RB)];
  for (int i = threadIdx.x; i < (1 << RB); i += RS_NT) h[i] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * RS_TILE * G;
  if (base + (uint64_t)RS_TILE * G <= n) {  // a full tile: two keys per 128-bit load, all loads in flight
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys + base);
    ulonglong2 kv[RS_IPT / 2];
    for (int g = 0; g < G; g++) {
#pragma unroll
      for (int r = 0; r < RS_IPT / 2; r++) kv[r] = __ldcs(k2 + (size_t)g * (RS_TILE / 2) + r * RS_NT + threadIdx.x);
#pragma unroll
      for (int r = 0; r < RS_IPT / 2; r++) {
        atomicAdd(&h[(uint32_t)((kv[r].x & HASH_BITS_MASK) >> shift) & dmask], 1u);
        atomicAdd(&h[(uint32_t)((kv[r].y & HASH_BITS_MASK) >> shift) & dmask], 1u);
      }
    }
  } else {
#pragma unroll 4
    for (int r = 0; r < RS_IPT * G; r++) {
      uint64_t i = base + (uint64_t)r * RS_NT + threadIdx.x;
      if (i < n) atomicAdd(&h[(uint32_t)((keys[i] & HASH_BITS_MASK) >> shift) & dmask], 1u);
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < (1 << RB); d += RS_NT) hist[(uint64_t)d * ntiles + blockIdx.x] = h[d];
}

// Stable scatter, warp-striped ranking: warp w owns items [w*256, w*256+256) of the tile, item j of
// lane l is w*256 + 32 j + l, so (warp, j, lane) order is index order.  Ranks come from match_any
// plus per-warp digit counters (no block barrier per item round).  STABLE = false (the first LSD
// pass over records that arrive in any order anyway: K1's tile-order output): one SMEM atomic per
// item on the warp's digit counter gives its rank (the ballot peer masks were ~36% of the pass).
#ifndef RS_UNSTABLE_MINB
#define RS_UNSTABLE_MINB 2
#endif
#ifndef RS_MINB_DEF
#define RS_MINB_DEF 2
#endif
template <int RB, bool STABLE, int G>
__global__ void __launch_bounds__(RS2_NT, STABLE ? RS_MINB_DEF : RS_UNSTABLE_MINB) k_rs_scatter2(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                       uint64_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                       uint64_t n, int shift, uint32_t dmask,
                                                       const uint64_t* __restrict__ goff, uint32_t ntiles,
                                                       const uint2* __restrict__ table, int L, uint32_t ahead) {
  // STABLE: one counter row per warp (ranks in (warp, item, lane) order).  Unstable: one row for the
  // CTA — the atomic's return value is the item's rank in its digit, no prefix over warps
  constexpr int NROW = STABLE ? RS2_NT / 32 : 1;
  extern __shared__ __align__(16) unsigned char rs_dyn[];
  uint32_t (*wcnt)[1 << RB] = reinterpret_cast<uint32_t (*)[1 << RB]>(rs_dyn + (size_t)RS_TILE * 12);
  __shared__ uint32_t dstart[(1 << RB) + 1];
  __shared__ uint32_t wsum[(1 << RB) / 32];
  __shared__ uint64_t s_goff[1 << RB];
  uint64_t* sk = reinterpret_cast<uint64_t*>(rs_dyn);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + RS_TILE);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // ntiles = histogram columns = CTAs; CTA c scatters tiles c G .. c G + G - 1 in order
  for (int d = tid; d < (1 << RB); d += RS2_NT) s_goff[d] = goff[(uint64_t)d * ntiles + blockIdx.x];
  for (int sub = 0; sub < G; sub++) {
  const uint64_t tile = (uint64_t)blockIdx.x * G + sub;
  if (tile * RS_TILE >= n) break;
  if (tid == 0) {  // into L2: this CTA's next tile, or (last tile) the first tile of the CTA launched after the resident wave
    const uint64_t t2 = sub + 1 < G ? tile + 1 : ((uint64_t)blockIdx.x + ahead) * G;  // ahead = resident CTAs (2 per SM)
    if (t2 * RS_TILE < n) {
      const uint64_t c2 = min((uint64_t)RS_TILE, n - t2 * RS_TILE);
      l2_prefetch_range(kin + t2 * RS_TILE, c2 * sizeof(uint64_t));
      l2_prefetch_range(vin + t2 * RS_TILE, c2 * sizeof(uint32_t));
    }
  }
  for (int i = tid; i < NROW * (1 << RB) / 4; i += RS2_NT) reinterpret_cast<uint4*>(&wcnt[0][0])[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const uint64_t base = tile * RS_TILE + (uint64_t)wid * (32 * RS2_IPT);
  const uint32_t lt = (1u << lane) - 1;
  uint64_t key[RS2_IPT];
  uint32_t val[RS2_IPT];
  uint32_t rk[RS2_IPT];
#pragma unroll
  for (int j = 0; j < RS2_IPT; j++) {  // all loads in flight before the ranking
    const uint64_t i = base + (uint64_t)j * 32 + lane;
    const bool ok = i < n;
    key[j] = ok ? __ldcs(kin + i) : 0;
    val[j] = ok ? __ldcs(vin + i) : 0;
  }
  if (table) {  // first bin-sort pass: the key gets its data-sized bin (k_seg_assign's rule) here
    const uint64_t lmask = (1ull << L) - 1;
#pragma unroll
    for (int j = 0; j < RS2_IPT; j++) {
      const uint64_t h = key[j] & HASH_BITS_MASK;
      const uint2 t = __ldg(table + (h >> L));
      const uint64_t b = t.x + (((h & lmask) * t.y) >> L);
      key[j] |= b << shift;
    }
  }
#pragma unroll
  for (int j = 0; j < RS2_IPT; j++) {
    const uint64_t i = base + (uint64_t)j * 32 + lane;
    const bool ok = i < n;
    const uint32_t d = ok ? ((uint32_t)((key[j] & HASH_BITS_MASK) >> shift) & dmask) : (1 << RB);
    if constexpr (!STABLE) {
      rk[j] = ok ? atomicAdd(&wcnt[0][d], 1u) : 0u;
      continue;
    }
    const uint32_t peers = warp_peers<RB>(d);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (lane == leader && ok) {
      old = wcnt[wid][d];
      wcnt[wid][d] = old + __popc(peers);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rk[j] = old + __popc(peers & lt);
  }
  __syncthreads();
  // digit tid (< 256): exclusive prefix over warps, tile total
  uint32_t acc = 0;
  if (tid < (1 << RB)) {
    if constexpr (STABLE) {
#pragma unroll
      for (int q = 0; q < RS2_NT / 32; q++) {
        const uint32_t c = wcnt[q][tid];
        wcnt[q][tid] = acc;
        acc += c;
      }
    } else {
      acc = wcnt[0][tid];
    }
  }
  // exclusive scan of the tile totals over the 256 digits (warps 0..7)
  uint32_t incl = acc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31 && tid < (1 << RB)) wsum[wid] = incl;
  __syncthreads();
  if (tid < (1 << RB)) {
    uint32_t before = 0;
#pragma unroll
    for (int q = 0; q < (1 << RB) / 32; q++) before += q < wid ? wsum[q] : 0u;
    dstart[tid] = before + incl - acc;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < RS2_IPT; j++) {
    const uint64_t i = base + (uint64_t)j * 32 + lane;
    if (i < n) {
      const uint32_t d = (uint32_t)((key[j] & HASH_BITS_MASK) >> shift) & dmask;
      const uint32_t slot = dstart[d] + (STABLE ? wcnt[wid][d] : 0u) + rk[j];
      sk[slot] = key[j];
      sv[slot] = val[j];
    }
  }
  __syncthreads();
  const uint32_t cnt = (uint32_t)min((uint64_t)RS_TILE, n - tile * RS_TILE);
  for (uint32_t s = tid; s < cnt; s += RS2_NT) {
    const uint64_t kk = sk[s];
    const uint32_t d = (uint32_t)((kk & HASH_BITS_MASK) >> shift) & dmask;
    const uint64_t dst = s_goff[d] + (s - dstart[d]);
    GOD_DCHECK(dst < n, "LSD scatter destination");
    kout[dst] = kk;
    vout[dst] = sv[s];
  }
  if constexpr (G > 1) {  // the next tile of this CTA continues each digit's run
    __syncthreads();
    if (tid < (1 << RB)) s_goff[tid] += acc;
    // (the next round's first barrier orders this against its readers)
  }
  }
}

// ---- bin sort (2k >= 36).  Minimizer hashes are skewed toward small values (each is the minimum
// of a window: density ~ (w+1)(1-u)^w at u = h / 4^k), so fixed-width hash buckets differ ~10x in
// size.  Instead each record gets a monotone bin number b(h) sized from the data: the top SEG_BITS
// hash bits select a segment t, which is cut into bins_t = ceil(c_t / BIN_TARGET) equal-width bins,
//   b(h) = base_t + floor(low(h) * bins_t / 2^L),   L = 2k - SEG_BITS, base = exclusive scan of bins_t,
// so bins hold ~BIN_TARGET records, b is non-decreasing in h, and a bin never spans two segments.
// b is stored in the free key bits above the hash; two stable 9-bit LSD passes order the records by
// b, then one CTA per bin sorts it in SMEM on the packed u64
//   v = low(h) << 33 | pos << 1 | strand       (integer order = (hash, pos) order; L <= 30),
// skipping digits that are constant across the bin.  Bins above BS_CAP (hashes with thousands of
// occurrences) go to a chunked global-memory kernel.
// CTA size of the per-bin kernels.  The bin capacity, the bin target and the SMEM tables scale with it,
// so 256 threads run 4 CTAs per SM where 512 run 2: more independent barrier domains per SM (the
// per-bin sort is a chain of ~12 block barriers).
#ifndef BS_NT_DEF
#define BS_NT_DEF 256
#endif
constexpr int BS_NT = BS_NT_DEF;
constexpr int BS_NW = BS_NT / 32;
constexpr int BS_IPT = 8;
constexpr int BS_CAP = BS_NT * BS_IPT;            // records of a bin held in SMEM (x2 buffers)
constexpr int BS_MSD_BITS = BS_NT == 512 ? 12 : BS_NT == 256 ? 11 : 10;  // log2(BS_CAP)
static_assert((1 << BS_MSD_BITS) == BS_CAP, "MSD placement: one bucket per record slot, 8 counters per thread");
constexpr uint32_t SMALL_BINS = BS_CAP;           // run-count histogram in SMEM (larger counts: a list)
constexpr int BS_SMEM = 2 * BS_CAP * 8 + (int)SMALL_BINS * 4;
constexpr uint32_t S_MAX = BS_CAP / 2;            // directory slots per bin (k_bin_build: first[S + 1] in SMEM)
constexpr int BB_SMEM = BS_SMEM + (S_MAX + 1) * 4;
constexpr int BS_MINB = 1024 / BS_NT;             // resident CTAs per SM the kernels are sized for
constexpr int BS_BIG_MINB = BS_NT >= 512 ? 1 : 2;  // ... of k_bucket_sort_big (138 registers unconstrained)
constexpr int SEG_BITS = 12;

// Run statistics (K3) produced by the sort kernels when they can: count histogram (small counts) +
// list of large counts, number of distinct hashes.  (Per-record run lengths are not stored: the
// kept-entry pass re-derives each record's run extent from its neighbours, capped at tau + 1.)
struct RunOut {
  uint32_t* hist_small;
  uint32_t* large;
  uint32_t* n_large;
  unsigned long long* n_distinct;
};

// one run [i, i + L) of equal hashes found by a thread: record it (SMEM histogram `h`; runs of
// length 1, the vast majority, are counted in a register: one SMEM counter would serialise them)
struct RunAcc {
  uint32_t nd = 0, ones = 0;
};
__device__ __forceinline__ void run_emit(const RunOut& ro, uint32_t* h, uint64_t L, RunAcc& acc) {
  const uint32_t c = L < 0xFFFFFFFFull ? (uint32_t)L : 0xFFFFFFFFu;
  if (c == 1) ++acc.ones;
  else if (c < SMALL_BINS) atomicAdd(&h[c], 1u);
  else ro.large[atomicAdd(ro.n_large, 1u)] = c;
  ++acc.nd;
}
__device__ __forceinline__ void run_flush(const RunOut& ro, uint32_t* h, RunAcc acc) {
  for (int o = 16; o; o >>= 1) {
    acc.nd += __shfl_xor_sync(0xffffffffu, acc.nd, o);
    acc.ones += __shfl_xor_sync(0xffffffffu, acc.ones, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (acc.nd) atomicAdd(ro.n_distinct, (unsigned long long)acc.nd);
    if (acc.ones) atomicAdd(&h[1], acc.ones);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (int)SMALL_BINS; i += blockDim.x)
    if (h[i]) atomicAdd(&ro.hist_small[i], h[i]);
}
// records next to i (excluding i) in one direction with hash hv, capped at lim: galloping then
// binary search
__device__ __forceinline__ uint64_t run_side(const uint64_t* __restrict__ k, uint64_t n, uint64_t i, uint64_t hv,
                                             uint64_t lim, bool fwd, uint64_t hm) {
  auto same = [&](uint64_t d) -> bool {
    if (fwd) return i + d < n && (k[i + d] & hm) == hv;
    return d <= i && (k[i - d] & hm) == hv;
  };
  uint64_t good = 0, d = 1;
  while (d <= lim && same(d)) { good = d; d <<= 1; }
  uint64_t bad = d <= lim ? d : lim + 1;
  while (bad - good > 1) {
    const uint64_t mid = good + (bad - good) / 2;
    if (same(mid)) good = mid;
    else bad = mid;
  }
  return good;
}

// length of the run of hash hv containing record i: exact if <= cap, else some value > cap
__device__ __forceinline__ uint64_t run_len_capped(const uint64_t* __restrict__ k, uint64_t n, uint64_t i, uint64_t hv,
                                                   uint64_t cap, uint64_t hm) {
  const uint64_t lim = cap + 1;
  return 1 + run_side(k, n, i, hv, lim, false, hm) + run_side(k, n, i, hv, lim, true, hm);
}

constexpr uint32_t BIN_TARGET = BS_CAP / 4 * 3;  // measured at BS_CAP = 4096: 2048 13.9 ms, 2560 13.7, 3072 13.6, 3584 14.5 (stage 3, human)
constexpr int BIN_DIGIT = 9;                      // LSD digit over b
constexpr int BIN_RANK_MAX = 1024;                // buckets up to this size: ranked by counting, else LSD
static_assert(RS_BINS * BS_NW == BS_NT * 8, "block scan assumes 8 counters per thread");

// records per top-SEG_BITS segment over a sample: one block of 32 consecutive records (256 B, one
// coalesced warp load) out of every `stride` blocks.  K1 emits records in tile (position) order, so a
// block's hashes are independent of its index and the sample is uniform.  The counts only size the
// bins (every segment gets >= 1 bin, so a sampled count never lets a bin span two segments).
__global__ void k_seg_hist(const uint64_t* __restrict__ k, uint64_t n, int L, uint32_t* segc, uint32_t stride) {
  __shared__ uint32_t h[1 << SEG_BITS];
  for (int i = threadIdx.x; i < (1 << SEG_BITS); i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32; b * 32 * stride < n; b += nwarps) {
    const uint64_t i = b * 32 * stride + lane;
    if (i < n) atomicAdd(&h[(uint32_t)((k[i] & HASH_BITS_MASK) >> L)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (1 << SEG_BITS); i += blockDim.x)
    if (h[i]) atomicAdd(&segc[i], h[i]);
}

__global__ void __launch_bounds__(1024) k_seg_table(const uint32_t* __restrict__ segc, uint32_t target, uint2* table,
                                                    uint32_t* n_bins, uint32_t scale = 1, uint32_t min_bins = 0) {
  constexpr int PER = (1 << SEG_BITS) / 1024;
  __shared__ uint32_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t nb[PER], tsum = 0;
#pragma unroll
  for (int q = 0; q < PER; q++) {
    const uint32_t c = segc[tid * PER + q];
    nb[q] = max(min_bins, (uint32_t)(((uint64_t)c * scale + target - 1) / target));
    tsum += nb[q];
  }
  uint32_t incl = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  uint32_t before = incl - tsum;
  for (int q = 0; q < wid; q++) before += wsum[q];
#pragma unroll
  for (int q = 0; q < PER; q++) {
    table[tid * PER + q] = make_uint2(before, nb[q]);
    before += nb[q];
  }
  if (tid == 1023) *n_bins = before;
}

// directory slot map aligned with the bins: S slots per bin (k_bin_build writes its bin's slots)
__global__ void k_seg_slots(const uint2* __restrict__ table, uint32_t S, uint2* seg) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < (1u << SEG_BITS)) seg[t] = make_uint2(table[t].x * S, table[t].y * S);
}

// b(h) into the free key bits above the hash, one RS_TILE tile per CTA; also the tile histogram
// of the first LSD digit of b (the k_rs_hist of the first pass, fused)
__global__ void __launch_bounds__(RS_NT) k_seg_assign(uint64_t* __restrict__ k, uint64_t n, int L, int hbits,
                                                      const uint2* __restrict__ table, uint32_t dmask,
                                                      uint32_t* hist, uint32_t ntiles, int write_keys) {
  __shared__ uint32_t hh[1 << BIN_DIGIT];
  for (int i = threadIdx.x; i < (1 << BIN_DIGIT); i += RS_NT) hh[i] = 0;
  __syncthreads();
  const uint64_t lmask = (1ull << L) - 1;
  const uint64_t base = (uint64_t)blockIdx.x * RS_TILE * RS_GROUP;
  auto one = [&](uint64_t i, uint64_t kk) {
    const uint64_t h = kk & HASH_BITS_MASK;
    const uint2 t = __ldg(table + (h >> L));
    const uint64_t b = t.x + (((h & lmask) * t.y) >> L);
    if (write_keys) k[i] = kk | (b << hbits);
    atomicAdd(&hh[(uint32_t)b & dmask], 1u);
  };
  if (base + (uint64_t)RS_TILE * RS_GROUP <= n) {  // a full tile: two keys per 128-bit load, all loads in flight
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(k + base);
    ulonglong2 kv[RS_IPT / 2];
    for (int g = 0; g < RS_GROUP; g++) {
#pragma unroll
      for (int r = 0; r < RS_IPT / 2; r++) kv[r] = __ldcs(k2 + (size_t)g * (RS_TILE / 2) + r * RS_NT + threadIdx.x);
#pragma unroll
      for (int r = 0; r < RS_IPT / 2; r++) {
        const uint64_t i = base + (uint64_t)g * RS_TILE + 2 * ((uint64_t)r * RS_NT + threadIdx.x);
        one(i, kv[r].x);
        one(i + 1, kv[r].y);
      }
    }
  } else {
#pragma unroll 4
    for (int r = 0; r < RS_IPT * RS_GROUP; r++) {
      const uint64_t i = base + (uint64_t)r * RS_NT + threadIdx.x;
      if (i < n) one(i, k[i]);
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < (1 << BIN_DIGIT); d += RS_NT) hist[(uint64_t)d * ntiles + blockIdx.x] = hh[d];
}

__global__ void k_bucket_bounds(const uint64_t* __restrict__ k, uint64_t n, int lo_bits, uint32_t nb, uint64_t* bstart) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
    uint64_t lo = 0, hi = n;  // first record whose bits above lo_bits are >= b
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (((k[mid] & HASH_BITS_MASK) >> lo_bits) < b) lo = mid + 1;
      else hi = mid;
    }
    bstart[b] = lo;
  }
}

// One CTA-wide LSD pass: the n <= BS_CAP values v[] (thread item j = warp-striped index
// wid * 32 * BS_IPT + j * 32 + lane) are scattered into dst stably by bits [shift, shift + bits).
// cnt is digit-major with a padded row (cnt[d * CNT_LD + w], CNT_LD = BS_NW + 1, so that the lanes of
// a warp touching different digits hit different banks); on return cnt[d * CNT_LD] is the start of
// digit d in dst.  Ends with a barrier (dst complete, cnt readable).
constexpr int CNT_LD = BS_NW + 1;
constexpr int CNT_WORDS = RS_BINS * CNT_LD;
__device__ __forceinline__ void cta_rank_scatter(const uint64_t (&v)[BS_IPT], int n, int shift, uint32_t dmask,
                                                 uint64_t* dst, uint32_t* cnt, uint32_t* wsum) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < CNT_WORDS; i += BS_NT) cnt[i] = 0;
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1;
  uint32_t rk[BS_IPT];
#pragma unroll
  for (int j = 0; j < BS_IPT; j++) {
    const int i = wid * (32 * BS_IPT) + j * 32 + lane;
    const bool ok = i < n;
    const uint32_t d = ok ? (uint32_t)(v[j] >> shift) & dmask : RS_BINS;
    const uint32_t peers = warp_peers<RS_BITS>(d);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (lane == leader && ok) {
      old = cnt[d * CNT_LD + wid];
      cnt[d * CNT_LD + wid] = old + __popc(peers);
    }
    rk[j] = __shfl_sync(0xffffffffu, old, leader) + __popc(peers & lt);
  }
  __syncthreads();
  // block-wide exclusive scan of the 4096 counters in (digit, warp) order, 8 per thread
  constexpr int TPD = BS_NW / 8;  // threads per digit row (8 warp counters each)
  static_assert(BS_NW % 8 == 0 && RS_BINS * TPD == BS_NT, "one thread per 8 counters");
  uint32_t* row = cnt + (tid / TPD) * CNT_LD + (tid % TPD) * 8;
  uint32_t x[8];
  uint32_t tsum = 0;
#pragma unroll
  for (int q = 0; q < 8; q++) { const uint32_t c = row[q]; x[q] = tsum; tsum += c; }
  uint32_t incl = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  uint32_t before = incl - tsum;
#pragma unroll
  for (int q = 0; q < BS_NW; q++) before += q < wid ? wsum[q] : 0u;
#pragma unroll
  for (int q = 0; q < 8; q++) row[q] = x[q] + before;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < BS_IPT; j++) {
    const int i = wid * (32 * BS_IPT) + j * 32 + lane;
    if (i < n) {
      const uint32_t d = (uint32_t)(v[j] >> shift) & dmask;
      dst[cnt[d * CNT_LD + wid] + rk[j]] = v[j];
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void cta_load_striped(const uint64_t* src, int n, uint64_t (&v)[BS_IPT]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < BS_IPT; j++) {
    const int i = wid * (32 * BS_IPT) + j * 32 + lane;
    v[j] = i < n ? src[i] : 0;
  }
}

__global__ void __launch_bounds__(BS_NT, BS_MINB) k_bin_sort(uint64_t* __restrict__ k, uint32_t* __restrict__ v,
                                                       const uint64_t* __restrict__ bstart,
                                                       const uint32_t* __restrict__ n_bins, int L, int hbits,
                                                       uint32_t* big, uint32_t* n_big, RunOut ro) {
  extern __shared__ __align__(16) unsigned char bs_smem[];
  uint64_t* A = reinterpret_cast<uint64_t*>(bs_smem);
  uint64_t* Bf = A + BS_CAP;
  uint32_t* rh = reinterpret_cast<uint32_t*>(Bf + BS_CAP);  // [SMALL_BINS] run-count histogram
  for (int i = threadIdx.x; i < (int)SMALL_BINS; i += BS_NT) rh[i] = 0;
  __syncthreads();
  RunAcc racc;
  __shared__ __align__(16) uint32_t cnt[CNT_WORDS];
  __shared__ uint32_t wsum[BS_NW];
  __shared__ uint32_t s_or[BS_NW], s_and[BS_NW];
  __shared__ uint64_t s_vo[BS_NW], s_va[BS_NW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t lmask = (1ull << L) - 1, hmask = (1ull << hbits) - 1;
  const uint32_t lmax = (uint32_t)((1ull << (63 - hbits)) - 1);  // run length field above the hash (capped)
  const uint32_t nb = *n_bins;
  for (uint32_t c = blockIdx.x; c < nb; c += gridDim.x) {
    const uint64_t s = bstart[c], e = bstart[c + 1];
    const int n = (int)(e - s);
    if (threadIdx.x == 0 && c + gridDim.x < nb) {  // the CTA's next bin into L2 while this one is sorted
      const uint64_t s2 = bstart[c + gridDim.x], e2 = bstart[c + gridDim.x + 1];
      if (e2 - s2 > 1 && e2 - s2 <= (uint64_t)BS_CAP) {
        l2_prefetch_range(k + s2, (e2 - s2) * sizeof(uint64_t));
        l2_prefetch_range(v + s2, (e2 - s2) * sizeof(uint32_t));
      }
    }
    if (n <= 1) {
      if (n == 1 && threadIdx.x == 0) {
        k[s] = (k[s] & ~(hmask ^ HASH_BITS_MASK)) | (1ull << hbits);  // strip b, run length 1
        run_emit(ro, rh, 1, racc);
      }
      continue;
    }
    if (n > BS_CAP) {
      if (threadIdx.x == 0) big[atomicAdd(n_big, 1u)] = c;
      continue;
    }
    uint64_t x[BS_IPT];
    uint32_t lmin = 0xFFFFFFFFu, lmax = 0;
    uint64_t seg = 0;
#pragma unroll
    for (int j = 0; j < BS_IPT; j++) {  // all loads of the bin in flight at once
      const int i = wid * (32 * BS_IPT) + j * 32 + lane;
      uint64_t kk = 0;
      uint32_t pp = 0;
      if (i < n) {
        kk = __ldcs(k + s + i);
        pp = __ldcs(v + s + i);
        const uint32_t lo = (uint32_t)(kk & lmask);
        lmin = min(lmin, lo);
        lmax = max(lmax, lo);
        seg = (kk & hmask) >> L;
      }
      x[j] = ((kk & lmask) << 33) | ((uint64_t)pp << 1) | (kk >> 63);
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, d));
      lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, d));
    }
    if (lane == 0) { s_or[wid] = lmin; s_and[wid] = lmax; }
    if (wid == 0 && lane == 0) wsum[0] = (uint32_t)seg;  // every record of a bin has the same segment
    __syncthreads();
    uint32_t mn = 0xFFFFFFFFu, mx = 0;
#pragma unroll
    for (int q = 0; q < BS_NW; q++) { mn = min(mn, s_or[q]); mx = max(mx, s_and[q]); }
    const uint64_t segv = wsum[0];
    __syncthreads();
    // K1 emits records in tile order (any order within a bin): one-hash bins and buckets of very
    // frequent hashes are put in (hash, pos) order by an LSD over the packed bits that vary
    auto lsd_varying = [&](int top_bit) -> const uint64_t* {
      uint64_t o = 0, a = ~0ull;
#pragma unroll
      for (int j = 0; j < BS_IPT; j++) {
        const int i = wid * (32 * BS_IPT) + j * 32 + lane;
        if (i < n) { o |= x[j]; a &= x[j]; }
      }
#pragma unroll
      for (int d = 16; d; d >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, d);
        a &= __shfl_xor_sync(0xffffffffu, a, d);
      }
      if (lane == 0) { s_vo[wid] = o; s_va[wid] = a; }
      __syncthreads();
      uint64_t vo = 0, va = ~0ull;
#pragma unroll
      for (int q = 0; q < BS_NW; q++) { vo |= s_vo[q]; va &= s_va[q]; }
      const uint64_t vary = vo & ~va;
      __syncthreads();
      uint64_t* dst = A;
      bool first = true;
      for (int sh = 1; sh < top_bit; sh += RS_BITS) {
        const int bits = min(RS_BITS, top_bit - sh);
        const uint32_t dm = (1u << bits) - 1;
        if (((vary >> sh) & dm) == 0) continue;  // a constant digit: the pass is the identity
        if (!first) cta_load_striped(dst == A ? Bf : A, n, x);
        cta_rank_scatter(x, n, sh, dm, dst, cnt, wsum);
        dst = dst == A ? Bf : A;
        first = false;
      }
      if (first) {  // nothing varies (cannot happen: positions differ within a bin): the loaded order
#pragma unroll
        for (int j = 0; j < BS_IPT; j++) {
          const int i = wid * (32 * BS_IPT) + j * 32 + lane;
          if (i < n) A[i] = x[j];
        }
        __syncthreads();
        return A;
      }
      return dst == A ? Bf : A;
    };
    if (mn == mx) {  // one hash: sort by position
      const uint64_t* res = lsd_varying(33);
      for (int i = threadIdx.x; i < n; i += BS_NT) {
        const uint64_t pv = res[i];
        __stcs(k + s + i, ((segv << L) | (pv >> 33)) | ((uint64_t)min((uint32_t)n, lmax) << hbits) | ((pv & 1ull) << 63));
        __stcs(v + s + i, (uint32_t)(pv >> 1));
      }
      if (threadIdx.x == 0) {
        if ((uint32_t)n < SMALL_BINS) atomicAdd(&rh[n], 1u);
        else ro.large[atomicAdd(ro.n_large, 1u)] = (uint32_t)n;
        ++racc.nd;
      }
      __syncthreads();
      continue;
    }
    // (1) MSD placement by the top 12 bits of low(h) - mn (4096 buckets, ~1 record each), then an
    //     insertion sort of each bucket on the full packed value (unique: it contains pos)
    const int rbits = 32 - __clz(mx - mn);
    const int shb = rbits > BS_MSD_BITS ? rbits - BS_MSD_BITS : 0;
    {
      uint4* c4 = reinterpret_cast<uint4*>(cnt);
      c4[2 * threadIdx.x] = make_uint4(0, 0, 0, 0);
      c4[2 * threadIdx.x + 1] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    uint32_t bk[BS_IPT];
#pragma unroll
    for (int j = 0; j < BS_IPT; j++) {
      const int i = wid * (32 * BS_IPT) + j * 32 + lane;
      bk[j] = ((uint32_t)(x[j] >> 33) - mn) >> shb;
      if (i < n) atomicAdd(&cnt[bk[j]], 1u);
    }
    __syncthreads();
    uint32_t cmax;
    {
      uint4* c4 = reinterpret_cast<uint4*>(cnt);
      const uint4 p0 = c4[2 * threadIdx.x], p1 = c4[2 * threadIdx.x + 1];
      uint32_t y[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
      uint32_t tsum = 0, tmax = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) { const uint32_t c2 = y[q]; y[q] = tsum; tsum += c2; tmax = max(tmax, c2); }
      uint32_t incl = tsum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t2 = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t2;
      }
#pragma unroll
      for (int d = 16; d; d >>= 1) tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, d));
      if (lane == 31) wsum[wid] = incl;
      if (lane == 0) s_or[wid] = tmax;
      __syncthreads();
      uint32_t before = incl - tsum;
      cmax = 0;
#pragma unroll
      for (int q = 0; q < BS_NW; q++) { before += q < wid ? wsum[q] : 0u; cmax = max(cmax, s_or[q]); }
      c4[2 * threadIdx.x] = make_uint4(y[0] + before, y[1] + before, y[2] + before, y[3] + before);
      c4[2 * threadIdx.x + 1] = make_uint4(y[4] + before, y[5] + before, y[6] + before, y[7] + before);
    }
    __syncthreads();
    const uint64_t* res;
    if (cmax <= (uint32_t)BIN_RANK_MAX) {
#pragma unroll
      for (int j = 0; j < BS_IPT; j++) {
        const int i = wid * (32 * BS_IPT) + j * 32 + lane;
        if (i < n) A[atomicAdd(&cnt[bk[j]], 1u)] = x[j];
      }
      __syncthreads();
      // cnt[b] is now the end of bucket b.  Every element takes its rank in its bucket by counting
      // the smaller values (unique: they contain pos) and moves to Bf — measured faster than
      // per-bucket bitonic or insertion sorts at every bucket size up to the 1024 cap
      for (int p = threadIdx.x; p < n; p += BS_NT) {
        const uint64_t xv = A[p];
        const uint32_t b2 = ((uint32_t)(xv >> 33) - mn) >> shb;
        const int st = b2 ? (int)cnt[b2 - 1] : 0, en = (int)cnt[b2];
        int rank = 0;
        for (int q = st; q < en; q++) rank += A[q] < xv;
        Bf[st + rank] = xv;
      }
      __syncthreads();
      res = Bf;
    } else {
      // (2) a bucket with > 1024 records (a very frequent hash): stable LSD over the low(h) digits below
      //     the highest bit where mn and mx differ (bits above it are constant in the bin)
      if (threadIdx.x == 0) atomicAdd(n_big + 1, 1u);  // statistics: bins sorted this way
      const int hib = 32 - __clz(mn ^ mx);
      res = lsd_varying(33 + hib);
    }
    // K3 fused: runs never cross a bin (a hash lies in one bin).  Per-element run length from two
    // block scans over the run-head indices (start = last head <= i, end = first head > i); it is
    // stored in the key's free bits (capped) for the kept-entry pass, and heads record it in the
    // count histogram.
    uint32_t* Lsm = reinterpret_cast<uint32_t*>(res == A ? Bf : A);
    {
      // warp w owns items [w*256, w*256+256) as 8 rows of 32 (conflict-free SMEM access)
      const int wbase = wid * (32 * BS_IPT);
      uint32_t hm[BS_IPT];
      int wl = -1, wf = n;  // this warp's last / first head
#pragma unroll
      for (int q = 0; q < BS_IPT; q++) {
        const int idx = wbase + q * 32 + lane;
        bool h = false;
        if (idx < n) h = idx == 0 || (uint32_t)(res[idx - 1] >> 33) != (uint32_t)(res[idx] >> 33);
        hm[q] = __ballot_sync(0xffffffffu, h);
        if (hm[q]) {
          wl = wbase + q * 32 + 31 - __clz(hm[q]);
          if (wf == n) wf = wbase + q * 32 + __ffs(hm[q]) - 1;
        }
      }
      if (lane == 0) { s_or[wid] = (uint32_t)(wl + 1); s_and[wid] = (uint32_t)wf; }
      __syncthreads();
      int carry = -1, after = n;
#pragma unroll
      for (int q = 0; q < BS_NW; q++) {
        if (q < wid) carry = max(carry, (int)s_or[q] - 1);
        if (q > wid) after = min(after, (int)s_and[q]);
      }
      const uint32_t le = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1);  // lanes <= lane
      int st_[BS_IPT];
#pragma unroll
      for (int q = 0; q < BS_IPT; q++) {  // start = last head <= idx
        const uint32_t m = hm[q] & le;
        st_[q] = m ? wbase + q * 32 + 31 - __clz(m) : carry;
        if (hm[q]) carry = wbase + q * 32 + 31 - __clz(hm[q]);
      }
#pragma unroll
      for (int q = BS_IPT - 1; q >= 0; q--) {  // next head > idx
        const uint32_t m = hm[q] & ~le;
        const int nh = m ? wbase + q * 32 + __ffs(m) - 1 : after;
        const int idx = wbase + q * 32 + lane;
        if (idx < n) Lsm[idx] = (uint32_t)(nh - st_[q]);
        if (hm[q]) after = wbase + q * 32 + __ffs(hm[q]) - 1;
      }
    }
    __syncthreads();
    const uint64_t topv = segv << L;
    for (int i = threadIdx.x; i < n; i += BS_NT) {
      const uint64_t pv = res[i];
      const uint32_t rlen = Lsm[i];
      __stcs(k + s + i, (topv | (pv >> 33)) | ((uint64_t)min(rlen, lmax) << hbits) | ((pv & 1ull) << 63));
      __stcs(v + s + i, (uint32_t)(pv >> 1));
      if (i == 0 || (uint32_t)(res[i - 1] >> 33) != (uint32_t)(pv >> 33)) run_emit(ro, rh, rlen, racc);
    }
    __syncthreads();
  }
  run_flush(ro, rh, racc);
}

// in-place suffix minimum of f[0 .. m) by the whole CTA (BS_NT threads; ws: BS_NW words)
__device__ __forceinline__ void suffix_min_block(uint32_t* f, uint32_t m, uint32_t* ws) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t C = (m + BS_NT - 1) / BS_NT;
  const uint32_t b0 = threadIdx.x * C, b1 = min(b0 + C, m);
  uint32_t mn = 0xFFFFFFFFu;
  for (uint32_t q = b1; q > b0; q--) { mn = min(mn, f[q - 1]); f[q - 1] = mn; }
  uint32_t x = mn;  // inclusive suffix min over the lanes >= lane
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_down_sync(0xffffffffu, x, d);
    if (lane + d < 32) x = min(x, y);
  }
  if (lane == 0) ws[wid] = x;
  const uint32_t nxt = __shfl_down_sync(0xffffffffu, x, 1);
  __syncthreads();
  uint32_t after = lane < 31 ? nxt : 0xFFFFFFFFu;
#pragma unroll
  for (int q = 0; q < BS_NW; q++)
    if (q > wid) after = min(after, ws[q]);
  for (uint32_t q = b0; q < b1; q++) f[q] = min(f[q], after);
  __syncthreads();
}

__global__ void __launch_bounds__(BS_NT, BS_MINB) k_bin_build(const uint64_t* __restrict__ k, const uint32_t* __restrict__ v,
                                                        const uint64_t* __restrict__ bstart,
                                                        const uint32_t* __restrict__ n_bins, int L, int hbits,
                                                        uint32_t* big, uint32_t* n_big, RunOut ro,
                                                        const uint2* __restrict__ table,
                                                        const uint32_t* __restrict__ binseg, uint32_t S,
                                                        uint64_t* __restrict__ ent, DirRec* __restrict__ dir,
                                                        uint32_t* bin_ctr) {
  extern __shared__ __align__(16) unsigned char bs_smem[];
  uint64_t* A = reinterpret_cast<uint64_t*>(bs_smem);
  uint64_t* Bf = A + BS_CAP;
  uint32_t* rh = reinterpret_cast<uint32_t*>(Bf + BS_CAP);  // [SMALL_BINS] run-count histogram
  uint32_t* first = rh + SMALL_BINS;                          // [S + 1] first record of each slot of the bin
  for (int i = threadIdx.x; i < (int)SMALL_BINS; i += BS_NT) rh[i] = 0;
  __syncthreads();
  RunAcc racc;
  __shared__ __align__(16) uint32_t cnt[CNT_WORDS];
  __shared__ uint32_t wsum[BS_NW];
  __shared__ uint32_t s_or[BS_NW], s_and[BS_NW];
  __shared__ uint64_t s_vo[BS_NW], s_va[BS_NW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t lmask = (1ull << L) - 1, hmask = (1ull << hbits) - 1;
  const uint32_t nb = *n_bins;
  // Bins are claimed from a counter, one ahead (the first one is the CTA's index): a bin's cost varies
  // several-fold (a mid bin ~2.5 average bins), and a static round-robin left the CTAs with the most
  // of those running alone at the end (measured: 2056 mid bins cost 0.76 ms that way).
  __shared__ uint32_t s_next[2];
  uint32_t c = blockIdx.x, nxt = 0, it = 0;
  if (threadIdx.x == 0) nxt = atomicAdd(bin_ctr, 1u) + gridDim.x;
  while (c < nb) {
    uint32_t nn = 0;
    do {
    const uint64_t s = bstart[c], e = bstart[c + 1];
    const int n = (int)(e - s);
    if (threadIdx.x == 0) {
      s_next[it & 1u] = nxt;
      nn = atomicAdd(bin_ctr, 1u) + gridDim.x;  // the bin after the next (its latency hides under this bin)
      if (nxt < nb) {  // the CTA's next bin into L2 while this one is sorted
        const uint64_t s2 = bstart[nxt], e2 = bstart[nxt + 1];
        if (e2 - s2 > 1 && e2 - s2 <= (uint64_t)(2 * BS_CAP)) {
          l2_prefetch_range(k + s2, (e2 - s2) * sizeof(uint64_t));
          l2_prefetch_range(v + s2, (e2 - s2) * sizeof(uint32_t));
        }
      }
    }
    if (n == 0) {  // an empty bin: its S slots are empty
      for (uint32_t q = threadIdx.x; q < S; q += BS_NT) {
        uint4* o = reinterpret_cast<uint4*>(dir + (uint64_t)c * S + q);
        o[0] = make_uint4((uint32_t)s, (uint32_t)s, 0xFFFFFFFFu, 0xFFFFFFFFu);
        o[1] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
      }
      break;
    }
    if (n > 2 * BS_CAP) {
      if (threadIdx.x == 0) big[atomicAdd(n_big, 1u)] = c;
      break;
    }
    const uint64_t* res = nullptr;
    bool one = false;
    uint64_t segv = 0;
    const bool mid = n > BS_CAP;
    if (mid) {
      // BS_CAP < n <= 2 BS_CAP (a frequent hash on top of a full bin): the two buffers together hold the
      // bin; an in-place bitonic sort of the packed values (unique, so no stability is needed), padded
      // with ~0 to 2 BS_CAP.  (Through k_bucket_sort_big's chunked global-memory LSD such a bin cost
      // ~150 us; measured, round 2.)
      if (threadIdx.x == 0) atomicAdd(n_big + 2, 1u);  // statistics: bins sorted this way
      constexpr int N2 = 2 * BS_CAP;
      for (int i = threadIdx.x; i < N2; i += BS_NT) {
        uint64_t xv = ~0ull;
        if (i < n) {
          const uint64_t kk = __ldcs(k + s + i);
          const uint32_t pp = __ldcs(v + s + i);
          xv = ((kk & lmask) << 33) | ((uint64_t)pp << 1) | (kk >> 63);
        }
        A[i] = xv;
      }
      segv = (k[s] & hmask) >> L;
      __syncthreads();
      for (int kk2 = 2; kk2 <= N2; kk2 <<= 1) {
        for (int j = kk2 >> 1; j > 0; j >>= 1) {
          for (int t = threadIdx.x; t < N2 / 2; t += BS_NT) {
            const int lo = 2 * t - (t & (j - 1)), hi = lo + j;
            const uint64_t a = A[lo], b = A[hi];
            const bool up = (lo & kk2) == 0;
            if ((a > b) == up) { A[lo] = b; A[hi] = a; }
          }
          __syncthreads();
        }
      }
      res = A;
    } else {
    uint64_t x[BS_IPT];
    uint32_t lmin = 0xFFFFFFFFu, lmax = 0;
    uint64_t seg = 0;
#pragma unroll
    for (int j = 0; j < BS_IPT; j++) {  // all loads of the bin in flight at once
      const int i = wid * (32 * BS_IPT) + j * 32 + lane;
      uint64_t kk = 0;
      uint32_t pp = 0;
      if (i < n) {
        kk = __ldcs(k + s + i);
        pp = __ldcs(v + s + i);
        const uint32_t lo = (uint32_t)(kk & lmask);
        lmin = min(lmin, lo);
        lmax = max(lmax, lo);
        seg = (kk & hmask) >> L;
      }
      x[j] = ((kk & lmask) << 33) | ((uint64_t)pp << 1) | (kk >> 63);
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, d));
      lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, d));
    }
    if (lane == 0) { s_or[wid] = lmin; s_and[wid] = lmax; }
    if (wid == 0 && lane == 0) wsum[0] = (uint32_t)seg;  // every record of a bin has the same segment
    __syncthreads();
    uint32_t mn = 0xFFFFFFFFu, mx = 0;
#pragma unroll
    for (int q = 0; q < BS_NW; q++) { mn = min(mn, s_or[q]); mx = max(mx, s_and[q]); }
    segv = wsum[0];
    __syncthreads();
    // K1 emits records in tile order (any order within a bin): one-hash bins and buckets of very
    // frequent hashes are put in (hash, pos) order by an LSD over the packed bits that vary
    auto lsd_varying = [&](int top_bit) -> const uint64_t* {
      uint64_t o = 0, a = ~0ull;
#pragma unroll
      for (int j = 0; j < BS_IPT; j++) {
        const int i = wid * (32 * BS_IPT) + j * 32 + lane;
        if (i < n) { o |= x[j]; a &= x[j]; }
      }
#pragma unroll
      for (int d = 16; d; d >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, d);
        a &= __shfl_xor_sync(0xffffffffu, a, d);
      }
      if (lane == 0) { s_vo[wid] = o; s_va[wid] = a; }
      __syncthreads();
      uint64_t vo = 0, va = ~0ull;
#pragma unroll
      for (int q = 0; q < BS_NW; q++) { vo |= s_vo[q]; va &= s_va[q]; }
      const uint64_t vary = vo & ~va;
      __syncthreads();
      uint64_t* dst = A;
      bool first = true;
      for (int sh = 1; sh < top_bit; sh += RS_BITS) {
        const int bits = min(RS_BITS, top_bit - sh);
        const uint32_t dm = (1u << bits) - 1;
        if (((vary >> sh) & dm) == 0) continue;  // a constant digit: the pass is the identity
        if (!first) cta_load_striped(dst == A ? Bf : A, n, x);
        cta_rank_scatter(x, n, sh, dm, dst, cnt, wsum);
        dst = dst == A ? Bf : A;
        first = false;
      }
      if (first) {  // nothing varies (cannot happen: positions differ within a bin): the loaded order
#pragma unroll
        for (int j = 0; j < BS_IPT; j++) {
          const int i = wid * (32 * BS_IPT) + j * 32 + lane;
          if (i < n) A[i] = x[j];
        }
        __syncthreads();
        return A;
      }
      return dst == A ? Bf : A;
    };
    one = mn == mx;  // one hash: sort by position
    res = one ? lsd_varying(33) : nullptr;
    if (!one) {
    // (1) MSD placement by the top 12 bits of low(h) - mn (4096 buckets, ~1 record each), then an
    //     insertion sort of each bucket on the full packed value (unique: it contains pos)
    const int rbits = 32 - __clz(mx - mn);
    const int shb = rbits > BS_MSD_BITS ? rbits - BS_MSD_BITS : 0;
    {
      uint4* c4 = reinterpret_cast<uint4*>(cnt);
      c4[2 * threadIdx.x] = make_uint4(0, 0, 0, 0);
      c4[2 * threadIdx.x + 1] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    uint32_t bk[BS_IPT];
#pragma unroll
    for (int j = 0; j < BS_IPT; j++) {
      const int i = wid * (32 * BS_IPT) + j * 32 + lane;
      bk[j] = ((uint32_t)(x[j] >> 33) - mn) >> shb;
      if (i < n) atomicAdd(&cnt[bk[j]], 1u);
    }
    __syncthreads();
    uint32_t cmax;
    {
      uint4* c4 = reinterpret_cast<uint4*>(cnt);
      const uint4 p0 = c4[2 * threadIdx.x], p1 = c4[2 * threadIdx.x + 1];
      uint32_t y[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
      uint32_t tsum = 0, tmax = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) { const uint32_t c2 = y[q]; y[q] = tsum; tsum += c2; tmax = max(tmax, c2); }
      uint32_t incl = tsum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t2 = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t2;
      }
#pragma unroll
      for (int d = 16; d; d >>= 1) tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, d));
      if (lane == 31) wsum[wid] = incl;
      if (lane == 0) s_or[wid] = tmax;
      __syncthreads();
      uint32_t before = incl - tsum;
      cmax = 0;
#pragma unroll
      for (int q = 0; q < BS_NW; q++) { before += q < wid ? wsum[q] : 0u; cmax = max(cmax, s_or[q]); }
      c4[2 * threadIdx.x] = make_uint4(y[0] + before, y[1] + before, y[2] + before, y[3] + before);
      c4[2 * threadIdx.x + 1] = make_uint4(y[4] + before, y[5] + before, y[6] + before, y[7] + before);
    }
    __syncthreads();
    if (cmax <= (uint32_t)BIN_RANK_MAX) {
#pragma unroll
      for (int j = 0; j < BS_IPT; j++) {
        const int i = wid * (32 * BS_IPT) + j * 32 + lane;
        if (i < n) A[atomicAdd(&cnt[bk[j]], 1u)] = x[j];
      }
      __syncthreads();
      // cnt[b] is now the end of bucket b.  Every element takes its rank in its bucket by counting
      // the smaller values (unique: they contain pos) and moves to Bf — measured faster than
      // per-bucket bitonic or insertion sorts at every bucket size up to the 1024 cap
      for (int p = threadIdx.x; p < n; p += BS_NT) {
        const uint64_t xv = A[p];
        const uint32_t b2 = ((uint32_t)(xv >> 33) - mn) >> shb;
        const int st = b2 ? (int)cnt[b2 - 1] : 0, en = (int)cnt[b2];
        int rank = 0, q = st;
        if (q & 1) rank += A[q++] < xv;  // then two keys per 128-bit SMEM load
        for (; q + 1 < en; q += 2) {
          const ulonglong2 two = *reinterpret_cast<const ulonglong2*>(A + q);
          rank += (two.x < xv) + (two.y < xv);
        }
        if (q < en) rank += A[q] < xv;
        Bf[st + rank] = xv;
      }
      __syncthreads();
      res = Bf;
    } else {
      // (2) a bucket with > 1024 records (a very frequent hash): stable LSD over the low(h) digits below
      //     the highest bit where mn and mx differ (bits above it are constant in the bin)
      if (threadIdx.x == 0) atomicAdd(n_big + 1, 1u);  // statistics: bins sorted this way
      const int hib = 32 - __clz(mn ^ mx);
      res = lsd_varying(33 + hib);
    }
    }  // !one
    }  // !mid
    // K3 fused: runs never cross a bin (a hash lies in one bin).  A run head finds its run's end by
    // galloping over the sorted records (almost every run has one record: one comparison); round 2's
    // first version marked the heads in the other buffer and took a block suffix minimum (4 barriers
    // more per bin).
    // K5 + K6 fused: entries in final position (all of them: a hash with count > tau is dropped at
    // probe time, reading O7), then the bin's S directory slots (bins are unions of whole slots)
    const uint2 tb = table[segv];                  // (first bin, bins) of the bin's segment
    const uint64_t slots_t = (uint64_t)tb.y * S;   // slots of the segment
    const uint64_t qbase = (uint64_t)(c - tb.x) * S;
    for (uint32_t q = threadIdx.x; q <= S; q += BS_NT) first[q] = (uint32_t)n;
    __syncthreads();
    GOD_DCHECK(e <= bstart[nb] && (uint64_t)c * S + S <= (uint64_t)nb * S, "bin build: bin range");
    for (int i = threadIdx.x; i < n; i += BS_NT) {
      const uint64_t pv = res[i];
      __stcs(ent + s + i, ((pv >> 1) << 32) | ((pv >> 33) << 1) | (pv & 1ull));
      const uint32_t lo = (uint32_t)(pv >> 33);
      const bool head = i == 0 || (uint32_t)(res[i - 1] >> 33) != lo;
      if (one) {
        if (i == 0) run_emit(ro, rh, (uint64_t)n, racc);
      } else if (head) {
        int lo2 = i + 1, st = 1;  // gallop, then bisect, to the first record with another key
        while (lo2 + st <= n && (uint32_t)(res[lo2 + st - 1] >> 33) == lo) { lo2 += st; st <<= 1; }
        int hi2 = min(lo2 + st - 1, n);
        while (lo2 < hi2) {
          const int m2 = (lo2 + hi2) >> 1;
          if ((uint32_t)(res[m2] >> 33) == lo) lo2 = m2 + 1;
          else hi2 = m2;
        }
        run_emit(ro, rh, (uint64_t)(lo2 - i), racc);
      }
      if (head) {  // a slot starts at a run head: its first record
        const uint32_t q = (uint32_t)((((uint64_t)lo * slots_t) >> L) - qbase);
        GOD_DCHECK(q < S, "bin build: slot of a record inside its bin");
        const uint32_t qp = i ? (uint32_t)((((res[i - 1] >> 33) * slots_t) >> L) - qbase) : 0xFFFFFFFFu;
        if (q != qp) first[q] = (uint32_t)i;
      }
    }
    __syncthreads();
    suffix_min_block(first, S + 1, wsum);
    for (uint32_t q = threadIdx.x; q < S; q += BS_NT) {
      const uint32_t a0 = first[q], b0 = first[q + 1];
      uint32_t kk[DIR_KEYS];
      if (b0 - a0 <= DIR_PAIRS) {  // the entries themselves
        dir_pairs(b0 - a0, [&](int e2) {
          const uint64_t pv = res[a0 + e2];
          return ((pv >> 1) << 32) | ((pv >> 33) << 1) | (pv & 1ull);
        }, kk);
      } else if (b0 - a0 <= DIR_KEYS) {
#pragma unroll
        for (int e2 = 0; e2 < DIR_KEYS; e2++) kk[e2] = a0 + e2 < b0 ? (uint32_t)(res[a0 + e2] >> 33) : 0xFFFFFFFFu;
      } else {  // <= DIR_RUNS distinct keys: (key, run end) pairs; more: key[0] = ~0 (the probe searches)
#pragma unroll
        for (int e2 = 0; e2 < DIR_KEYS; e2++) kk[e2] = (e2 & 1) ? (uint32_t)(s + b0) : 0xFFFFFFFFu;
        uint32_t s0 = a0;
        for (int r = 0; r < DIR_RUNS && s0 < b0; r++) {
          const uint32_t ks = (uint32_t)(res[s0] >> 33);
          uint32_t lo2 = s0 + 1, st = 1;  // gallop, then bisect, to the first record with another key
          while (lo2 + st <= b0 && (uint32_t)(res[lo2 + st - 1] >> 33) == ks) { lo2 += st; st <<= 1; }
          uint32_t hi2 = min(lo2 + st - 1, b0);
          while (lo2 < hi2) {
            const uint32_t mid = (lo2 + hi2) >> 1;
            if ((uint32_t)(res[mid] >> 33) == ks) lo2 = mid + 1;
            else hi2 = mid;
          }
          kk[2 * r] = ks;
          kk[2 * r + 1] = (uint32_t)(s + lo2);
          s0 = lo2;
        }
        if (s0 < b0) kk[0] = 0xFFFFFFFFu;
      }
      uint4* o = reinterpret_cast<uint4*>(dir + (uint64_t)c * S + q);
      o[0] = make_uint4((uint32_t)(s + a0), (uint32_t)(s + b0), kk[0], kk[1]);
      o[1] = make_uint4(kk[2], kk[3], kk[4], kk[5]);
    }
    } while (0);
    __syncthreads();
    c = s_next[it & 1u];
    nxt = nn;
    ++it;
  }
  run_flush(ro, rh, racc);
}

// oversized bins (repeat-heavy hashes): the same LSD over the low bits, chunk by chunk through
// global memory (stable across chunks: chunks are taken in order, each digit's run appended)
__global__ void __launch_bounds__(BS_NT, BS_BIG_MINB) k_bucket_sort_big(uint64_t* __restrict__ k, uint32_t* __restrict__ v,
                                                              uint64_t* __restrict__ t0, uint64_t* __restrict__ t1,
                                                              const uint64_t* __restrict__ bstart, const uint32_t* big,
                                                              const uint32_t* n_big, int lo_bits, int hbits, RunOut ro,
                                                              uint64_t* __restrict__ ent) {
  extern __shared__ __align__(16) unsigned char bs_smem[];
  uint64_t* Bf = reinterpret_cast<uint64_t*>(bs_smem);
  uint32_t* rh = reinterpret_cast<uint32_t*>(Bf + 2 * BS_CAP);  // [SMALL_BINS] run-count histogram
  for (int i = threadIdx.x; i < (int)SMALL_BINS; i += BS_NT) rh[i] = 0;
  __syncthreads();
  RunAcc racc;
  __shared__ __align__(16) uint32_t cnt[CNT_WORDS];
  __shared__ uint32_t wsum[BS_NW];
  __shared__ uint64_t dbase[RS_BINS];
  __shared__ uint32_t hist[RS_BINS];
  const uint64_t lowmask = (1ull << lo_bits) - 1;
  const uint32_t nbig = *n_big;
  for (uint32_t q = blockIdx.x; q < nbig; q += gridDim.x) {
    const uint32_t b = big[q];
    const uint64_t s = bstart[b], e = bstart[b + 1], n = e - s;
    if (threadIdx.x == 0 && q + gridDim.x < nbig) {  // the CTA's next bin into L2 (its first 16 K records)
      const uint32_t b2 = big[q + gridDim.x];
      const uint64_t s2 = bstart[b2], n2 = min(bstart[b2 + 1] - s2, (uint64_t)16384);
      l2_prefetch_range(k + s2, n2 * sizeof(uint64_t));
      l2_prefetch_range(v + s2, n2 * sizeof(uint32_t));
    }
    const uint64_t top = ((k[s] & ((1ull << hbits) - 1)) >> lo_bits) << lo_bits;  // the bin's segment
    __shared__ unsigned long long s_diff;
    if (threadIdx.x == 0) s_diff = 0;
    __syncthreads();
    const uint64_t x0 = ((k[s] & lowmask) << 33) | ((uint64_t)v[s] << 1) | (k[s] >> 63);
    uint64_t diff = 0;  // packed bits that vary across the bin (records arrive in any order)
    for (uint64_t i = threadIdx.x; i < n; i += BS_NT) {
      const uint64_t kk = k[s + i];
      const uint64_t xv = ((kk & lowmask) << 33) | ((uint64_t)v[s + i] << 1) | (kk >> 63);
      diff |= xv ^ x0;
      t0[s + i] = xv;
    }
    for (int o = 16; o; o >>= 1) diff |= __shfl_xor_sync(0xffffffffu, diff, o);
    if ((threadIdx.x & 31) == 0 && diff) atomicOr(&s_diff, (unsigned long long)diff);
    __syncthreads();
    const uint64_t vary = s_diff;
    uint64_t* src = t0 + s;
    uint64_t* dst = t1 + s;
    for (int sh = 1; sh < 33 + lo_bits; sh += RS_BITS) {  // (pos, then low hash) digits, LSD
      const int bits = min(RS_BITS, 33 + lo_bits - sh);
      const uint32_t dmask = (1u << bits) - 1;
      const int shift = sh;
      if (((vary >> sh) & dmask) == 0) continue;  // a constant digit: the stable pass is the identity
      for (int i = threadIdx.x; i < RS_BINS; i += BS_NT) hist[i] = 0;
      __syncthreads();
      for (uint64_t i = threadIdx.x; i < n; i += BS_NT) atomicAdd(&hist[(uint32_t)(src[i] >> shift) & dmask], 1u);
      __syncthreads();
      if (threadIdx.x == 0) {
        uint64_t acc = 0;
        for (int d = 0; d < RS_BINS; d++) { dbase[d] = acc; acc += hist[d]; }
      }
      __syncthreads();
      for (uint64_t c0 = 0; c0 < n; c0 += BS_CAP) {
        const int cn = (int)min((uint64_t)BS_CAP, n - c0);
        uint64_t x[BS_IPT];
        cta_load_striped(src + c0, cn, x);
        cta_rank_scatter(x, cn, shift, dmask, Bf, cnt, wsum);
        // Bf: the chunk sorted by digit; digit d's run starts at cnt[d * CNT_LD], its slot is dbase[d]
        for (int i = threadIdx.x; i < cn; i += BS_NT) {
          const uint64_t pv = Bf[i];
          const uint32_t d = (uint32_t)(pv >> shift) & dmask;
          dst[dbase[d] + (i - cnt[d * CNT_LD])] = pv;
        }
        __syncthreads();
        if (threadIdx.x < RS_BINS) {  // advance by this chunk's count of digit threadIdx.x
          const uint32_t d = threadIdx.x;
          const uint32_t nxt = d + 1 < RS_BINS ? cnt[(d + 1) * CNT_LD] : (uint32_t)cn;
          dbase[d] += nxt - cnt[d * CNT_LD];
        }
        __syncthreads();
      }
      uint64_t* t = src; src = dst; dst = t;
    }
    for (uint64_t i = threadIdx.x; i < n; i += BS_NT) {
      const uint64_t pv = src[i];
      k[s + i] = (top | (pv >> 33)) | ((pv & 1ull) << 63);
      v[s + i] = (uint32_t)(pv >> 1);
      if (ent) ent[s + i] = ((pv >> 1) << 32) | ((pv >> 33) << 1) | (pv & 1ull);
    }
    __syncthreads();
    // K3 fused: every record finds its run's extent in the bin (galloping both ways), stores the
    // length in the key's free bits (capped) for the kept-entry pass; run heads record it
    {
      const uint64_t hm = (1ull << hbits) - 1, lmax = (1ull << (63 - hbits)) - 1;
      const uint64_t* kb = k + s;
      for (uint64_t i = threadIdx.x; i < n; i += BS_NT) {
        const uint64_t hv = kb[i] & hm;
        const uint64_t back = run_side(kb, n, i, hv, n, false, hm);
        const uint64_t L = 1 + back + run_side(kb, n, i, hv, n, true, hm);
        if (back == 0) run_emit(ro, rh, L, racc);
        k[s + i] = (kb[i] & ~(lmax << hbits)) | ((L < lmax ? L : lmax) << hbits);
      }
    }
    __syncthreads();
  }
  run_flush(ro, rh, racc);
}

// K6 for the oversized bins (sorted by k_bucket_sort_big into k and ent): each slot's first record by
// binary search (slot numbers are non-decreasing in the sorted records), then the slot records
__global__ void __launch_bounds__(BS_NT) k_big_dir(const uint64_t* __restrict__ k, const uint64_t* __restrict__ bstart,
                                                   const uint32_t* big, const uint32_t* n_big, int L, int hbits,
                                                   const uint2* __restrict__ table, uint32_t S,
                                                   const uint64_t* __restrict__ ent, DirRec* __restrict__ dir) {
  const uint64_t lmask = (1ull << L) - 1, hmask = (1ull << hbits) - 1;
  const uint32_t nbig = *n_big;
  for (uint32_t qb = blockIdx.x; qb < nbig; qb += gridDim.x) {
    const uint32_t c = big[qb];
    const uint64_t s = bstart[c], n = bstart[c + 1] - s;
    const uint2 tb = table[(k[s] & hmask) >> L];
    const uint64_t slots_t = (uint64_t)tb.y * S, qbase = (uint64_t)(c - tb.x) * S;
    auto key = [&](uint64_t i) -> uint32_t { return (uint32_t)(k[s + i] & lmask); };
    auto slot = [&](uint64_t i) -> uint64_t { return (((uint64_t)key(i) * slots_t) >> L) - qbase; };
    auto first_at = [&](uint64_t q) -> uint64_t {  // first record with slot >= q
      uint64_t lo = 0, hi = n;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (slot(mid) < q) lo = mid + 1;
        else hi = mid;
      }
      return lo;
    };
    for (uint32_t q = threadIdx.x; q < S; q += BS_NT) {
      const uint64_t a0 = first_at(q), b0 = first_at(q + 1);
      uint32_t kk[DIR_KEYS];
      if (b0 - a0 <= DIR_PAIRS) {  // the entries themselves
        dir_pairs((uint32_t)(b0 - a0), [&](int e2) { return ent[s + a0 + e2]; }, kk);
      } else if (b0 - a0 <= DIR_KEYS) {
#pragma unroll
        for (int e2 = 0; e2 < DIR_KEYS; e2++) kk[e2] = a0 + e2 < b0 ? key(a0 + e2) : 0xFFFFFFFFu;
      } else {
#pragma unroll
        for (int e2 = 0; e2 < DIR_KEYS; e2++) kk[e2] = (e2 & 1) ? (uint32_t)(s + b0) : 0xFFFFFFFFu;
        uint64_t s0 = a0;
        for (int r = 0; r < DIR_RUNS && s0 < b0; r++) {
          const uint32_t ks = key(s0);
          uint64_t lo2 = s0 + 1, st = 1;
          while (lo2 + st <= b0 && key(lo2 + st - 1) == ks) { lo2 += st; st <<= 1; }
          uint64_t hi2 = min(lo2 + st - 1, b0);
          while (lo2 < hi2) {
            const uint64_t mid = (lo2 + hi2) >> 1;
            if (key(mid) == ks) lo2 = mid + 1;
            else hi2 = mid;
          }
          kk[2 * r] = ks;
          kk[2 * r + 1] = (uint32_t)(s + lo2);
          s0 = lo2;
        }
        if (s0 < b0) kk[0] = 0xFFFFFFFFu;
      }
      uint4* o = reinterpret_cast<uint4*>(dir + (uint64_t)c * S + q);
      o[0] = make_uint4((uint32_t)(s + a0), (uint32_t)(s + b0), kk[0], kk[1]);
      o[1] = make_uint4(kk[2], kk[3], kk[4], kk[5]);
    }
  }
}

// K3: runs of equal hashes in the sorted records (one run = one distinct hash, P:286 (3)).  The
// thread holding a run head finds the run end (linear for short runs, exponential + binary search
// for long ones) and adds its length to the count histogram
// (SMEM bins for counts < SMALL_BINS, a list for the rare larger ones) used by the cutoff.
__global__ void k_runs(const uint64_t* __restrict__ k, uint64_t n, RunOut ro) {
  __shared__ uint32_t h[SMALL_BINS];
  for (int i = threadIdx.x; i < (int)SMALL_BINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  RunAcc racc;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t hv = k[i] & HASH_BITS_MASK;
    if (i > 0 && (k[i - 1] & HASH_BITS_MASK) == hv) continue;
    uint64_t e = i + 1;
    while (e < n && e - i < 8 && (k[e] & HASH_BITS_MASK) == hv) ++e;
    if (e - i == 8 && e < n && (k[e] & HASH_BITS_MASK) == hv) {
      uint64_t lo = e, step = 8;  // key(lo) == hv
      while (lo + step < n && (k[lo + step] & HASH_BITS_MASK) == hv) { lo += step; step <<= 1; }
      uint64_t hi = lo + step < n ? lo + step : n;  // first index with a different key is in (lo, hi]
      while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if ((k[mid] & HASH_BITS_MASK) == hv) lo = mid;
        else hi = mid;
      }
      e = hi;
    }
    run_emit(ro, h, e - i, racc);
  }
  run_flush(ro, h, racc);
}

struct CutState {
  uint64_t n_entries, n_distinct, m, tau;
  uint64_t kept_entries, kept_distinct;
};

// tau = (m+1)-th largest count (reading O7: tau = a_{n-m-1}); one block.
__global__ void __launch_bounds__(1024) k_tau(const uint32_t* hist_small, const uint32_t* large, const uint32_t* n_large_p,
                                              const uint64_t* nd_p, uint64_t n_entries, uint32_t mode, uint32_t num,
                                              uint32_t den, uint32_t max_occ, CutState* cs) {
  __shared__ uint32_t bins[256];
  __shared__ uint32_t s_prefix, s_mask;
  __shared__ uint64_t s_need;
  const uint64_t nd = *nd_p;
  const uint32_t nl = *n_large_p;
  uint64_t m = 0, tau = 0;
  if (mode == 1) {
    tau = max_occ;
  } else {
    m = den ? (uint64_t)(((unsigned __int128)nd * num) / den) : 0;
    if (nd == 0 || m >= nd) {
      tau = 0;
    } else if (m + 1 <= nl) {
      // radix select the (m+1)-th largest among the large counts (32-bit, 4 x 8-bit digits)
      if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; s_need = m + 1; }
      __syncthreads();
      for (int sh = 24; sh >= 0; sh -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) bins[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
          const uint32_t v = large[i];
          if ((v & s_mask) == s_prefix) atomicAdd(&bins[(v >> sh) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          uint64_t need = s_need;
          for (int d = 255; d >= 0; d--) {
            if (bins[d] >= need) { s_prefix |= (uint32_t)d << sh; break; }
            need -= bins[d];
          }
          s_need = need;
          s_mask |= 255u << sh;
        }
        __syncthreads();
      }
      tau = s_prefix;
    } else {
      if (threadIdx.x == 0) {
        uint64_t cum = nl;  // counts >= SMALL_BINS
        uint64_t v = SMALL_BINS;
        while (v > 0) {
          --v;
          cum += hist_small[v];
          if (cum >= m + 1) break;
        }
        s_need = v;
      }
      __syncthreads();
      tau = s_need;
    }
  }
  // kept distinct hashes and entries: counts <= tau (histogram bins and the large list)
  __shared__ unsigned long long s_kd, s_ke;
  if (threadIdx.x == 0) { s_kd = 0; s_ke = 0; }
  __syncthreads();
  unsigned long long kd = 0, ke = 0;
  for (uint32_t c = threadIdx.x; c < SMALL_BINS && c <= tau; c += blockDim.x) {
    kd += hist_small[c];
    ke += (unsigned long long)c * hist_small[c];
  }
  for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x)
    if (large[i] <= tau) { kd += 1; ke += large[i]; }
  atomicAdd(&s_kd, kd);
  atomicAdd(&s_ke, ke);
  __syncthreads();
  if (threadIdx.x == 0) {
    cs->n_entries = n_entries;
    cs->n_distinct = nd;
    cs->m = m;
    cs->tau = tau;
    cs->kept_entries = s_ke;
    cs->kept_distinct = s_kd;
  }
}

// K5: kept entries in order, one pass: a record is kept iff its run length <= tau (reading O7);
// tiles of KW_TILE records (warp-striped), ballot compaction, tile offsets by decoupled look-back.
// Writes the entry (pos << 32 | low hash << 1 | strand) and its directory slot.
constexpr int KW_NT = 256, KW_IPT = 16, KW_TILE = KW_NT * KW_IPT;
__global__ void __launch_bounds__(KW_NT) k_keep_write(const uint64_t* __restrict__ k, const uint32_t* __restrict__ pos,
                                                      uint64_t n, int hbits, const CutState* cs,
                                                      IndexView iv, uint64_t* ent, uint32_t* dir1, uint64_t* status,
                                                      uint32_t* tile_ctr) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t wtot[KW_NT / 32];
  __shared__ uint64_t s_excl;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t tau = cs->tau;
  const uint64_t hm = (1ull << hbits) - 1, lmax = (1ull << (63 - hbits)) - 1;
  const uint64_t base = tile * KW_TILE + (uint64_t)wid * (32 * KW_IPT);
  uint32_t masks[KW_IPT];
  uint32_t wc = 0;
#pragma unroll 4
  for (int j = 0; j < KW_IPT; j++) {
    const uint64_t i = base + (uint64_t)j * 32 + lane;
    bool keep = false;
    if (i < n) {
      const uint64_t v = k[i];
      const uint64_t rlf = (v >> hbits) & lmax;  // run length from the bin sort (0: not recorded)
      if (rlf != 0 && (rlf < lmax || tau < lmax)) keep = rlf <= tau;
      else keep = run_len_capped(k, n, i, v & hm, tau, hm) <= tau;
    }
    masks[j] = __ballot_sync(0xffffffffu, keep);
    wc += __popc(masks[j]);
  }
  if (lane == 0) wtot[wid] = wc;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = lane < KW_NT / 32 ? wtot[lane] : 0u;
    uint32_t incl = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, KW_NT / 32 - 1);
    const uint64_t ex = lb_exclusive_warp(status, tile, total);
    if (lane < KW_NT / 32) wtot[lane] = incl - t;  // warp exclusive prefix within the tile
    if (lane == 0) s_excl = ex;
  }
  __syncthreads();
  uint64_t run = s_excl + wtot[wid];
  const uint32_t lt = (1u << lane) - 1;
  const uint64_t lowmask = (1ull << iv.low_bits) - 1;
#pragma unroll
  for (int j = 0; j < KW_IPT; j++) {
    const uint32_t m = masks[j];
    const bool mine = (m >> lane) & 1u;
    uint32_t slot = 0;
    uint64_t d = 0;
    if (mine) {
      const uint64_t i = base + (uint64_t)j * 32 + lane;
      const uint64_t v = k[i];
      const uint64_t h = v & hm;
      d = run + __popc(m & lt);
      ent[d] = ((uint64_t)pos[i] << 32) | ((h & lowmask) << 1) | (v >> 63);
      slot = (uint32_t)index_slot(iv, h);
    }
    // K6a fused: the first entry of each slot (entries are in slot order).  The previous kept entry
    // of this round decides; the first kept lane of a round cannot see its predecessor and takes an
    // atomic minimum (a plain store only ever writes the true first entry, so the two commute).
    const uint32_t before = m & lt;
    const int prev = before ? 31 - __clz(before) : lane;
    const uint32_t pslot = __shfl_sync(0xffffffffu, slot, prev);
    if (mine) {
      if (!before) atomicMin(dir1 + slot, (uint32_t)d);
      else if (pslot != slot) dir1[slot] = (uint32_t)d;
    }
    run += __popc(m);
  }
}


// K6b: empty slots take the next non-empty slot's first entry: a suffix-min over dir[0 .. 2^B],
// single pass, tiles processed right to left with a decoupled look-back on the running minimum.
constexpr int DF_NT = 256, DF_IPT = 16, DF_TILE = DF_NT * DF_IPT;
__global__ void __launch_bounds__(DF_NT) k_dir_suffix_min(const uint32_t* dir, uint64_t n, uint64_t* status, uint32_t* ctr,
                                                          const uint64_t* __restrict__ ent, uint64_t n_slots,
                                                          DirRec* __restrict__ rec) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t warp_min[DF_NT / 32];
  __shared__ uint32_t s_carry;
  if (threadIdx.x == 0) s_tile = atomicAdd(ctr, 1u);
  __syncthreads();
  const uint64_t ntiles = (n + DF_TILE - 1) / DF_TILE;
  const uint64_t rt = s_tile;                 // look-back order: right to left
  const uint64_t t = ntiles - 1 - rt;         // tile position
  const uint64_t base = t * DF_TILE + (uint64_t)threadIdx.x * DF_IPT;
  uint32_t v[DF_IPT];
#pragma unroll
  for (int i = 0; i < DF_IPT; i++) v[i] = base + i < n ? dir[base + i] : 0xFFFFFFFFu;
  // thread-local suffix minima
#pragma unroll
  for (int i = DF_IPT - 2; i >= 0; i--) v[i] = min(v[i], v[i + 1]);
  // block suffix-min of the per-thread minima (v[0]); reverse inclusive scan over threads
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v[0];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_down_sync(0xffffffffu, x, d);
    if (lane + d < 32) x = min(x, y);
  }
  if (lane == 0) warp_min[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t ws = lane < DF_NT / 32 ? warp_min[lane] : 0xFFFFFFFFu;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_down_sync(0xffffffffu, ws, d);
      if (lane + d < 32) ws = min(ws, y);
    }
    if (lane < DF_NT / 32) warp_min[lane] = ws;  // inclusive suffix min over warps >= lane
    if (lane == 0) {  // look-back over the tiles to the right (running min in the value field)
      const uint64_t agg = ws;
      uint64_t carry = 0xFFFFFFFFull;
      if (rt == 0) {
        lb_store(&status[0], LB_INC | agg);
      } else {
        lb_store(&status[rt], LB_AGG | agg);
        int64_t j = (int64_t)rt - 1;
        while (true) {
          const uint64_t s = lb_load(&status[j]);
          const uint64_t f = s & ~LB_VAL;
          if (f == 0) continue;
          carry = min(carry, s & LB_VAL);
          if (f == LB_INC) break;
          --j;
        }
        lb_store(&status[rt], LB_INC | min(carry, agg));
      }
      s_carry = (uint32_t)carry;
    }
  }
  __syncthreads();
  // suffix min of the threads after me within the block, then of the tiles to the right
  uint32_t after = 0xFFFFFFFFu;
  {
    const uint32_t in_warp = __shfl_down_sync(0xffffffffu, x, 1);
    if (lane < 31) after = in_warp;
    if (lane == 31 && wid + 1 < DF_NT / 32) after = warp_min[wid + 1];
    else if (lane < 31 && wid + 1 < DF_NT / 32) after = min(after, warp_min[wid + 1]);
  }
  after = min(after, s_carry);
  // K6c fused: slot s holds the kept entries [d(s), d(s + 1)); the tile's final d values go to SMEM
  // (d(tile end) = the carry from the right), then consecutive threads write consecutive 32-B slot
  // records (coalesced) with the low-bit keys of each slot's first entries
  __shared__ uint32_t sd[DF_TILE + 1];
#pragma unroll
  for (int i = 0; i < DF_IPT; i++) sd[threadIdx.x * DF_IPT + i] = min(v[i], after);
  if (threadIdx.x == 0) sd[DF_TILE] = s_carry;
  __syncthreads();
  const uint64_t t0 = t * DF_TILE;
  for (uint32_t q = threadIdx.x; q < (uint32_t)DF_TILE; q += DF_NT) {
    const uint64_t sl = t0 + q;
    if (sl >= n_slots) break;
    const uint32_t a = sd[q], b = sd[q + 1];
    uint32_t kk[DIR_KEYS];
    if (b - a <= DIR_PAIRS) {  // the entries themselves
      dir_pairs(b - a, [&](int e) { return ent[a + e]; }, kk);
    } else if (b - a <= DIR_KEYS) {
#pragma unroll
      for (int e = 0; e < DIR_KEYS; e++) kk[e] = a + e < b ? (uint32_t)ent[a + e] >> 1 : 0xFFFFFFFFu;
    } else {
      // a long slot (frequent hashes: probed in proportion to their counts) holding <= DIR_RUNS
      // distinct keys: (key, run end) pairs, so its probes also read the record only; more keys:
      // key[0] = ~0 and the probe searches the entries
#pragma unroll
      for (int e = 0; e < DIR_KEYS; e++) kk[e] = (e & 1) ? b : 0xFFFFFFFFu;
      uint32_t s0 = a;
      int r = 0;
      for (; r < DIR_RUNS && s0 < b; r++) {
        const uint32_t ks = (uint32_t)ent[s0] >> 1;
        uint32_t lo = s0 + 1, st = 1;  // gallop, then bisect, to the first entry with another key
        while (lo + st <= b && ((uint32_t)ent[lo + st - 1] >> 1) == ks) { lo += st; st <<= 1; }
        uint32_t hi = min(lo + st - 1, b);
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (((uint32_t)ent[mid] >> 1) == ks) lo = mid + 1;
          else hi = mid;
        }
        kk[2 * r] = ks;
        kk[2 * r + 1] = lo;
        s0 = lo;
      }
      if (s0 < b) kk[0] = 0xFFFFFFFFu;
    }
    uint4* o = reinterpret_cast<uint4*>(rec + sl);
    o[0] = make_uint4(a, b, kk[0], kk[1]);
    o[1] = make_uint4(kk[2], kk[3], kk[4], kk[5]);
  }
}

__global__ void k_put_u32(uint32_t* p, uint32_t v) { *p = v; }

}  // namespace

namespace {
__global__ void k_count_queries(god::IndexView v, const uint64_t* __restrict__ hashes, uint64_t n, uint32_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint2 r = probe_range(v, hashes[i]);
    out[i] = r.y - r.x;
  }
}


// the full hash of entry e: its slot (largest s with dir[s].start <= e) gives the top bits
__device__ __forceinline__ uint64_t entry_hash(const god::IndexView& v, uint64_t e) {
  uint64_t lo = 0, hi = v.n_slots - 1;
  while (lo < hi) {
    uint64_t mid = (lo + hi + 1) >> 1;
    if (v.dir[mid].start <= e) lo = mid;
    else hi = mid - 1;
  }
  uint64_t top = lo;
  if (v.seg) {  // mode 1: the segment whose slot range holds slot lo = the largest t with seg[t].x <= lo
    uint32_t a = 0, b = (1u << DIR_SEG_BITS) - 1;
    while (a < b) {
      const uint32_t mid = (a + b + 1) >> 1;
      if (v.seg[mid].x <= lo) a = mid;
      else b = mid - 1;
    }
    top = a;
  }
  return (top << v.low_bits) | ((uint32_t)v.ent[e] >> 1);
}

__global__ void k_dump(god::IndexView v, uint64_t* hash, uint32_t* pos, uint8_t* strand) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < v.n_kept; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t en = v.ent[e];
    if (hash) hash[e] = entry_hash(v, e);
    if (pos) pos[e] = (uint32_t)(en >> 32);
    if (strand) strand[e] = (uint8_t)(en & 1u);
  }
}

// bin-built index (all entries held, cutoff at probe time): keep flag per entry, then the kept ones
__global__ void k_dump_flag(god::IndexView v, uint32_t* keep) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < v.n_ent; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 r = probe_range_all(v, entry_hash(v, e));
    keep[e] = (r.y - r.x) <= v.tau ? 1u : 0u;
  }
}
__global__ void k_dump_sel(god::IndexView v, const uint32_t* keep, const uint64_t* at, uint64_t* hash, uint32_t* pos,
                           uint8_t* strand) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < v.n_ent; e += (uint64_t)gridDim.x * blockDim.x) {
    if (!keep[e]) continue;
    const uint64_t o = at[e];
    const uint64_t en = v.ent[e];
    if (hash) hash[o] = entry_hash(v, e);
    if (pos) pos[o] = (uint32_t)(en >> 32);
    if (strand) strand[o] = (uint8_t)(en & 1u);
  }
}

// CTAs of a kernel resident on the whole GPU (the wave after which a tile-per-CTA grid continues)
template <typename F>
uint32_t resident_ctas(F kernel, int nt, size_t smem) {
  int per_sm = 0;
  GOD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nt, smem));
  return (uint32_t)std::max(1, per_sm) * (uint32_t)num_sms();
}

inline uint32_t floor_log2(uint64_t v) { return v ? 63u - (uint32_t)__builtin_clzll(v) : 0u; }
}  // namespace


void build_index(const Params& P, const uint8_t* ref, const uint64_t* ref_offsets, uint32_t n_refs,
                 const god_cutoff& cut, god_index* ix, cudaStream_t st, const SeqStream* ss) {
  Scratch scr(st, POOL_BUILD);
  ix->P = P;
  memset(&ix->st, 0, sizeof(ix->st));
  ix->st.k = P.k; ix->st.w = P.w; ix->st.p = P.pat.p; ix->st.x = P.pat.x;
  // K1: reference minimizers, position order (phase 0, global positions)
  NvtxRange nvtx12("stage 1+2: sparsify + minimizers (K1)");
  JobSet js = make_jobs(P, ref_offsets, n_refs, nullptr, 0, 0, true, st, scr);
  Records rec;
  const uint64_t est = js.total_pos / (uint64_t)(P.w + 1) * 2 + js.total_pos / 8 + 4096;
  const bool bin_sort = 2 * P.k >= 36 && 2 * P.k - SEG_BITS <= 30 && !getenv("GOD_SORT_FULL");
  // the bin sort orders every bin by the packed (hash, pos) key, so K1 may emit records in tile order
  run_extract(P, ref, js.seq_bytes, js.jobs, js.kb, js.n, js.total_pos, false, false, rec, st, scr, est, "extract_ref",
              js.x2p(), bin_sort ? ORDER_NONE : ORDER_GLOBAL, ss);
  const uint64_t n = rec.n;
  nvtxRangePop();  // (nvtx12's destructor pops the range pushed next)
  nvtxRangePushA("stage 3: sort, count, cutoff, table");
  // K2: stable LSD radix sort on the 2k hash bits
  uint64_t* k0 = rec.hz;
  uint32_t* v0 = rec.pos;
  uint32_t* segc = nullptr;  // records per top-12-bit hash segment (bin sort and directory map)
  // K3 outputs (filled by the bin sort when it runs, else by k_runs)
  RunOut ro;
  ro.hist_small = scr.alloc<uint32_t>(SMALL_BINS);
  ro.large = scr.alloc<uint32_t>(n / SMALL_BINS + 1);
  ro.n_large = scr.alloc<uint32_t>(1);
  uint64_t* nd_d = scr.alloc<uint64_t>(1);
  ro.n_distinct = reinterpret_cast<unsigned long long*>(nd_d);
  GOD_CUDA(cudaMemsetAsync(ro.hist_small, 0, SMALL_BINS * sizeof(uint32_t), st));
  GOD_CUDA(cudaMemsetAsync(ro.n_large, 0, sizeof(uint32_t), st));
  GOD_CUDA(cudaMemsetAsync(nd_d, 0, sizeof(uint64_t), st));
  bool runs_done = false;
  // K6 directory.  mode 1 (2k - 12 in [2, 30]): data-sized monotone slot map over the top-12-bit
  // segments, ~DIR_TARGET entries per slot (minimizer hashes are skewed toward small values, and so
  // are the probes; a fixed hash-bit prefix leaves ~20 entries in the dense slots).  mode 0: the top
  // B hash bits, B = clamp(floor(log2 n_kept), 2k - 31, min(2k, 28)).
  const uint32_t hb = 2 * P.k;
  const bool mode1 = hb >= 14 && hb - DIR_SEG_BITS <= 30 && !getenv("GOD_DIR_MODE0");
  const char* dt = getenv("GOD_DIR_TARGET");  // test hook: entries per slot
  const uint32_t DIR_TARGET = dt ? (uint32_t)std::max(1, atoi(dt)) : 2u;
  uint32_t B = 0, low_bits = 0;
  uint64_t n_slots = 0;
  uint2* seg = nullptr;
  bool built = false;  // the bin sort wrote the entries and the directory (bin_sort && mode1)
  uint32_t S_dir = 0;
  if (n > 1) {
    uint64_t* k1 = scr.alloc<uint64_t>(n);
    uint32_t* v1 = scr.alloc<uint32_t>(n);
    const uint32_t ntiles = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
    uint32_t* hist = scr.alloc<uint32_t>((uint64_t)(1u << BIN_DIGIT) * ntiles);
    uint64_t* goff = scr.alloc<uint64_t>((uint64_t)(1u << BIN_DIGIT) * ntiles);
    static DeviceOnce attr_once;
    attr_once.run([] {
      GOD_CUDA(cudaFuncSetAttribute(k_rs_scatter2<RS_BITS, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    rs_dyn_smem(RS_BITS, true)));
      GOD_CUDA(cudaFuncSetAttribute(k_rs_scatter2<BIN_DIGIT, true, RS_GROUP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    rs_dyn_smem(BIN_DIGIT, true)));
      GOD_CUDA(cudaFuncSetAttribute(k_rs_scatter2<BIN_DIGIT, false, RS_GROUP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    rs_dyn_smem(BIN_DIGIT, false)));
      GOD_CUDA(cudaFuncSetAttribute(k_bin_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, BS_SMEM));
      GOD_CUDA(cudaFuncSetAttribute(k_bin_build, cudaFuncAttributeMaxDynamicSharedMemorySize, BB_SMEM));
      GOD_CUDA(cudaFuncSetAttribute(k_bucket_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, BS_SMEM));
    });
    const int hbits = 2 * P.k;
    // gc: tiles per CTA / histogram column (RS_GROUP on the bin-sort path, 1 on the full LSD)
    auto lsd_pass = [&](auto rb, auto gc, int shift, int bits, bool have_hist = false, const uint2* table = nullptr,
                        int L = 0, bool stable = true) {
      constexpr int RB = decltype(rb)::value;
      constexpr int G = decltype(gc)::value;
      const uint32_t dmask = (1u << bits) - 1;
      const uint32_t ncols = (ntiles + G - 1) / G;
      if (!have_hist) GOD_LAUNCH("k_rs_hist", (k_rs_hist<RB, G>), ncols, RS_NT, 0, st, k0, n, shift, dmask, hist, ncols);
      scan_exclusive_u32_to_u64(hist, goff, (uint64_t)(1u << RB) * ncols, nullptr, st, scr, "scan_sort_hist");
      if (stable)
        GOD_LAUNCH("k_rs_scatter", (k_rs_scatter2<RB, true, G>), ncols, RS2_NT, rs_dyn_smem(RB, true), st, k0, v0, k1, v1, n,
                   shift, dmask, goff, ncols, table, L, resident_ctas(k_rs_scatter2<RB, true, G>, RS2_NT, rs_dyn_smem(RB, true)));
      else
        GOD_LAUNCH("k_rs_scatter", (k_rs_scatter2<RB, false, G>), ncols, RS2_NT, rs_dyn_smem(RB, false), st, k0, v0, k1, v1, n,
                   shift, dmask, goff, ncols, table, L, resident_ctas(k_rs_scatter2<RB, false, G>, RS2_NT, rs_dyn_smem(RB, false)));
      std::swap(k0, k1);
      std::swap(v0, v1);
    };
    if (bin_sort) {
      // K2 bin sort (see the comment above k_seg_hist)
      const int L = hbits - SEG_BITS;
      segc = scr.alloc<uint32_t>(1u << SEG_BITS);
      uint2* table = scr.alloc<uint2>(1u << SEG_BITS);
      uint32_t* n_bins_d = scr.alloc<uint32_t>(1);
      GOD_CUDA(cudaMemsetAsync(segc, 0, (1u << SEG_BITS) * sizeof(uint32_t), st));
      // large inputs: a 1/16 sample in whole 256-B blocks (k_seg_hist 0.44 -> 0.03 ms on human; the bins come
      // out within ~2% of the target, which the dynamically claimed k_bin_build absorbs.  Round 2's
      // first try, every 16th RECORD, still read every DRAM line and cost k_bin_build 0.6 ms under the
      // static bin assignment of the time)
      const uint32_t seg_stride = getenv("GOD_SEG_SAMPLE") ? (uint32_t)std::max(1, atoi(getenv("GOD_SEG_SAMPLE")))
                                                           : (n >= (1ull << 24) ? 16u : 1u);
      GOD_LAUNCH("k_seg_hist", k_seg_hist, 4u * num_sms(), 512, 0, st, k0, n, L, segc, seg_stride);
      const char* bt = getenv("GOD_BIN_TARGET");  // test hook: bin size (default BIN_TARGET)
      const uint64_t base_target = bt ? std::max(1, atoi(bt)) : BIN_TARGET;
      // Two LSD passes order up to 2^18 bins.  An input that would need bins above the target for that
      // (human '1': 517 M records) takes a third pass over the bin bits that fit above the hash instead:
      // bins beyond the SMEM capacity fall to the bitonic / global paths (measured on human '1': stage 3
      // 46 ms with 2 passes and 2125-record bins against the 2048 capacity).
      const int bin_bits_max = std::min(3 * BIN_DIGIT, 63 - hbits);
      const bool three = !getenv("GOD_BIN_2PASS") && bin_bits_max > 2 * BIN_DIGIT &&
                         ((n + n / 16) / ((1u << (2 * BIN_DIGIT)) - (1u << SEG_BITS)) + 1 > base_target ||
                          getenv("GOD_BIN_3PASS"));
      const int bin_bits = three ? bin_bits_max : 2 * BIN_DIGIT;
      const uint32_t target =
          (uint32_t)std::max<uint64_t>(base_target, (n + n / 16) / ((1ull << bin_bits) - (1u << SEG_BITS)) + 1);
      GOD_LAUNCH("k_seg_table", k_seg_table, 1, 1024, 0, st, segc, target, table, n_bins_d, seg_stride,
                 seg_stride > 1 ? 1u : 0u);
      // the first pass's tile histograms of the bins; the first scatter assigns the bins itself
      const uint32_t ncols = (ntiles + RS_GROUP - 1) / RS_GROUP;
      GOD_LAUNCH("k_seg_assign", k_seg_assign, ncols, RS_NT, 0, st, k0, n, L, hbits, table, (1u << BIN_DIGIT) - 1, hist,
                 ncols, 0);
      // the first pass need not be stable: the records arrive from K1 in tile order
      using GC = std::integral_constant<int, RS_GROUP>;
      lsd_pass(std::integral_constant<int, BIN_DIGIT>(), GC(), hbits, BIN_DIGIT, true, table, L, getenv("GOD_RS_STABLE1") != nullptr);
      lsd_pass(std::integral_constant<int, BIN_DIGIT>(), GC(), hbits + BIN_DIGIT, BIN_DIGIT);
      if (three) lsd_pass(std::integral_constant<int, BIN_DIGIT>(), GC(), hbits + 2 * BIN_DIGIT, bin_bits - 2 * BIN_DIGIT);
      const uint32_t nb = d2h_scalar(n_bins_d, st);
      uint64_t* bstart = scr.alloc<uint64_t>((uint64_t)nb + 1);
      uint32_t* big = scr.alloc<uint32_t>(nb ? nb : 1);
      uint32_t* n_big = scr.alloc<uint32_t>(4);  // [1], [2]: statistics (bins sorted by the LSD / bitonic paths); [3]: bin claims
      GOD_CUDA(cudaMemsetAsync(n_big, 0, 4 * sizeof(uint32_t), st));
      GOD_LAUNCH("k_bucket_bounds", k_bucket_bounds, grid_for((uint64_t)nb + 1, 256), 256, 0, st, k0, n, hbits, nb,
                 bstart);
      if (mode1) {
        // K5 + K6 fused into the bin sort: the directory slots are cut from the same segment table, S per
        // bin (slots_t = S * bins_t), so every bin owns whole slots; entries go to their final place
        built = true;
        S_dir = std::max(1u, std::min(S_MAX, target / DIR_TARGET));
        n_slots = (uint64_t)S_dir * nb;
        GOD_REQUIRE(n < 0xFFFFFFFFull, "index has >= 2^32 entries");
        GOD_CUDA(cudaMallocFromPoolAsync((void**)&seg, (1u << SEG_BITS) * sizeof(uint2), god_pool(POOL_INDEX), st));
        GOD_LAUNCH("k_seg_slots", k_seg_slots, (1u << SEG_BITS) / 256, 256, 0, st, table, S_dir, seg);
        GOD_CUDA(cudaMallocFromPoolAsync((void**)&ix->dir, std::max<uint64_t>(n_slots, 1) * sizeof(DirRec), god_pool(POOL_INDEX), st));
        GOD_CUDA(cudaMallocFromPoolAsync((void**)&ix->ent, n * sizeof(uint64_t), god_pool(POOL_INDEX), st));
        GOD_LAUNCH("k_bin_build", k_bin_build, (unsigned)BS_MINB * num_sms(), BS_NT, BB_SMEM, st, k0, v0, bstart, n_bins_d, L, hbits,
                   big, n_big, ro, table, nullptr, S_dir, ix->ent, ix->dir, n_big + 3);
      } else {
        GOD_LAUNCH("k_bin_sort", k_bin_sort, (unsigned)BS_MINB * num_sms(), BS_NT, BS_SMEM, st, k0, v0, bstart, n_bins_d, L, hbits, big,
                   n_big, ro);
      }
      runs_done = true;
      const uint32_t hb_big = d2h_scalar(n_big, st);
      if (getenv("GOD_DEBUG_BUCKETS"))
        fprintf(stderr, "[bins] n=%llu bins=%u target=%u big=%u lsd=%u mid=%u S=%u\n", (unsigned long long)n, nb, target,
                hb_big, d2h_scalar(n_big + 1, st), d2h_scalar(n_big + 2, st), S_dir);
      if (hb_big) {
        GOD_LAUNCH("k_bucket_sort_big", k_bucket_sort_big, std::min(hb_big, (uint32_t)(BS_BIG_MINB * num_sms())), BS_NT, BS_SMEM, st, k0,
                   v0, /*t0=*/k1, /*t1=*/k0, bstart, big, n_big, L, hbits, ro, built ? ix->ent : nullptr);
        if (built)
          GOD_LAUNCH("k_big_dir", k_big_dir, std::min(hb_big, 4u * (uint32_t)num_sms()), BS_NT, 0, st, k0, bstart, big,
                     n_big, L, hbits, table, S_dir, ix->ent, ix->dir);
      }
    } else {
      // K2 full stable LSD over the 2k hash bits (position order kept within equal hashes)
      for (int shift = 0; shift < hbits; shift += RS_BITS)
        lsd_pass(std::integral_constant<int, RS_BITS>(), std::integral_constant<int, 1>(), shift, std::min(RS_BITS, hbits - shift));
    }
  }
  // K3: runs (distinct hashes) + count histogram (unless the bin sort produced them); K4: tau
  uint32_t* hist_small = ro.hist_small;
  uint32_t* large = ro.large;
  uint32_t* n_large = ro.n_large;
  CutState* cs = scr.alloc<CutState>(1);
  if (n && !runs_done)
    GOD_LAUNCH("k_runs", k_runs, min(grid_for(n, 512), 8u * num_sms()), 512, 0, st, k0, n, ro);
  GOD_LAUNCH("k_tau", k_tau, 1, 1024, 0, st, hist_small, large, n_large, nd_d, n, cut.mode, cut.frac_num, cut.frac_den, cut.max_occ, cs);
  CutState hcs;
  d2h_small(&hcs, cs, sizeof(CutState), st);
  GOD_CUDA(cudaStreamSynchronize(st));
  const uint64_t nd = hcs.n_distinct;
  const uint64_t n_kept = hcs.kept_entries;
  GOD_REQUIRE(n_kept < 0xFFFFFFFFull, "index has >= 2^32 kept entries");
  if (built) {
    low_bits = hb - DIR_SEG_BITS;
    B = floor_log2(n_slots);
  } else if (mode1) {
    if (!segc) {
      segc = scr.alloc<uint32_t>(1u << SEG_BITS);
      GOD_CUDA(cudaMemsetAsync(segc, 0, (1u << SEG_BITS) * sizeof(uint32_t), st));
      if (n) GOD_LAUNCH("k_seg_hist", k_seg_hist, 4u * num_sms(), 512, 0, st, k0, n, (int)(hb - SEG_BITS), segc, 1u);
    }
    GOD_CUDA(cudaMallocFromPoolAsync((void**)&seg, (1u << SEG_BITS) * sizeof(uint2), god_pool(POOL_INDEX), st));
    uint32_t* ns_d = scr.alloc<uint32_t>(1);
    GOD_LAUNCH("k_seg_table", k_seg_table, 1, 1024, 0, st, segc, DIR_TARGET, seg, ns_d);
    n_slots = d2h_scalar(ns_d, st);
    if (n_slots == 0) n_slots = 1;
    low_bits = hb - DIR_SEG_BITS;
    B = floor_log2(n_slots);
  } else {
    const uint32_t lg = floor_log2(n_kept ? n_kept : 1);
    B = lg;
    const uint32_t Bmin = hb > 31 ? hb - 31 : 0;
    const uint32_t Bmax = hb < 28 ? hb : 28;
    B = B < Bmin ? Bmin : (B > Bmax ? Bmax : B);
    low_bits = hb - B;
    n_slots = 1ull << B;
  }
  ix->st.n_entries_all = n;
  ix->st.n_distinct_all = nd;
  ix->st.m = hcs.m;
  ix->st.tau = hcs.tau;
  ix->st.kept_entries = n_kept;
  ix->st.dropped_entries = n - n_kept;
  ix->st.kept_distinct = hcs.kept_distinct;
  ix->st.dropped_distinct = nd - hcs.kept_distinct;
  ix->st.dir_bits = B;
  ix->st.dir_mode = mode1 ? 1u : 0u;
  ix->st_alloc = st;
  ix->seg = seg;
  ix->low_bits = low_bits;
  ix->n_slots = n_slots;
  if (built) {  // every entry is in ent; hashes above tau are dropped at probe time
    ix->n_ent = n;
    ix->tau_probe = (uint32_t)std::min<uint64_t>(hcs.tau, 0xFFFFFFFEull);
    GOD_CUDA(cudaStreamSynchronize(st));
    return;
  }
  ix->n_ent = n_kept;
  ix->tau_probe = 0xFFFFFFFFu;
  GOD_CUDA(cudaMallocFromPoolAsync((void**)&ix->dir, n_slots * sizeof(DirRec), god_pool(POOL_INDEX), st));
  uint32_t* dir1 = scr.alloc<uint32_t>(n_slots + 1);  // first entry per slot (+ n_kept), then pairs
  GOD_CUDA(cudaMallocFromPoolAsync((void**)&ix->ent, (n_kept ? n_kept : 1) * sizeof(uint64_t), god_pool(POOL_INDEX), st));
  const uint64_t nd1 = n_slots + 1;
  GOD_CUDA(cudaMemsetAsync(dir1, 0xFF, nd1 * sizeof(uint32_t), st));
  if (n) {  // K5: kept entries (+ K6a: the first entry of every non-empty slot)
    const uint64_t tiles = (n + KW_TILE - 1) / KW_TILE;
    uint64_t* kst = scr.alloc<uint64_t>(tiles);
    uint32_t* kctr = scr.alloc<uint32_t>(1);
    GOD_CUDA(cudaMemsetAsync(kst, 0, tiles * sizeof(uint64_t), st));
    GOD_CUDA(cudaMemsetAsync(kctr, 0, sizeof(uint32_t), st));
    GOD_LAUNCH("k_keep_write", k_keep_write, (unsigned)tiles, KW_NT, 0, st, k0, v0, n, (int)(2 * P.k), cs, ix->view(),
               ix->ent, dir1, kst, kctr);
  }
  GOD_LAUNCH("k_put_u32", k_put_u32, 1, 1, 0, st, dir1 + n_slots, (uint32_t)n_kept);
  {  // K6b + K6c: suffix minimum over the slots, then the 32-B slot records, one pass
    const uint64_t nt = (nd1 + DF_TILE - 1) / DF_TILE;
    uint64_t* dst = scr.alloc<uint64_t>(nt);
    uint32_t* dctr = scr.alloc<uint32_t>(1);
    GOD_CUDA(cudaMemsetAsync(dst, 0, nt * sizeof(uint64_t), st));
    GOD_CUDA(cudaMemsetAsync(dctr, 0, sizeof(uint32_t), st));
    GOD_LAUNCH("k_dir_suffix_min", k_dir_suffix_min, (unsigned)nt, DF_NT, 0, st, dir1, nd1, dst, dctr, ix->ent,
               n_slots, ix->dir);
  }
  GOD_CUDA(cudaStreamSynchronize(st));
  if (const char* dd = getenv("GOD_DEBUG_DIR")) {  // developer aid: dump the intermediates
    auto dump = [&](const char* name, const void* p, size_t bytes) {
      std::vector<char> h(bytes);
      cudaMemcpy(h.data(), p, bytes, cudaMemcpyDeviceToHost);
      std::string f = std::string(dd) + "/" + name + ".bin";
      FILE* fp = fopen(f.c_str(), "wb");
      if (fp) { fwrite(h.data(), 1, bytes, fp); fclose(fp); }
    };
    dump("rec_hz", rec.hz, n * 8); dump("sorted_hz", k0, n * 8); dump("sorted_pos", v0, n * 4);
    dump("dir1", dir1, (n_slots + 1) * 4);
    dump("ent", ix->ent, n_kept * 8); dump("dir", ix->dir, n_slots * sizeof(DirRec));
  }
}

void index_count(const god_index* ix, const uint64_t* hashes, uint64_t n, uint32_t* counts, cudaStream_t st) {
  if (!n) return;
  GOD_LAUNCH("k_count_queries", k_count_queries, grid_for(n, 256), 256, 0, st, ix->view(), hashes, n, counts);
}

void index_dump(const god_index* ix, uint64_t* hash, uint32_t* pos, uint8_t* strand, cudaStream_t st) {
  if (!ix->st.kept_entries) return;
  if (ix->tau_probe == 0xFFFFFFFFu) {  // ent holds exactly the kept entries
    GOD_LAUNCH("k_dump", k_dump, grid_for(ix->st.kept_entries, 256), 256, 0, st, ix->view(), hash, pos, strand);
    return;
  }
  Scratch scr(st);
  const uint64_t n = ix->n_ent;
  uint32_t* keep = scr.alloc<uint32_t>(n);
  uint64_t* at = scr.alloc<uint64_t>(n);
  uint64_t* tot = scr.alloc<uint64_t>(1);
  GOD_LAUNCH("k_dump_flag", k_dump_flag, grid_for(n, 256), 256, 0, st, ix->view(), keep);
  scan_exclusive_u32_to_u64(keep, at, n, tot, st, scr, "scan_dump");
  GOD_LAUNCH("k_dump_sel", k_dump_sel, grid_for(n, 256), 256, 0, st, ix->view(), keep, at, hash, pos, strand);
  GOD_CUDA(cudaStreamSynchronize(st));
}

}  // namespace god
