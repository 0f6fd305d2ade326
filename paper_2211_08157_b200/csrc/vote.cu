// vote.cu — location voting (section 3.4; Fig. 8) with the rescue location
// (P:398), on the anchors of god_seed_reads.  Readings V1-V6: DESIGN.md §2 / include/god.h.
//
// Per read, every anchor becomes a unique 64-bit sort key
//     strand << 63 | (diag + 2^32) << 29 | fp << ib | i
// i = the anchor's index in the read (ib = max(5, ceil(log2 n)) bits: the key carries its payload);
// fp = the top 29 - ib bits of a mix of the canonical k-mer of the anchor's read minimizer (equal
// canonical k-mer <=> equal hash, H_k being a bijection); diag fits 34 bits (forward ref - read in
// (-2^32, 2^32), reverse ref + read_end in [0, 2^33)).  Sorting the keys is step (2) ("a single
// sorted list of all adjusted matching locations").  All anchors of a true location share one
// (strand, diag), so V2's "(hash, strand, diag) once" must not compare every pair of the group: the
// fingerprint orders each (strand, diag) group by hash, and only neighbours with equal
// (strand, diag, fp) compare their exact canonical k-mers.  The canonical k-mer is read from the
// read's bytes once per read minimizer (anchors of one minimizer share read_pos).  The sweep (step
// (3)) follows the chain of cluster heads: the next Delta0 is the first anchor beyond Delta0 + D.
//
// Reads are bucketed by anchor count n: n <= 16 / n <= 32 -> 16 / 32 lanes per read, everything in
// registers (shuffle bitonic sort, ballots); n <= 128 / n <= 512 -> one warp per read on a 3 / 12 KB
// shared-memory slice; n <= 2048 -> one CTA per read in shared memory; larger -> one CTA per read
// on global scratch.
// Results go to per-read slots (max(1, min(n / V, max_pairs)) each: winners are disjoint clusters of
// >= V votes); a scan of the per-read counts and a
// compaction give the CSR output.
#include <algorithm>

#include "internal.cuh"

namespace god {
namespace {

constexpr uint64_t DIAG_MASK = (1ull << 34) - 1;   // of dk = key >> 29: strand at bit 34, biased diag below
constexpr int64_t DIAG_BIAS = 1ll << 32;
constexpr uint32_t VOTE_IDX_MAX = 1u << 29;        // anchors per read
constexpr uint32_t VOTE_WSM = 128;                 // warp-per-read shared-memory path (8 warps per CTA)
constexpr uint32_t VOTE_WSM2 = 512;                // ... larger slices (4 warps per CTA)
constexpr uint32_t VOTE_MID = 2048;                // CTA-per-read shared-memory path
constexpr int VOTE_NT = 256;
constexpr unsigned FULL = 0xffffffffu;

struct VoteArgs {
  const uint8_t* reads;
  const uint64_t* roff;
  const uint8_t* ph;
  const god_anchor* an;
  const uint64_t* aoff;
  Pattern pat;
  int32_t k;
  uint32_t D, V, mp;
  const uint64_t* slot_off;   // first result slot of each read
  god_vote* res;              // result slots
  uint32_t* cnt;              // results per read
  uint32_t* bad;              // anchors inconsistent with the phases
  bool an16;                  // an is 16-B aligned: one 128-bit load per anchor
};

__device__ __forceinline__ god_anchor load_anchor(const VoteArgs& A, uint64_t i) {
  if (A.an16) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(A.an) + i);
    return god_anchor{u.x, u.y, u.z, u.w};
  }
  return A.an[i];
}

// Read coordinates are < 2^32 (god.h limits): 32-bit pattern arithmetic, with the divisions by p
// and x short-cut for the paper's patterns ('1': p = 1; '10': p = 2, x = 1).
__device__ __forceinline__ uint32_t div_p(const Pattern& P, uint32_t d, uint32_t& rem) {
  if (P.p == 1) { rem = 0; return d; }
  if (P.p == 2) { rem = d & 1u; return d >> 1; }
  rem = d % P.p;
  return d / P.p;
}
__device__ __forceinline__ uint32_t div_x(const Pattern& P, uint32_t q, uint32_t& rem) {
  if (P.x == 1) { rem = 0; return q; }
  rem = q % P.x;
  return q / P.x;
}
__device__ __forceinline__ bool is_included(const Pattern& P, uint32_t pos, uint32_t a) {
  uint32_t rem;
  div_p(P, pos - a, rem);
  return pos >= a && ((P.bits >> rem) & 1ull);
}
// patterned index q of an included original position (inverse of orig_of)
__device__ __forceinline__ uint32_t q_of(const Pattern& P, uint32_t pos, uint32_t a) {
  uint32_t rem;
  const uint32_t blk = div_p(P, pos - a, rem);
  return blk * P.x + P.ones_before[rem];
}
__device__ __forceinline__ uint32_t orig32(const Pattern& P, uint32_t q, uint32_t a) {
  uint32_t rem;
  const uint32_t blk = div_x(P, q, rem);
  return a + blk * P.p + P.one[rem];
}

// canonical k-mer of the read's patterned k-mer starting at original position pos (phase a)
__device__ uint64_t canon_at_generic(const uint8_t* rd, uint32_t L, const Pattern& P, uint32_t a, int k, uint32_t pos) {
  const uint32_t q = q_of(P, pos, a);
  uint32_t rr;
  uint32_t base = a + div_x(P, q, rr) * P.p;
  uint64_t fwd = 0, rev = 0;
  for (int i = 0; i < k; i++) {
    const uint32_t o = base + P.one[rr];
    if (++rr == P.x) { rr = 0; base += P.p; }
    const uint32_t c = o < L ? (base_code(__ldg(rd + o)) & 3u) : 0u;
    fwd = (fwd << 2) | c;
    rev |= (uint64_t)(3u - c) << (2 * i);
  }
  return fwd < rev ? fwd : rev;
}

// x = 1 and p <= 2 ('1', '10', '01'): the k bases sit at pos + i p.  Aligned 32-bit loads (each
// holds >= 1 byte of the k-mer's span, so none can fault), 2-bit codes of 4 bytes at once
// (A0 C1 G2 T3 either case; a minimizer k-mer has no N), the reverse complement by bit reversal.
__device__ uint64_t canon_at(const uint8_t* rd, uint32_t L, const Pattern& P, uint32_t a, int k, uint32_t pos) {
  if (P.x != 1 || P.p > 2 || pos + (uint32_t)(k - 1) * P.p >= L)
    return canon_at_generic(rd, L, P, a, k, pos);
  const uintptr_t pb = reinterpret_cast<uintptr_t>(rd + pos), pa = pb & ~(uintptr_t)3;
  const uint32_t sh = (uint32_t)(pb - pa);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(pa);
  uint64_t fwd = 0;
  int got;  // codes shifted in
  if (P.p == 1) {
    const int nw = (int)((sh + (uint32_t)k + 3) >> 2);
    for (int i = 0; i < nw; i++) {
      const uint32_t v = __ldg(w + i);
      const uint32_t c = ((v >> 1) ^ (v >> 2)) & 0x03030303u;
      fwd = (fwd << 8) | ((c * 0x40100401u) >> 24);  // the 4 codes, first byte most significant
    }
    got = 4 * nw;
    fwd >>= 2 * (got - (int)sh - k);
  } else {
    const uint32_t span = sh + 2u * (uint32_t)(k - 1) + 1u;
    const int nw = (int)((span + 3) >> 2);
    const uint32_t odd = sh & 1u;  // the k-mer's bytes are the odd (or even) bytes of each word
    for (int i = 0; i < nw; i++) {
      const uint32_t v = __ldg(w + i) >> (8 * odd);
      const uint32_t c = ((v >> 1) ^ (v >> 2)) & 0x00030003u;
      fwd = (fwd << 4) | ((c << 2) & 0xCu) | (c >> 16);
    }
    got = 2 * nw;
    fwd >>= 2 * (got - (int)(sh >> 1) - k);
  }
  const uint64_t m = (1ull << (2 * k)) - 1;
  fwd &= m;
  // reverse complement: complement, reverse the order of the 2-bit codes
  uint64_t x = __brevll(~fwd);
  x = ((x >> 1) & 0x5555555555555555ull) | ((x & 0x5555555555555555ull) << 1);
  const uint64_t rev = x >> (64 - 2 * k);
  return fwd < rev ? fwd : rev;
}

__device__ __forceinline__ uint32_t idx_bits(uint32_t n) {
  const uint32_t b = n <= 1 ? 0 : 32 - __clz(n - 1);
  return b < 5 ? 5 : b;
}

// V1: the sort key of one anchor (fingerprint of its canonical k-mer in the bits below the diag).
// Sets bad if the anchor cannot come from this read and phase.
__device__ __forceinline__ uint64_t vote_key(const VoteArgs& A, const god_anchor& an, uint32_t a, uint32_t L,
                                             uint64_t canon, uint32_t ib, uint32_t i, bool& bad) {
  const uint32_t z = an.strand & 1u;
  if (an.read_pos >= L || !is_included(A.pat, an.read_pos, a)) bad = true;
  int64_t diag;
  if (z == 0) {
    diag = (int64_t)an.ref_pos - (int64_t)an.read_pos;
  } else {
    const uint32_t end = orig32(A.pat, q_of(A.pat, an.read_pos, a) + (uint32_t)A.k - 1, a);
    if (end >= L) bad = true;
    diag = (int64_t)an.ref_pos + (int64_t)end;
  }
  const uint32_t fb = 29 - ib;
  const uint64_t fp = fb ? ((canon * 0x9E3779B97F4A7C15ull) >> (64 - fb)) : 0ull;
  return ((uint64_t)z << 63) | ((uint64_t)(diag + DIAG_BIAS) << 29) | (fp << ib) | i;
}

__device__ __forceinline__ int64_t dk_diag(uint64_t dk) { return (int64_t)(dk & DIAG_MASK) - DIAG_BIAS; }

// is anchor dk beyond the cluster head dh: other strand, or diag - Delta0 > D (dk >= dh: sorted)
__device__ __forceinline__ bool beyond(uint64_t dk, uint64_t dh, uint64_t D) {
  return (dk >> 34) != (dh >> 34) || (dk & DIAG_MASK) - (dh & DIAG_MASK) > D;
}

// V4 order of two clusters: more votes first, then strand, then Delta0 (dk orders (strand, diag))
__device__ __forceinline__ bool better(uint32_t va, uint64_t da, uint32_t vb, uint64_t db) {
  return va > vb || (va == vb && da < db);
}

__device__ __forceinline__ void put_result(const VoteArgs& A, uint32_t r, uint32_t rank, uint64_t dh, uint32_t votes,
                                           uint32_t rescued, uint32_t rlo, uint32_t rhi, uint32_t qlo, uint32_t qhi) {
  god_vote v;
  v.read_id = r;
  v.strand = (uint32_t)(dh >> 34);
  v.diag = dk_diag(dh);
  v.votes = votes;
  v.rescued = rescued;
  v.ref_lo = rlo;
  v.ref_hi = rhi;
  v.read_lo = qlo;
  v.read_hi = qhi;
  A.res[A.slot_off[r] + rank] = v;
}

// ------------------------------------------------------------------ bucketing + result slots
constexpr int VC_NT = 1024;   // classify: one list reservation per class and block of 1024 reads
constexpr int VC_CLASSES = 6;
__global__ void __launch_bounds__(VC_NT) k_vote_classify(const uint64_t* __restrict__ aoff, uint32_t n_reads,
                                                         uint32_t mp, uint32_t V, uint64_t* __restrict__ slots,
                                                         uint32_t* __restrict__ lists, uint32_t* __restrict__ nlist,
                                                         uint64_t* __restrict__ big_off,
                                                         uint64_t* __restrict__ big_total, uint32_t* __restrict__ bad) {
  constexpr int NW = VC_NT / 32;
  __shared__ uint32_t s_cnt[VC_CLASSES][NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t r0 = blockIdx.x * blockDim.x; r0 < n_reads; r0 += stride) {  // block-uniform trip count
    const uint32_t r = r0 + threadIdx.x;
    uint64_t n = 0;
    if (r < n_reads) {
      n = aoff[r + 1] - aoff[r];
      // result slots: winners are disjoint clusters of >= V votes (each vote an anchor), so at most
      // n / V of them (max_pairs caps it further); a rescue location needs one
      uint64_t sl = n / (V ? V : 1u);
      if (mp && sl > mp) sl = mp;
      slots[r] = n == 0 ? 0 : (sl ? sl : 1);
    }
    if (n >= VOTE_IDX_MAX) { atomicAdd(bad + 1, 1u); n = 0; }
    const int c = n == 0 ? -1 : n <= 16 ? 0 : n <= 32 ? 1 : n <= VOTE_WSM ? 2 : n <= VOTE_WSM2 ? 3 : n <= VOTE_MID ? 4 : 5;
    uint32_t mine = 0;  // ballot of this lane's class
#pragma unroll
    for (int q = 0; q < VC_CLASSES; q++) {
      const uint32_t m = __ballot_sync(FULL, c == q);
      if (c == q) mine = m;
      if (lane == 0) s_cnt[q][warp] = __popc(m);
    }
    __syncthreads();
    if (threadIdx.x < VC_CLASSES) {  // one reservation per class: exclusive prefix over the warps
      const int q = threadIdx.x;
      uint32_t tot = 0;
      for (int w = 0; w < NW; w++) { const uint32_t x = s_cnt[q][w]; s_cnt[q][w] = tot; tot += x; }
      const uint32_t base = tot ? atomicAdd(nlist + q, tot) : 0u;
      for (int w = 0; w < NW; w++) s_cnt[q][w] += base;
    }
    __syncthreads();
    if (c >= 0) {
      const uint32_t j = s_cnt[c][warp] + __popc(mine & ((1u << lane) - 1u));
      lists[(uint64_t)c * n_reads + j] = r;
      if (c == 5) big_off[j] = atomicAdd((unsigned long long*)big_total, (unsigned long long)(n + 2));
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ n <= SEG: SEG lanes per read, registers
// SEG = 16 (two reads per warp) or 32.  Every loop that shuffles runs a warp-uniform trip count.
template <int SEG>
__global__ void __launch_bounds__(VOTE_NT) k_vote_warp(VoteArgs A, const uint32_t* __restrict__ list, uint32_t nlist) {
  constexpr uint32_t SB = SEG == 32 ? FULL : ((1u << SEG) - 1u);
  const int lane = threadIdx.x & 31, sl = lane & (SEG - 1), sbase = lane & ~(SEG - 1);
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / SEG;
  if (__all_sync(FULL, gw >= nlist)) return;  // warp-uniform
  const bool active = gw < nlist;
  const uint32_t r = active ? list[gw] : 0u;
  const uint64_t a0 = active ? A.aoff[r] : 0;
  const uint32_t n = active ? (uint32_t)(A.aoff[r + 1] - a0) : 0u;
  const uint64_t rb = active ? A.roff[r] : 0;
  const uint32_t L = active ? (uint32_t)(A.roff[r + 1] - rb) : 0u;
  const uint32_t ph = active ? A.ph[r] : 0u;
  const uint64_t D = A.D ? A.D : L;
  const bool valid = sl < (int)n;
  const uint32_t le = (sl == 31) ? FULL : ((2u << sl) - 1u);
  auto ballot = [&](bool p) { return (__ballot_sync(FULL, p) >> sbase) & SB; };
  god_anchor an = {0, 0, 0, 0};
  if (valid) an = load_anchor(A, a0 + sl);
  // canonical k-mer once per read minimizer (a run of equal read_pos), then broadcast
  const uint32_t prev_rp = __shfl_up_sync(FULL, an.read_pos, 1, SEG);
  const bool rhead = valid && (sl == 0 || prev_rp != an.read_pos);
  uint64_t canon = 0;
  if (rhead && an.read_pos < L && is_included(A.pat, an.read_pos, ph))
    canon = canon_at(A.reads + rb, L, A.pat, ph, A.k, an.read_pos);
  const uint32_t hm = ballot(rhead) & le;
  canon = __shfl_sync(FULL, canon, hm ? 31 - __clz(hm) : 0, SEG);
  bool bad = false;
  uint64_t key = ~0ull;
  if (valid) key = vote_key(A, an, ph, L, canon, 5, (uint32_t)sl, bad);
  const bool seg_bad = ballot(bad) != 0;
  if (seg_bad && sl == 0) atomicAdd(A.bad, 1u);
  // step (2): bitonic sort of the SEG keys (pads ~0 sink to the end)
#pragma unroll
  for (int size = 2; size <= SEG; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t o = __shfl_xor_sync(FULL, key, stride);
      const bool up = (sl & size) == 0 || size == SEG;
      const bool lower = (sl & stride) == 0;
      key = (lower == up) ? (key < o ? key : o) : (key > o ? key : o);
    }
  }
  const int src = (int)(key & 31u);
  const uint32_t ref = __shfl_sync(FULL, an.ref_pos, src, SEG);
  const uint32_t qp = __shfl_sync(FULL, an.read_pos, src, SEG);
  const uint64_t cn = __shfl_sync(FULL, canon, src, SEG);
  const uint64_t dk = key >> 29;
  // V2: a repeat of (hash, strand, diag) is no new vote: walk back over equal (strand, diag, fp)
  bool dup = false, walking = valid;
  for (int o = 1; __any_sync(FULL, walking); o++) {
    const uint64_t ko = __shfl_up_sync(FULL, key, o, SEG);
    const uint64_t co = __shfl_up_sync(FULL, cn, o, SEG);
    if (walking) {
      if (sl < o || (ko >> 5) != (key >> 5)) walking = false;
      else if (co == cn) { dup = true; walking = false; }
    }
  }
  // step (3): the chain of cluster heads
  uint32_t starts = 0, s = 0;
  while (__any_sync(FULL, s < n)) {
    const bool live = s < n;
    const uint64_t dh = __shfl_sync(FULL, dk, live ? (int)s : 0, SEG);
    const uint32_t b = ballot(valid && sl > (int)s && beyond(dk, dh, D));
    if (live) {
      starts |= 1u << s;
      s = b ? (uint32_t)(__ffs(b) - 1) : n;
    }
  }
  const int cid = __popc(starts & le) - 1;
  const uint32_t newmask = ballot(valid && !dup);
  // member spans: segmented suffix min/max (clusters are contiguous)
  uint32_t rlo = ref, rhi = ref, qlo = qp, qhi = qp;
#pragma unroll
  for (int o = 1; o < SEG; o <<= 1) {
    const uint32_t a1 = __shfl_down_sync(FULL, rlo, o, SEG), a2 = __shfl_down_sync(FULL, rhi, o, SEG);
    const uint32_t a3 = __shfl_down_sync(FULL, qlo, o, SEG), a4 = __shfl_down_sync(FULL, qhi, o, SEG);
    const int oc = __shfl_down_sync(FULL, cid, o, SEG);
    if (sl + o < (int)n && oc == cid) {
      rlo = min(rlo, a1); rhi = max(rhi, a2); qlo = min(qlo, a3); qhi = max(qhi, a4);
    }
  }
  const bool head = valid && ((starts >> sl) & 1u);
  uint32_t votes = 0;
  if (head) {
    const uint32_t after = starts & ~le;
    const uint32_t e = after ? (uint32_t)(__ffs(after) - 1) : n;
    const uint32_t range = (e >= 32 ? FULL : ((1u << e) - 1u)) & ~((1u << sl) - 1u);
    votes = __popc(newmask & range);
  }
  // step (4) / rescue
  const uint32_t winmask = ballot(head && votes >= A.V);
  const bool rescue = winmask == 0;
  const uint32_t candmask = rescue ? starts : winmask;
  const bool cand = (candmask >> sl) & 1u;
  uint32_t rank = 0;
  for (uint32_t m = candmask; __any_sync(FULL, m != 0);) {
    const int j = m ? __ffs(m) - 1 : 0;
    const uint32_t vj = __shfl_sync(FULL, votes, j, SEG);
    const uint64_t dj = __shfl_sync(FULL, dk, j, SEG);
    if (m) {
      rank += j != sl && better(vj, dj, votes, dk);
      m &= m - 1;
    }
  }
  const uint32_t limit = rescue ? 1u : (A.mp ? A.mp : 32u);
  if (!active || seg_bad) return;
  if (cand && rank < limit) put_result(A, r, rank, dk, votes, rescue ? 1u : 0u, rlo, rhi, qlo, qhi);
  if (sl == 0) A.cnt[r] = n ? min((uint32_t)__popc(candmask), limit) : 0u;
}

// ------------------------------------------------------------------ n > 32: a group of NT threads per read
// NT = 32 (one warp, shared-memory slice) or VOTE_NT (one CTA, shared memory or global scratch).
// Arrays of a read with n anchors: key[n], canon[n] (until the new-vote flags are set; its bytes
// then hold chead[n + 1] (cluster heads) and cv[n] (votes)), aux[n] (read_pos, then new-vote flags,
// then their prefix), crank[n] (run heads, then cluster-head flags, then the winner list); ctr[4]
// (clusters, winners, bad, new votes).
struct GroupArrays {
  uint64_t* key;
  uint64_t* canon;
  uint32_t* aux;
  uint32_t* chead;
  uint32_t* cv;
  uint32_t* crank;
  uint32_t* ctr;
};

template <int NT>
__device__ __forceinline__ void gsync() {
  if (NT == 32) __syncwarp();
  else __syncthreads();
}

// Exclusive scan of two 0/1 flag arrays over [0, n) by a group of NT threads (chunks of NT):
// fa -> heads (compacted indices of the set flags into `out`, count returned via *total_a),
// fb -> exclusive prefix written over fb (total via *total_b).
template <int NT>
__device__ void group_scan_flags(uint32_t n, const uint32_t* fa, uint32_t* out, uint32_t* fb, uint32_t* ws,
                                 uint32_t* total_a, uint32_t* total_b, int t) {
  const int lane = t & 31, warp = t >> 5;
  constexpr int NW = NT / 32;
  uint32_t base_a = 0, base_b = 0;
  for (uint32_t c0 = 0; c0 < n; c0 += NT) {
    const uint32_t i = c0 + t;
    const uint32_t a = i < n ? fa[i] : 0u, b = i < n ? fb[i] : 0u;
    const uint32_t ba = __ballot_sync(FULL, a), bb = __ballot_sync(FULL, b);
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t pa = __popc(ba & lt), pb = __popc(bb & lt);
    uint32_t wa = 0, wb = 0, ta = __popc(ba), tb = __popc(bb);
    if (NW > 1) {
      if (lane == 0) { ws[warp] = ta; ws[NW + warp] = tb; }
      __syncthreads();
      ta = 0; tb = 0;
      for (int q = 0; q < NW; q++) {
        const uint32_t xa = ws[q], xb = ws[NW + q];
        if (q < warp) { wa += xa; wb += xb; }
        ta += xa; tb += xb;
      }
      __syncthreads();
    }
    if (a) out[base_a + wa + pa] = i;
    if (i < n) fb[i] = base_b + wb + pb;
    base_a += ta;
    base_b += tb;
  }
  if (t == 0) { *total_a = base_a; *total_b = base_b; }
}

// hidx[i] = the largest h <= i starting a run of equal rp (h == 0 or rp[h-1] != rp[h]), by a
// chunked max-scan over the group (NT = 32: one warp; else warps combined through ws)
template <int NT>
__device__ void group_head_scan(uint32_t n, const uint32_t* rp, uint32_t* hidx, uint32_t* ws, int t) {
  const int lane = t & 31, warp = t >> 5;
  constexpr int NW = NT / 32;
  uint32_t carry = 0;
  for (uint32_t c0 = 0; c0 < n; c0 += NT) {
    const uint32_t i = c0 + t;
    uint32_t v = (i < n && (i == 0 || rp[i - 1] != rp[i])) ? i : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(FULL, v, o);
      if (lane >= o) v = max(v, u);
    }
    uint32_t chunk_max;
    if (NW > 1) {
      if (lane == 31) ws[warp] = v;
      __syncthreads();
      uint32_t before = 0;
      chunk_max = 0;
      for (int q = 0; q < NW; q++) {
        if (q < warp) before = max(before, ws[q]);
        chunk_max = max(chunk_max, ws[q]);
      }
      __syncthreads();
      v = max(v, before);
    } else {
      chunk_max = __shfl_sync(FULL, v, 31);
    }
    v = max(v, carry);
    if (i < n) hidx[i] = v;
    carry = max(carry, chunk_max);
  }
}

template <int NT>
__device__ void vote_group(const VoteArgs& A, uint32_t r, const GroupArrays& S, uint32_t* ws, int t) {
  const int lane = t & 31, warp = t >> 5;
  constexpr int NW = NT / 32;
  const uint64_t a0 = A.aoff[r];
  const uint32_t n = (uint32_t)(A.aoff[r + 1] - a0);
  const uint64_t rb = A.roff[r];
  const uint32_t L = (uint32_t)(A.roff[r + 1] - rb);
  const uint32_t ph = A.ph[r];
  const uint64_t D = A.D ? A.D : L;
  const uint32_t ib = idx_bits(n);
  const uint64_t imask = (1ull << ib) - 1;
  if (t == 0) { S.ctr[0] = 0; S.ctr[1] = 0; S.ctr[2] = 0; S.ctr[3] = 0; }
  for (uint32_t i = t; i < n; i += NT) S.aux[i] = __ldg(&A.an[a0 + i].read_pos);
  gsync<NT>();
  // canonical k-mer once per read minimizer (heads of runs of equal read_pos)
  for (uint32_t i = t; i < n; i += NT) {
    const uint32_t rp = S.aux[i];
    if ((i == 0 || S.aux[i - 1] != rp) && rp < L && is_included(A.pat, rp, ph))
      S.canon[i] = canon_at(A.reads + rb, L, A.pat, ph, A.k, rp);
  }
  gsync<NT>();
  // head of each run of equal read_pos (one read minimizer): segmented max-scan of head indices
  group_head_scan<NT>(n, S.aux, S.crank, ws, t);
  gsync<NT>();
  // keys; a non-head takes its head's canonical k-mer (heads are not written in this phase)
  bool bad = false;
  for (uint32_t i = t; i < n; i += NT) {
    const god_anchor an = load_anchor(A, a0 + i);
    const uint32_t j = S.crank[i];
    uint64_t c = 0;
    if (an.read_pos < L && is_included(A.pat, an.read_pos, ph)) c = S.canon[j];
    if (j != i) S.canon[i] = c;
    S.key[i] = vote_key(A, an, ph, L, c, ib, i, bad);
  }
  if (bad) S.ctr[2] = 1;
  gsync<NT>();
  if (S.ctr[2]) {
    if (t == 0) atomicAdd(A.bad, 1u);
    return;
  }
  // step (2): bitonic sort, all comparators ascending (mirror first step), virtual +inf past n
  // (strides are powers of two: index arithmetic by shifts)
  uint32_t lg = 0;
  while ((1u << lg) < n) ++lg;
  const uint32_t N2 = 1u << lg;
  for (uint32_t ls = 1; ls <= lg; ++ls) {  // size = 2^ls
    const uint32_t lh = ls - 1, half = 1u << lh;
    for (uint32_t q = t; q < N2 / 2; q += NT) {
      const uint32_t base = (q >> lh) << ls, off = q & (half - 1);
      const uint32_t i = base + off, j = base + (2u * half) - 1 - off;
      if (j < n) {
        const uint64_t x = S.key[i], y = S.key[j];
        if (y < x) { S.key[i] = y; S.key[j] = x; }
      }
    }
    gsync<NT>();
    for (int lstr = (int)lh - 1; lstr >= 0; --lstr) {
      const uint32_t stride = 1u << lstr;
      for (uint32_t q = t; q < N2 / 2; q += NT) {
        const uint32_t i = ((q >> lstr) << (lstr + 1)) | (q & (stride - 1)), j = i + stride;
        if (j < n) {
          const uint64_t x = S.key[i], y = S.key[j];
          if (y < x) { S.key[i] = y; S.key[j] = x; }
        }
      }
      gsync<NT>();
    }
  }
  // V2 new-vote flags (aux): walk back over equal (strand, diag, fp); clear the head flags (crank)
  for (uint32_t i = t; i < n; i += NT) {
    const uint64_t ki = S.key[i] >> ib;
    const uint64_t ci = S.canon[S.key[i] & imask];
    uint32_t fresh = 1;
    for (uint32_t j = i; j-- > 0 && (S.key[j] >> ib) == ki;)
      if (S.canon[S.key[j] & imask] == ci) { fresh = 0; break; }
    S.aux[i] = fresh;
    S.crank[i] = 0;
  }
  gsync<NT>();
  // step (3): cluster heads.  A gap > D (or a strand change) between sorted neighbours always starts
  // a cluster; inside a gap-free segment the chain Delta0 -> first anchor beyond Delta0 + D is
  // walked by the segment's first thread.
  for (uint32_t i = t; i < n; i += NT) {
    if (i > 0 && !beyond(S.key[i] >> 29, S.key[i - 1] >> 29, D)) continue;
    uint32_t s = i;
    while (true) {
      S.crank[s] = 1;
      const uint64_t dh = S.key[s] >> 29;
      // first e > s beyond Delta0: gallop, then binary search
      uint32_t e = s + 1;
      if (e < n && !beyond(S.key[e] >> 29, dh, D)) {
        uint32_t lo = e, step = 1;  // key[lo] not beyond
        while (lo + step < n && !beyond(S.key[lo + step] >> 29, dh, D)) { lo += step; step <<= 1; }
        uint32_t hi = min(lo + step, n);  // beyond at hi, or hi == n
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (beyond(S.key[mid] >> 29, dh, D)) hi = mid;
          else lo = mid;
        }
        e = hi;
      }
      if (e >= n || beyond(S.key[e] >> 29, S.key[e - 1] >> 29, D)) break;  // segment ends: its own walker
      s = e;
    }
  }
  gsync<NT>();
  // heads -> chead[0..C), new-vote flags -> exclusive prefix (votes of a cluster = a difference)
  group_scan_flags<NT>(n, S.crank, S.chead, S.aux, ws, &S.ctr[0], &S.ctr[3], t);
  gsync<NT>();
  const uint32_t C = S.ctr[0], nfresh = S.ctr[3];
  if (t == 0) S.chead[C] = n;
  gsync<NT>();
  for (uint32_t c = t; c < C; c += NT) {
    const uint32_t e = S.chead[c + 1];
    const uint32_t v = (e < n ? S.aux[e] : nfresh) - S.aux[S.chead[c]];
    S.cv[c] = v;
    if (v >= A.V) S.crank[atomicAdd(&S.ctr[1], 1u)] = c;  // winner list (order irrelevant: ranked below)
  }
  gsync<NT>();
  const uint32_t W = S.ctr[1];
  const bool rescue = W == 0;
  const uint32_t limit = rescue ? 1u : (A.mp ? min(A.mp, W) : W);
  if (!rescue && W > 64) {
    // step (4), many winners (a long read with a small V): sort the winner list by (votes desc, diagonal
    // asc), the same all-ascending bitonic network with a virtual worst element past W, O(W log^2 W)
    // instead of the W^2 comparisons of the counting below; aux[rank] = cluster for rank < limit
    auto worse = [&](uint32_t ca, uint32_t cb) {  // cluster ca ranks after cluster cb
      return better(S.cv[cb], S.key[S.chead[cb]] >> 29, S.cv[ca], S.key[S.chead[ca]] >> 29);
    };
    uint32_t lg = 0;
    while ((1u << lg) < W) ++lg;
    const uint32_t N2 = 1u << lg;
    for (uint32_t ls = 1; ls <= lg; ++ls) {
      const uint32_t lh = ls - 1, half = 1u << lh;
      for (uint32_t q = t; q < N2 / 2; q += NT) {
        const uint32_t base = (q >> lh) << ls, off = q & (half - 1);
        const uint32_t i = base + off, j = base + (2u * half) - 1 - off;
        if (j < W) {
          const uint32_t x = S.crank[i], y = S.crank[j];
          if (worse(x, y)) { S.crank[i] = y; S.crank[j] = x; }
        }
      }
      gsync<NT>();
      for (int lstr = (int)lh - 1; lstr >= 0; --lstr) {
        const uint32_t stride = 1u << lstr;
        for (uint32_t q = t; q < N2 / 2; q += NT) {
          const uint32_t i = ((q >> lstr) << (lstr + 1)) | (q & (stride - 1)), j = i + stride;
          if (j < W) {
            const uint32_t x = S.crank[i], y = S.crank[j];
            if (worse(x, y)) { S.crank[i] = y; S.crank[j] = x; }
          }
        }
        gsync<NT>();
      }
    }
    for (uint32_t w = t; w < limit; w += NT) S.aux[w] = S.crank[w];
  } else if (!rescue) {
    // step (4): rank the winners; aux[rank] = cluster for rank < limit
    for (uint32_t w = t; w < W; w += NT) {
      const uint32_t c = S.crank[w], v = S.cv[c];
      const uint64_t dc = S.key[S.chead[c]] >> 29;
      uint32_t rank = 0;
      for (uint32_t j = 0; j < W && rank < limit; j++) {
        const uint32_t cj = S.crank[j];
        rank += cj != c && better(S.cv[cj], S.key[S.chead[cj]] >> 29, v, dc);
      }
      if (rank < limit) S.aux[rank] = c;
    }
  } else {
    // rescue: the best cluster
    uint32_t bc = 0xffffffffu, bv = 0;
    uint64_t bd = ~0ull;
    for (uint32_t c = t; c < C; c += NT) {
      const uint32_t v = S.cv[c];
      const uint64_t d = S.key[S.chead[c]] >> 29;
      if (bc == 0xffffffffu || better(v, d, bv, bd)) { bc = c; bv = v; bd = d; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint32_t oc = __shfl_xor_sync(FULL, bc, o), ov = __shfl_xor_sync(FULL, bv, o);
      const uint64_t od = __shfl_xor_sync(FULL, bd, o);
      if (oc != 0xffffffffu && (bc == 0xffffffffu || better(ov, od, bv, bd))) { bc = oc; bv = ov; bd = od; }
    }
    if (NW > 1) {
      if (lane == 0) ws[warp] = bc;
      __syncthreads();
      if (t == 0) {
        uint32_t best = ws[0];
        for (int q = 1; q < NW; q++) {
          const uint32_t c = ws[q];
          if (c == 0xffffffffu) continue;
          if (best == 0xffffffffu ||
              better(S.cv[c], S.key[S.chead[c]] >> 29, S.cv[best], S.key[S.chead[best]] >> 29))
            best = c;
        }
        S.aux[0] = best;
      }
    } else if (t == 0) {
      S.aux[0] = bc;
    }
  }
  gsync<NT>();
  // spans of the output clusters: one warp per cluster
  for (uint32_t rank = warp; rank < limit; rank += NW) {
    const uint32_t c = S.aux[rank];
    uint32_t rlo = 0xffffffffu, rhi = 0, qlo = 0xffffffffu, qhi = 0;
    for (uint32_t i = S.chead[c] + lane; i < S.chead[c + 1]; i += 32) {
      const god_anchor an = load_anchor(A, a0 + (S.key[i] & imask));
      rlo = min(rlo, an.ref_pos); rhi = max(rhi, an.ref_pos);
      qlo = min(qlo, an.read_pos); qhi = max(qhi, an.read_pos);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      rlo = min(rlo, __shfl_xor_sync(FULL, rlo, o)); rhi = max(rhi, __shfl_xor_sync(FULL, rhi, o));
      qlo = min(qlo, __shfl_xor_sync(FULL, qlo, o)); qhi = max(qhi, __shfl_xor_sync(FULL, qhi, o));
    }
    if (lane == 0) put_result(A, r, rank, S.key[S.chead[c]] >> 29, S.cv[c], rescue ? 1u : 0u, rlo, rhi, qlo, qhi);
  }
  if (t == 0) A.cnt[r] = limit;
}

// Layout (24 B per anchor): key | canon, whose bytes chead / cv reuse once the new-vote flags are
// set (canon is not read after that) | aux | crank.
__device__ __forceinline__ GroupArrays carve(unsigned char* base, uint32_t cap, uint32_t* ctr) {
  GroupArrays S;
  S.key = reinterpret_cast<uint64_t*>(base);
  S.canon = S.key + cap;
  S.chead = reinterpret_cast<uint32_t*>(S.canon);      // cap + 1 entries
  S.cv = S.chead + cap + 1;                             // cap entries (ends 4 B past canon[cap-1])
  S.aux = reinterpret_cast<uint32_t*>(S.key + 2 * (size_t)cap + 1);
  S.crank = S.aux + cap;
  S.ctr = ctr;
  return S;
}
__host__ __device__ constexpr size_t group_bytes(uint32_t cap) { return (size_t)cap * 24 + 16; }

// 32 < n <= CAP: one warp per read, WPB warps per CTA, a shared-memory slice each
template <uint32_t CAP, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_vote_wsm(VoteArgs A, const uint32_t* __restrict__ list, uint32_t nlist) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t ctr[WPB][4];
  const int warp = threadIdx.x >> 5;
  const uint32_t wid = blockIdx.x * WPB + warp;
  if (wid >= nlist) return;  // warp-uniform
  const GroupArrays S = carve(smem + warp * group_bytes(CAP), CAP, ctr[warp]);
  vote_group<32>(A, list[wid], S, nullptr, threadIdx.x & 31);
}

// VOTE_WSM < n <= VOTE_MID: one CTA per read in shared memory
__global__ void __launch_bounds__(VOTE_NT) k_vote_mid(VoteArgs A, const uint32_t* __restrict__ list) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t ctr[4], ws[2 * (VOTE_NT / 32)];
  vote_group<VOTE_NT>(A, list[blockIdx.x], carve(smem, VOTE_MID, ctr), ws, threadIdx.x);
}

// n > VOTE_MID: one CTA per read on global scratch (32 (n + 2) bytes per read >= group_bytes(n + 1))
__global__ void __launch_bounds__(VOTE_NT) k_vote_big(VoteArgs A, const uint32_t* __restrict__ list,
                                                      const uint64_t* __restrict__ big_off, unsigned char* scratch) {
  __shared__ uint32_t ctr[4], ws[2 * (VOTE_NT / 32)];
  const uint32_t r = list[blockIdx.x];
  const uint32_t n = (uint32_t)(A.aoff[r + 1] - A.aoff[r]);
  const uint64_t o = big_off[blockIdx.x];  // sum of (n + 2) of the big reads placed before
  vote_group<VOTE_NT>(A, r, carve(scratch + o * 32, n + 1, ctr), ws, threadIdx.x);
}

// ------------------------------------------------------------------ compaction into the CSR output
__global__ void k_vote_copy(const god_vote* __restrict__ res, const uint64_t* __restrict__ slot_off,
                            const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ out_off, uint32_t n_reads,
                            god_vote* __restrict__ out) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_reads; r += gridDim.x * blockDim.x) {
    const uint32_t c = cnt[r];
    const god_vote* s = res + slot_off[r];
    god_vote* d = out + out_off[r];
    for (uint32_t j = 0; j < c; j++) d[j] = s[j];
  }
}

}  // namespace

uint64_t vote_reads(const god_index* ix, const uint8_t* reads, const uint64_t* roff, uint32_t n_reads,
                    const uint8_t* phases, const god_anchor* anchors, const uint64_t* aoff, const god_vote_params& vp,
                    god_vote* out, uint64_t* out_off, uint64_t cap, cudaStream_t st) {
  Scratch scr(st);
  uint64_t* slot_off = scr.alloc<uint64_t>((size_t)n_reads + 1);
  uint32_t* lists = scr.alloc<uint32_t>(6ull * n_reads + 1);
  uint32_t* ctr = scr.alloc<uint32_t>(8);        // nlist[6], bad[2]
  uint64_t* big_total = scr.alloc<uint64_t>(1);
  uint64_t* big_off = scr.alloc<uint64_t>((size_t)n_reads + 1);
  uint32_t* cnt = scr.alloc<uint32_t>((size_t)n_reads + 1);
  GOD_CUDA(cudaMemsetAsync(ctr, 0, 8 * sizeof(uint32_t), st));
  GOD_CUDA(cudaMemsetAsync(big_total, 0, sizeof(uint64_t), st));
  GOD_CUDA(cudaMemsetAsync(cnt, 0, ((size_t)n_reads + 1) * sizeof(uint32_t), st));
  GOD_CUDA(cudaMemsetAsync(slot_off, 0, ((size_t)n_reads + 1) * sizeof(uint64_t), st));
  const int nsm = num_sms();
  if (n_reads)
    GOD_LAUNCH("k_vote_classify", k_vote_classify, std::min<unsigned>(grid_for(n_reads, VC_NT), nsm * 2u), VC_NT, 0, st,
               aoff, n_reads, vp.max_pairs, vp.V, slot_off, lists, ctr, big_off, big_total, ctr + 6);
  scan_exclusive_u64(slot_off, slot_off, (uint64_t)n_reads + 1, nullptr, st, scr, "scan_vote_slots");
  uint32_t h[8];
  d2h_small(h, ctr, sizeof(h), st);
  uint64_t hb[2];
  d2h_small(&hb[0], slot_off + n_reads, 8, st);
  d2h_small(&hb[1], big_total, 8, st);
  GOD_CUDA(cudaStreamSynchronize(st));
  GOD_REQUIRE(h[7] == 0, "a read has >= 2^29 anchors");
  god_vote* res = scr.alloc<god_vote>(hb[0] ? hb[0] : 1);
  VoteArgs A;
  A.reads = reads;
  A.roff = roff;
  A.ph = phases;
  A.an = anchors;
  A.an16 = (reinterpret_cast<uintptr_t>(anchors) & 15u) == 0;
  A.aoff = aoff;
  A.pat = ix->P.pat;
  A.k = ix->P.k;
  A.D = vp.D;
  A.V = vp.V;
  A.mp = vp.max_pairs;
  A.slot_off = slot_off;
  A.res = res;
  A.cnt = cnt;
  A.bad = ctr + 6;
  static DeviceOnce attr_once;
  constexpr int WPB1 = 8, WPB2 = 4;
  const size_t sm_wsm = WPB1 * group_bytes(VOTE_WSM), sm_wsm2 = WPB2 * group_bytes(VOTE_WSM2),
               sm_mid = group_bytes(VOTE_MID);
  attr_once.run([&] {
    GOD_CUDA(cudaFuncSetAttribute(k_vote_wsm<VOTE_WSM, WPB1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_wsm));
    GOD_CUDA(cudaFuncSetAttribute(k_vote_wsm<VOTE_WSM2, WPB2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sm_wsm2));
    GOD_CUDA(cudaFuncSetAttribute(k_vote_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_mid));
  });
  if (h[0])
    GOD_LAUNCH("k_vote_warp16", k_vote_warp<16>, grid_for((uint64_t)h[0] * 16, VOTE_NT), VOTE_NT, 0, st, A, lists, h[0]);
  if (h[1])
    GOD_LAUNCH("k_vote_warp", k_vote_warp<32>, grid_for((uint64_t)h[1] * 32, VOTE_NT), VOTE_NT, 0, st, A,
               lists + n_reads, h[1]);
  if (h[2])
    GOD_LAUNCH("k_vote_wsm", (k_vote_wsm<VOTE_WSM, WPB1>), grid_for(h[2], WPB1), WPB1 * 32, sm_wsm, st, A,
               lists + 2ull * n_reads, h[2]);
  if (h[3])
    GOD_LAUNCH("k_vote_wsm2", (k_vote_wsm<VOTE_WSM2, WPB2>), grid_for(h[3], WPB2), WPB2 * 32, sm_wsm2, st, A,
               lists + 3ull * n_reads, h[3]);
  if (h[4]) GOD_LAUNCH("k_vote_mid", k_vote_mid, h[4], VOTE_NT, sm_mid, st, A, lists + 4ull * n_reads);
  if (h[5]) {
    unsigned char* gs = scr.alloc<unsigned char>(hb[1] * 32 + 64);
    GOD_LAUNCH("k_vote_big", k_vote_big, h[5], VOTE_NT, 0, st, A, lists + 5ull * n_reads, big_off, gs);
  }
  scan_exclusive_u32_to_u64(cnt, out_off, (uint64_t)n_reads + 1, nullptr, st, scr, "scan_vote_out");
  uint32_t nbad = 0;
  uint64_t tot = 0;
  d2h_small(&nbad, ctr + 6, 4, st);
  d2h_small(&tot, out_off + n_reads, 8, st);
  GOD_CUDA(cudaStreamSynchronize(st));
  GOD_REQUIRE(nbad == 0, "anchors inconsistent with the reads' phases (read_pos not an included position)");
  if (tot <= cap && tot && n_reads)
    GOD_LAUNCH("k_vote_copy", k_vote_copy, std::min<unsigned>(grid_for(n_reads, 256), nsm * 8u), 256, 0, st, res,
               slot_off, cnt, out_off, n_reads, out);
  return tot;
}

}  // namespace god
