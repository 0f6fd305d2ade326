// vote.cu — location voting (section 3.4; Fig. 8) with the rescue location
// (P:398), on the anchors of god_seed_reads.  Readings V1-V6: DESIGN.md §2 / include/god.h.
//
// Per read, the anchors become 64-bit sort keys  strand << 63 | (diag + 2^32) << 29 | i
// (i = the anchor's index in the read, so keys are unique and carry their payload; diag fits 34
// bits: forward ref - read in (-2^32, 2^32), reverse ref + read_end in [0, 2^33)).  Sorting the keys
// is step (2) ("a single sorted list of all adjusted matching locations"); equal (strand, diag)
// groups are adjacent, so V2's "(hash, strand, diag) once" is a comparison of canonical k-mers
// (equal canonical k-mer <=> equal hash: H_k is a bijection) inside a group — groups of more than
// one anchor are rare (tandem repeats), and the canonical k-mer is re-read from the read bytes
// only there.  The sweep (step (3)) follows the chain of cluster heads: the next Delta0 is the
// first anchor beyond Delta0 + D.
//
// Reads are bucketed by anchor count: <= 32 anchors -> one warp per read, keys in registers
// (shuffle bitonic sort, ballots for the sweep); <= VOTE_MID anchors -> one CTA per read, keys in
// shared memory; larger -> one CTA per read on global scratch.  Results go to per-read slots
// (min(n, max_pairs) each), then a scan of the per-read counts and a compaction give the CSR output.
#include <algorithm>

#include "internal.cuh"

namespace god {
namespace {

constexpr int VOTE_IDX_BITS = 29;
constexpr uint64_t VOTE_IDX_MASK = (1ull << VOTE_IDX_BITS) - 1;
constexpr uint64_t DIAG_MASK = (1ull << 34) - 1;   // dk = key >> 29: strand at bit 34, biased diag below
constexpr int64_t DIAG_BIAS = 1ll << 32;
constexpr uint32_t VOTE_MID = 2048;   // anchors per read kept in shared memory
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
};

__device__ __forceinline__ bool is_included(const Pattern& P, uint64_t pos, uint32_t a) {
  return pos >= a && ((P.bits >> ((pos - a) % P.p)) & 1ull);
}
// patterned index q of an included original position (inverse of orig_of)
__device__ __forceinline__ uint64_t q_of(const Pattern& P, uint64_t pos, uint32_t a) {
  const uint64_t d = pos - a;
  return (d / P.p) * P.x + P.ones_before[d % P.p];
}

// V1: the sort key of one anchor.  Sets *bad if the anchor cannot come from this read and phase.
__device__ __forceinline__ uint64_t vote_key(const VoteArgs& A, const god_anchor& an, uint32_t a, uint64_t L,
                                             uint32_t i, bool& bad) {
  const uint32_t z = an.strand & 1u;
  if (!is_included(A.pat, an.read_pos, a) || an.read_pos >= L) bad = true;
  int64_t diag;
  if (z == 0) {
    diag = (int64_t)an.ref_pos - (int64_t)an.read_pos;
  } else {
    const uint64_t end = orig_of(A.pat, q_of(A.pat, an.read_pos, a) + (uint64_t)A.k - 1, a);
    if (end >= L) bad = true;
    diag = (int64_t)an.ref_pos + (int64_t)end;
  }
  return ((uint64_t)z << 63) | ((uint64_t)(diag + DIAG_BIAS) << VOTE_IDX_BITS) | i;
}

// canonical k-mer of the read's patterned k-mer starting at original position pos (phase a)
__device__ uint64_t canon_at(const uint8_t* rd, uint64_t L, const Pattern& P, uint32_t a, int k, uint32_t pos) {
  const uint64_t q = q_of(P, pos, a);
  uint64_t fwd = 0, rev = 0;
  for (int i = 0; i < k; i++) {
    const uint64_t o = orig_of(P, q + i, a);
    const uint32_t c = o < L ? (base_code(rd[o]) & 3u) : 0u;
    fwd = (fwd << 2) | c;
    rev |= (uint64_t)(3u - c) << (2 * i);
  }
  return fwd < rev ? fwd : rev;
}

__device__ __forceinline__ int64_t dk_diag(uint64_t dk) { return (int64_t)(dk & DIAG_MASK) - DIAG_BIAS; }

// is anchor (dk) beyond the cluster head (dh): other strand, or diag - Delta0 > D
__device__ __forceinline__ bool beyond(uint64_t dk, uint64_t dh, uint64_t D) {
  return (dk >> 34) != (dh >> 34) || (dk & DIAG_MASK) - (dh & DIAG_MASK) > D;
}

// V4 order of two clusters: more votes first, then strand, then Delta0 (dk orders (strand, diag))
__device__ __forceinline__ bool better(uint32_t va, uint64_t da, uint32_t vb, uint64_t db) {
  return va > vb || (va == vb && da < db);
}

// ------------------------------------------------------------------ bucketing + result slots
__global__ void k_vote_classify(const uint64_t* __restrict__ aoff, uint32_t n_reads, uint32_t mp,
                                uint64_t* __restrict__ slots, uint32_t* __restrict__ lists,
                                uint32_t* __restrict__ nlist, uint64_t* __restrict__ big_off,
                                uint64_t* __restrict__ big_total, uint32_t* __restrict__ bad) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_reads; r += gridDim.x * blockDim.x) {
    const uint64_t n = aoff[r + 1] - aoff[r];
    slots[r] = n == 0 ? 0 : (mp && n > mp ? mp : n);
    if (n == 0) continue;
    if (n > VOTE_IDX_MASK) { atomicAdd(bad + 1, 1u); continue; }
    if (n <= 32) {
      lists[atomicAdd(nlist + 0, 1u)] = r;
    } else if (n <= VOTE_MID) {
      lists[n_reads + atomicAdd(nlist + 1, 1u)] = r;
    } else {
      const uint32_t j = atomicAdd(nlist + 2, 1u);
      lists[2ull * n_reads + j] = r;
      big_off[j] = atomicAdd((unsigned long long*)big_total, (unsigned long long)(n + 1));  // n + 1 heads
    }
  }
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

// ------------------------------------------------------------------ <= 32 anchors: one warp per read
__global__ void __launch_bounds__(VOTE_NT) k_vote_warp(VoteArgs A, const uint32_t* __restrict__ list, uint32_t nlist) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (uint32_t)((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
  if (wid >= nlist) return;  // warp-uniform
  const uint32_t r = list[wid];
  const uint64_t a0 = A.aoff[r];
  const uint32_t n = (uint32_t)(A.aoff[r + 1] - a0);
  const uint64_t rb = A.roff[r], L = A.roff[r + 1] - rb;
  const uint32_t ph = A.ph[r];
  const uint64_t D = A.D ? A.D : L;
  bool bad = false;
  uint64_t key = ~0ull;
  god_anchor an = {0, 0, 0, 0};
  if (lane < (int)n) {
    an = A.an[a0 + lane];
    key = vote_key(A, an, ph, L, (uint32_t)lane, bad);
  }
  if (__any_sync(FULL, bad)) {
    if (lane == 0) atomicAdd(A.bad, 1u);
    return;
  }
  // step (2): bitonic sort of the 32 keys across the warp (pads ~0 sink to the end)
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t o = __shfl_xor_sync(FULL, key, stride);
      const bool up = (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      key = (lower == up) ? (key < o ? key : o) : (key > o ? key : o);
    }
  }
  const bool valid = lane < (int)n;
  const int src = (int)(key & 31u);
  const uint32_t ref = __shfl_sync(FULL, an.ref_pos, src);
  const uint32_t qp = __shfl_sync(FULL, an.read_pos, src);
  const uint64_t dk = key >> VOTE_IDX_BITS;
  // V2: a repeat of (hash, strand, diag) is no new vote
  const uint64_t dprev = __shfl_up_sync(FULL, dk, 1), dnext = __shfl_down_sync(FULL, dk, 1);
  const bool grp = valid && ((lane > 0 && dprev == dk) || (lane + 1 < (int)n && dnext == dk));
  bool dup = false;
  if (__any_sync(FULL, grp)) {
    const uint64_t c = grp ? canon_at(A.reads + rb, L, A.pat, ph, A.k, qp) : 0ull;
    for (int j = 0; j < 31; j++) {
      const uint64_t cj = __shfl_sync(FULL, c, j), dj = __shfl_sync(FULL, dk, j);
      dup |= grp && j < lane && dj == dk && cj == c;
    }
  }
  // step (3): the chain of cluster heads
  uint32_t starts = 0;
  for (uint32_t s = 0; s < n;) {
    starts |= 1u << s;
    const uint64_t dh = __shfl_sync(FULL, dk, (int)s);
    const uint32_t b = __ballot_sync(FULL, valid && lane > (int)s && beyond(dk, dh, D));
    s = b ? (uint32_t)(__ffs(b) - 1) : n;
  }
  const uint32_t le = (lane == 31) ? FULL : ((2u << lane) - 1u);
  const int cid = __popc(starts & le) - 1;
  const uint32_t newmask = __ballot_sync(FULL, valid && !dup);
  // member spans: segmented suffix min/max (clusters are contiguous)
  uint32_t rlo = ref, rhi = ref, qlo = qp, qhi = qp;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t a1 = __shfl_down_sync(FULL, rlo, o), a2 = __shfl_down_sync(FULL, rhi, o);
    const uint32_t a3 = __shfl_down_sync(FULL, qlo, o), a4 = __shfl_down_sync(FULL, qhi, o);
    const int oc = __shfl_down_sync(FULL, cid, o);
    if (lane + o < (int)n && oc == cid) {
      rlo = min(rlo, a1); rhi = max(rhi, a2); qlo = min(qlo, a3); qhi = max(qhi, a4);
    }
  }
  const bool head = valid && ((starts >> lane) & 1u);
  uint32_t votes = 0;
  if (head) {
    const uint32_t after = starts & ~le;
    const uint32_t e = after ? (uint32_t)(__ffs(after) - 1) : n;
    const uint32_t range = (e >= 32 ? FULL : ((1u << e) - 1u)) & ~((1u << lane) - 1u);
    votes = __popc(newmask & range);
  }
  // step (4) / rescue
  const uint32_t winmask = __ballot_sync(FULL, head && votes >= A.V);
  const bool rescue = winmask == 0;
  const bool cand = rescue ? head : ((winmask >> lane) & 1u);
  const uint32_t candmask = rescue ? starts : winmask;
  uint32_t rank = 0;
  for (int j = 0; j < 32; j++) {
    const uint32_t vj = __shfl_sync(FULL, votes, j);
    const uint64_t dj = __shfl_sync(FULL, dk, j);
    rank += ((candmask >> j) & 1u) && j != lane && better(vj, dj, votes, dk);
  }
  const uint32_t limit = rescue ? 1u : (A.mp ? A.mp : 32u);
  if (cand && rank < limit) put_result(A, r, rank, dk, votes, rescue ? 1u : 0u, rlo, rhi, qlo, qhi);
  if (lane == 0) A.cnt[r] = min((uint32_t)__popc(candmask), limit);
}

// ------------------------------------------------------------------ > 32 anchors: one CTA per read
// Arrays (shared memory for <= VOTE_MID anchors, else global scratch): key[n]; flag[n] (1 = new
// vote); per cluster: head index, votes and spans.
struct CtaArrays {
  uint64_t* key;
  uint32_t* flag;
  uint32_t* chead;
  uint32_t* cvotes;
  uint32_t* crank;
};

__device__ void vote_cta(const VoteArgs& A, uint32_t r, const CtaArrays& S) {
  __shared__ uint32_t s_nclust, s_nwin, s_bad;
  const int tid = threadIdx.x;
  const uint64_t a0 = A.aoff[r];
  const uint32_t n = (uint32_t)(A.aoff[r + 1] - a0);
  const uint64_t rb = A.roff[r], L = A.roff[r + 1] - rb;
  const uint32_t ph = A.ph[r];
  const uint64_t D = A.D ? A.D : L;
  if (tid == 0) { s_bad = 0; s_nclust = 0; s_nwin = 0; }
  __syncthreads();
  bool bad = false;
  for (uint32_t i = tid; i < n; i += VOTE_NT) {
    const god_anchor an = A.an[a0 + i];
    S.key[i] = vote_key(A, an, ph, L, i, bad);
  }
  if (bad) s_bad = 1;
  __syncthreads();
  if (s_bad) {
    if (tid == 0) atomicAdd(A.bad, 1u);
    return;
  }
  // step (2): bitonic sort, all comparators ascending (mirror first step), virtual +inf past n
  uint32_t N2 = 1;
  while (N2 < n) N2 <<= 1;
  for (uint32_t size = 2; size <= N2; size <<= 1) {
    const uint32_t half = size >> 1;
    for (uint32_t t = tid; t < N2 / 2; t += VOTE_NT) {
      const uint32_t blk = t / half, off = t % half;
      const uint32_t i = blk * size + off, j = blk * size + size - 1 - off;
      if (j < n) {
        const uint64_t x = S.key[i], y = S.key[j];
        if (y < x) { S.key[i] = y; S.key[j] = x; }
      }
    }
    __syncthreads();
    for (uint32_t stride = half >> 1; stride > 0; stride >>= 1) {
      for (uint32_t t = tid; t < N2 / 2; t += VOTE_NT) {
        const uint32_t i = (t / stride) * 2 * stride + (t % stride), j = i + stride;
        if (j < n) {
          const uint64_t x = S.key[i], y = S.key[j];
          if (y < x) { S.key[i] = y; S.key[j] = x; }
        }
      }
      __syncthreads();
    }
  }
  // V2: new-vote flags
  for (uint32_t i = tid; i < n; i += VOTE_NT) {
    const uint64_t dk = S.key[i] >> VOTE_IDX_BITS;
    uint32_t fresh = 1;
    if (i > 0 && (S.key[i - 1] >> VOTE_IDX_BITS) == dk) {
      const uint32_t qi = A.an[a0 + (S.key[i] & VOTE_IDX_MASK)].read_pos;
      const uint64_t ci = canon_at(A.reads + rb, L, A.pat, ph, A.k, qi);
      for (uint32_t j = i; j-- > 0 && (S.key[j] >> VOTE_IDX_BITS) == dk;) {
        const uint32_t qj = A.an[a0 + (S.key[j] & VOTE_IDX_MASK)].read_pos;
        if (canon_at(A.reads + rb, L, A.pat, ph, A.k, qj) == ci) { fresh = 0; break; }
      }
    }
    S.flag[i] = fresh;
  }
  // step (3): the chain of cluster heads (one thread; binary search for the first anchor beyond D)
  if (tid == 0) {
    uint32_t c = 0;
    for (uint32_t s = 0; s < n;) {
      S.chead[c++] = s;
      const uint64_t dh = S.key[s] >> VOTE_IDX_BITS;
      uint32_t lo = s + 1, hi = n;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (beyond(S.key[mid] >> VOTE_IDX_BITS, dh, D)) hi = mid;
        else lo = mid + 1;
      }
      s = lo;
    }
    S.chead[c] = n;
    s_nclust = c;
  }
  __syncthreads();
  const uint32_t C = s_nclust;
  uint32_t wins = 0;
  for (uint32_t c = tid; c < C; c += VOTE_NT) {
    uint32_t v = 0;
    for (uint32_t i = S.chead[c]; i < S.chead[c + 1]; i++) v += S.flag[i];
    S.cvotes[c] = v;
    wins += v >= A.V;
  }
  atomicAdd(&s_nwin, wins);
  __syncthreads();
  const bool rescue = s_nwin == 0;
  const uint32_t limit = rescue ? 1u : (A.mp ? A.mp : 0xffffffffu);
  for (uint32_t c = tid; c < C; c += VOTE_NT) {
    const uint32_t v = S.cvotes[c];
    if (!rescue && v < A.V) continue;
    const uint64_t dc = S.key[S.chead[c]] >> VOTE_IDX_BITS;
    uint32_t rank = 0;
    for (uint32_t j = 0; j < C && rank < limit; j++) {
      const uint32_t vj = S.cvotes[j];
      if (j == c || (!rescue && vj < A.V)) continue;
      rank += better(vj, S.key[S.chead[j]] >> VOTE_IDX_BITS, v, dc);
    }
    if (rank >= limit) continue;
    uint32_t rlo = 0xffffffffu, rhi = 0, qlo = 0xffffffffu, qhi = 0;
    for (uint32_t i = S.chead[c]; i < S.chead[c + 1]; i++) {
      const god_anchor an = A.an[a0 + (S.key[i] & VOTE_IDX_MASK)];
      rlo = min(rlo, an.ref_pos); rhi = max(rhi, an.ref_pos);
      qlo = min(qlo, an.read_pos); qhi = max(qhi, an.read_pos);
    }
    put_result(A, r, rank, dc, v, rescue ? 1u : 0u, rlo, rhi, qlo, qhi);
  }
  if (tid == 0) A.cnt[r] = rescue ? 1u : min(s_nwin, limit);
}

__global__ void __launch_bounds__(VOTE_NT) k_vote_mid(VoteArgs A, const uint32_t* __restrict__ list) {
  extern __shared__ __align__(16) unsigned char smem[];
  CtaArrays S;
  S.key = reinterpret_cast<uint64_t*>(smem);
  S.flag = reinterpret_cast<uint32_t*>(S.key + VOTE_MID);
  S.chead = S.flag + VOTE_MID;
  S.cvotes = S.chead + VOTE_MID + 1;
  S.crank = nullptr;
  vote_cta(A, list[blockIdx.x], S);
}

__global__ void __launch_bounds__(VOTE_NT) k_vote_big(VoteArgs A, const uint32_t* __restrict__ list,
                                                      const uint64_t* __restrict__ big_off, uint64_t* gkey,
                                                      uint32_t* gflag, uint32_t* ghead, uint32_t* gvotes) {
  const uint64_t o = big_off[blockIdx.x];
  CtaArrays S;
  S.key = gkey + o;
  S.flag = gflag + o;
  S.chead = ghead + o;
  S.cvotes = gvotes + o;
  S.crank = nullptr;
  vote_cta(A, list[blockIdx.x], S);
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
  uint32_t* lists = scr.alloc<uint32_t>(3ull * n_reads + 1);
  uint32_t* ctr = scr.alloc<uint32_t>(8);        // nlist[3], bad[2]
  uint64_t* big_total = scr.alloc<uint64_t>(1);
  uint64_t* big_off = scr.alloc<uint64_t>((size_t)n_reads + 1);
  uint32_t* cnt = scr.alloc<uint32_t>((size_t)n_reads + 1);
  GOD_CUDA(cudaMemsetAsync(ctr, 0, 8 * sizeof(uint32_t), st));
  GOD_CUDA(cudaMemsetAsync(big_total, 0, sizeof(uint64_t), st));
  GOD_CUDA(cudaMemsetAsync(cnt, 0, ((size_t)n_reads + 1) * sizeof(uint32_t), st));
  GOD_CUDA(cudaMemsetAsync(slot_off, 0, ((size_t)n_reads + 1) * sizeof(uint64_t), st));
  const int nsm = num_sms();
  if (n_reads)
    GOD_LAUNCH("k_vote_classify", k_vote_classify, std::min<unsigned>(grid_for(n_reads, 256), nsm * 8u), 256, 0, st,
               aoff, n_reads, vp.max_pairs, slot_off, lists, ctr, big_off, big_total, ctr + 3);
  scan_exclusive_u64(slot_off, slot_off, (uint64_t)n_reads + 1, nullptr, st, scr, "scan_vote_slots");
  uint32_t h[8];
  GOD_CUDA(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, st));
  uint64_t hb[2];
  GOD_CUDA(cudaMemcpyAsync(&hb[0], slot_off + n_reads, 8, cudaMemcpyDeviceToHost, st));
  GOD_CUDA(cudaMemcpyAsync(&hb[1], big_total, 8, cudaMemcpyDeviceToHost, st));
  GOD_CUDA(cudaStreamSynchronize(st));
  GOD_REQUIRE(h[4] == 0, "a read has >= 2^29 anchors");
  god_vote* res = scr.alloc<god_vote>(hb[0] ? hb[0] : 1);
  VoteArgs A;
  A.reads = reads;
  A.roff = roff;
  A.ph = phases;
  A.an = anchors;
  A.aoff = aoff;
  A.pat = ix->P.pat;
  A.k = ix->P.k;
  A.D = vp.D;
  A.V = vp.V;
  A.mp = vp.max_pairs;
  A.slot_off = slot_off;
  A.res = res;
  A.cnt = cnt;
  A.bad = ctr + 3;
  if (h[0]) GOD_LAUNCH("k_vote_warp", k_vote_warp, grid_for((uint64_t)h[0] * 32, VOTE_NT), VOTE_NT, 0, st, A, lists, h[0]);
  if (h[1]) {
    const size_t sm = VOTE_MID * sizeof(uint64_t) + (3 * VOTE_MID + 1) * sizeof(uint32_t);
    static bool attr = false;
    if (!attr) {
      GOD_CUDA(cudaFuncSetAttribute(k_vote_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      attr = true;
    }
    GOD_LAUNCH("k_vote_mid", k_vote_mid, h[1], VOTE_NT, sm, st, A, lists + n_reads);
  }
  if (h[2]) {
    const uint64_t tb = hb[1];
    uint64_t* gkey = scr.alloc<uint64_t>(tb);
    uint32_t* gflag = scr.alloc<uint32_t>(tb);
    uint32_t* ghead = scr.alloc<uint32_t>(tb);
    uint32_t* gvotes = scr.alloc<uint32_t>(tb);
    GOD_LAUNCH("k_vote_big", k_vote_big, h[2], VOTE_NT, 0, st, A, lists + 2ull * n_reads, big_off, gkey, gflag,
               ghead, gvotes);
  }
  scan_exclusive_u32_to_u64(cnt, out_off, (uint64_t)n_reads + 1, nullptr, st, scr, "scan_vote_out");
  uint32_t nbad = 0;
  uint64_t tot = 0;
  GOD_CUDA(cudaMemcpyAsync(&nbad, ctr + 3, 4, cudaMemcpyDeviceToHost, st));
  GOD_CUDA(cudaMemcpyAsync(&tot, out_off + n_reads, 8, cudaMemcpyDeviceToHost, st));
  GOD_CUDA(cudaStreamSynchronize(st));
  GOD_REQUIRE(nbad == 0, "anchors inconsistent with the reads' phases (read_pos not an included position)");
  if (tot <= cap && tot && n_reads)
    GOD_LAUNCH("k_vote_copy", k_vote_copy, std::min<unsigned>(grid_for(n_reads, 256), nsm * 8u), 256, 0, st, res,
               slot_off, cnt, out_off, n_reads, out);
  return tot;
}

}  // namespace god
