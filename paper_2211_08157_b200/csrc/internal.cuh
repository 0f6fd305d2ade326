// internal.cuh — cross-file declarations of libgod (kernels are in extract.cu, index.cu, seed.cu).
#pragma once
#include "common.cuh"

namespace god {

// One extraction job = one (sequence, phase) pair: the patterned sequence PQ_s of P:300 (s = 0
// and a global position base for the reference).  Its k-mer starts occupy the global
// position range [kb[j], kb[j] + nk] of the extraction index space; the last slot is a separator
// (a window barrier) so that no window ever spans two jobs.
struct __align__(16) Job {  // 32 B: two 128-bit accesses
  uint64_t seq_off;   // first byte of the sequence
  uint64_t len;       // bytes
  uint64_t pos_base;  // added to output positions
  uint32_t phase;     // s
  uint32_t nk;        // k-mer starts processed (may be capped below the full count)
};

// Position-ordered minimizer records: hz = hash | strand << 63, pos = pos_base + original start.
struct Records {
  uint64_t* hz = nullptr;
  uint32_t* pos = nullptr;
  uint32_t* job = nullptr;      // optional: job index per record
  uint64_t* job_off = nullptr;  // optional: [n_jobs + 1] first record of each job
  uint64_t* job_end = nullptr;  // with job_off: [n_jobs] one past each job's last record
  uint64_t n = 0;               // records written (host)
  uint64_t cap = 0;
  uint32_t* cnt = nullptr;      // optional probe results (seeding)
  uint32_t* beg = nullptr;
};

// Layout of the jobs for the specialised kernel (extract2.cu), when make_jobs built it: kb = exclusive
// scan of the k-mer counts padded to multiples of w, cw = exclusive scan of the 16-base code words
// (both with the total at [n]); nk_sum = the k-mer starts.
struct X2Layout {
  const uint64_t* kb = nullptr;
  const uint64_t* cw = nullptr;
  uint64_t total_pos = 0, nk_sum = 0;
  uint64_t max_job_blocks = 0;  // padded w-blocks of the longest job
};
// What record order a caller of the extraction needs:
//   ORDER_GLOBAL  position order across all jobs (god_minimizers' CSR output)
//   ORDER_JOB     each job's records contiguous and in position order, jobs anywhere (job_off/job_end)
//   ORDER_NONE    any order (the index build sorts by (hash, pos))
enum RecOrder { ORDER_GLOBAL = 0, ORDER_JOB = 1, ORDER_NONE = 2 };
// true iff run_extract2 has a specialised kernel for these parameters
bool x2_supported(const Params& P);

// The sequence buffer is still arriving from the host, chunk by chunk, on a copy stream (god_build_index
// with a host reference): chunk i = bytes [i * chunk_bytes, (i + 1) * chunk_bytes) is complete when
// arrived[i] has fired.  The unordered specialised K1 then runs each range of tiles as soon as the chunks
// it reads are in (stage 1+2 hidden under the transfer); every other consumer calls wait_all first.
struct SeqStream {
  uint64_t chunk_bytes = 0;
  std::vector<cudaEvent_t> arrived;
  void wait_all(cudaStream_t st) const {
    for (cudaEvent_t e : arrived) GOD_CUDA(cudaStreamWaitEvent(st, e, 0));
  }
};

// Run the fused sparsify + minimizer kernel over device jobs (kb = exclusive scan of nk + 1,
// total_pos = kb[n_jobs]; both unused when x2 carries the specialised layout).  Allocates rec arrays
// from `scr` (capacity grown on demand), fills rec.n (synchronizes once to read the count).
void run_extract(const Params& P, const uint8_t* seq, uint64_t seq_bytes, const Job* jobs, const uint64_t* kb,
                 uint32_t n_jobs, uint64_t total_pos, bool want_job, bool want_job_off, Records& rec, cudaStream_t st,
                 Scratch& scr, uint64_t cap_hint, const char* tag = "k_extract", const X2Layout* x2 = nullptr,
                 RecOrder order = ORDER_GLOBAL, const SeqStream* ss = nullptr);
// Specialised register-resident kernel (extract2.cu) for x == 1 patterns of period 1 to 3 (and the
// '110' / '1110' shapes) and (k, w) in {(21,11), (19,19), (15,10), (19,16)}; returns false if not
// applicable.
// order: see RecOrder (weaker orders let K1 write each tile at an atomically claimed offset instead
// of through a decoupled look-back)
bool run_extract2(const Params& P, const uint8_t* seq, uint64_t seq_bytes, const Job* jobs, uint32_t n_jobs,
                  bool want_job, bool want_job_off, Records& rec, cudaStream_t st, Scratch& scr,
                  uint64_t cap_hint, const char* tag, const X2Layout* x2 = nullptr, RecOrder order = ORDER_GLOBAL,
                  const SeqStream* ss = nullptr);

// Build jobs for n sequences: phase from `phases` (nullable -> 0) or, if p_all != 0, one job per
// (sequence, s) for s < p_all (job index = seq * p_all + s).  nk capped at kcap (0 = no cap).
// Returns device jobs, kb (exclusive scan of nk+1) and total positions.
struct JobSet {
  Job* jobs = nullptr;
  uint64_t* kb = nullptr;   // generic layout (null when x2 is set: the specialised kernel runs)
  uint32_t n = 0;
  uint64_t total_pos = 0;
  uint64_t seq_bytes = 0;   // offsets[n_seqs]: bytes of the sequence buffer
  X2Layout x2;              // specialised layout, built in the same pass when x2_supported(P)
  const X2Layout* x2p() const { return x2.kb ? &x2 : nullptr; }
};
JobSet make_jobs(const Params& P, const uint64_t* offsets, uint32_t n_seqs, const uint8_t* phases, uint32_t p_all,
                 uint32_t kcap, bool global_pos, cudaStream_t st, Scratch& scr);

// ------------------------------------------------------------------------------------ index
// Device view of the seed index (P:286 (3): key = hash, value = sorted start locations).
// ent[e] = pos << 32 | low_hash << 1 | strand, entries in (hash, pos) order.
// dir[s] = slot record (32 B, one sector): kept-entry range [start, end) of slot s and the keys
//          (low hash bits) of its first DIR_KEYS entries, so a probe is one random sector unless
//          the slot holds more than DIR_KEYS entries.
// Slot of a hash:
//   mode 0: the top B = dir_bits hash bits (low_bits = 2k - B);
//   mode 1 (seg != null): data-sized and monotone: segment t = top DIR_SEG_BITS hash bits,
//           slot = seg[t].x + floor(low(h) * seg[t].y / 2^low_bits), low_bits = 2k - DIR_SEG_BITS,
//           seg[t].y ~ (entries in segment t) / 2, so slots hold ~2 entries however skewed the
//           minimizer hashes are (they are window minima: dense at small values).
constexpr int DIR_SEG_BITS = 12;
constexpr int DIR_KEYS = 6;
constexpr int DIR_RUNS = DIR_KEYS / 2;
constexpr int DIR_PAIRS = DIR_KEYS / 2;
struct __align__(32) DirRec {
  uint32_t start, end;
  // end - start <= DIR_PAIRS: the slot's entries themselves, (key | strand << 31, pos) x DIR_PAIRS
  //   (unused pairs (0xFFFFFFFF, 0)): a probe that finds ONE entry with its key has the anchor's
  //   position and strand from this sector and never touches `ent` (round 2: one dependent random
  //   access less per such record; keys are < 2^31, so bit 31 is free).
  // end - start <= DIR_KEYS: the keys of the slot's entries, 0xFFFFFFFF past the end.
  // longer: (key, end of its run) x DIR_RUNS for a slot of <= DIR_RUNS distinct keys (unused pairs
  // (0xFFFFFFFF, end)); key[0] = 0xFFFFFFFF for more (keys are < 2^31, so ~0 is never one)
  uint32_t key[DIR_KEYS];
};
// the six payload words of a slot record holding <= DIR_PAIRS entries; entry(i) = the slot's i-th
// entry in `ent` form (pos << 32 | key << 1 | strand)
template <typename F>
__device__ __forceinline__ void dir_pairs(uint32_t n, F entry, uint32_t (&kk)[DIR_KEYS]) {
#pragma unroll
  for (int e = 0; e < DIR_PAIRS; e++) {
    if ((uint32_t)e < n) {
      const uint64_t en = entry(e);
      kk[2 * e] = ((uint32_t)en >> 1) | ((uint32_t)en << 31);
      kk[2 * e + 1] = (uint32_t)(en >> 32);
    } else {
      kk[2 * e] = 0xFFFFFFFFu;
      kk[2 * e + 1] = 0u;
    }
  }
}
struct IndexView {
  const DirRec* dir;
  const uint64_t* ent;
  const uint2* seg;
  uint32_t dir_bits;
  uint32_t low_bits;
  uint64_t n_kept;
  uint64_t n_slots;
  uint64_t n_ent;   // entries held: all of them (tau != ~0, the bin-built index) or only the kept ones
  uint32_t tau;     // occurrence cutoff applied at probe time: a hash with more entries is absent (O7)
};

// slot of hash h; ~0 if h lies in a segment without slots (mode 1: no reference minimizer there)
__device__ __forceinline__ uint64_t index_slot(const IndexView& v, uint64_t h) {
  if (v.seg) {
    const uint2 t = __ldg(v.seg + (h >> v.low_bits));
    if (!t.y) return ~0ull;
    return t.x + (((h & ((1ull << v.low_bits) - 1)) * t.y) >> v.low_bits);
  }
  return h >> v.low_bits;
}

// [begin, end) of the kept entries whose hash == h ("examines the presence of the extracted
// minimizers (their hash values) in the seed index").  The slot record answers a slot of
// <= DIR_KEYS entries (almost all) or <= DIR_RUNS distinct keys from one 32-B sector; a longer
// slot is searched in the entries.
// *one (if not null): the entry itself (`ent` form) when the slot record holds it and it is the
// only entry with this hash, else ~0
__device__ __forceinline__ uint2 probe_range_all(const IndexView& v, uint64_t h, uint64_t* one = nullptr) {
  if (one) *one = ~0ull;
  const uint64_t slot = index_slot(v, h);
  if (slot == ~0ull) return make_uint2(0, 0);
  GOD_DCHECK(slot < v.n_slots, "probe: directory slot");
  const uint32_t key = (uint32_t)(h & ((1ull << v.low_bits) - 1));
  const uint4 r0 = __ldg(reinterpret_cast<const uint4*>(v.dir + slot));
  const uint4 r1 = __ldg(reinterpret_cast<const uint4*>(v.dir + slot) + 1);
  const uint32_t lo = r0.x, hi = r0.y;
  GOD_DCHECK(lo <= hi && hi <= v.n_ent, "probe: slot entry range inside the entries");
  if (hi - lo <= DIR_PAIRS) {  // the slot's entries are in the record
    const uint32_t k3[DIR_PAIRS] = {r0.z, r1.x, r1.z}, p3[DIR_PAIRS] = {r0.w, r1.y, r1.w};
    uint32_t below = 0, eq = 0, pp = 0, zz = 0;
#pragma unroll
    for (int q = 0; q < DIR_PAIRS; q++) {
      const uint32_t kq = k3[q] & 0x7FFFFFFFu;
      const bool in = (uint32_t)q < hi - lo;
      below += in && kq < key;
      if (in && kq == key) { eq++; pp = p3[q]; zz = k3[q] >> 31; }
    }
    if (one && eq == 1) *one = ((uint64_t)pp << 32) | ((uint64_t)key << 1) | zz;
    return make_uint2(lo + below, lo + below + eq);
  }
  if (hi - lo <= DIR_KEYS) {  // every key of the slot is in the record
    const uint32_t k6[DIR_KEYS] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    uint32_t below = 0, eq = 0;
#pragma unroll
    for (int q = 0; q < DIR_KEYS; q++) {
      below += k6[q] < key;
      eq += k6[q] == key;
    }
    return make_uint2(lo + below, lo + below + eq);
  }
  if (r0.z != 0xFFFFFFFFu) {  // <= DIR_RUNS distinct keys: (key, run end) pairs
    if (key == r0.z) return make_uint2(lo, r0.w);
    if (key == r1.x) return make_uint2(r0.w, r1.y);
    if (key == r1.z) return make_uint2(r1.y, r1.w);
    const uint32_t at = key < r0.z ? lo : key < r1.x ? r0.w : key < r1.z ? r1.y : r1.w;
    return make_uint2(at, at);
  }
  // more keys: both ends equal the key -> the whole slot, else search the entries
  const uint32_t kf = (uint32_t)__ldg(v.ent + lo) >> 1, kl = (uint32_t)__ldg(v.ent + hi - 1) >> 1;
  if (kf == key && kl == key) return make_uint2(lo, hi);
  if (kf > key || kl < key) return make_uint2(lo, lo);
  uint32_t a = lo, b = hi;  // lower bound
  while (a < b) {
    const uint32_t mid = (a + b) >> 1;
    if (((uint32_t)__ldg(v.ent + mid) >> 1) < key) a = mid + 1;
    else b = mid;
  }
  uint32_t c = a, d = hi;  // upper bound
  while (c < d) {
    const uint32_t mid = (c + d) >> 1;
    if (((uint32_t)__ldg(v.ent + mid) >> 1) <= key) c = mid + 1;
    else d = mid;
  }
  return make_uint2(a, c);
}
// the kept entries with hash h: a hash with more than tau entries is dropped (reading O7)
__device__ __forceinline__ uint2 probe_range(const IndexView& v, uint64_t h, uint64_t* one = nullptr) {
  const uint2 r = probe_range_all(v, h, one);
  return r.y - r.x > v.tau ? make_uint2(r.x, r.x) : r;
}

}  // namespace god

struct god_index {
  god::Params P;
  god_index_stats st;
  god::DirRec* dir = nullptr;
  uint64_t* ent = nullptr;
  uint2* seg = nullptr;       // mode 1 slot map (null in mode 0)
  uint32_t low_bits = 0;
  uint64_t n_slots = 0;
  uint64_t n_ent = 0;              // entries in ent (all of them when tau_probe != ~0)
  uint32_t tau_probe = 0xFFFFFFFFu;  // cutoff applied at probe time (~0: ent holds the kept entries only)
  cudaStream_t st_alloc = 0;
  god::IndexView view() const {
    return god::IndexView{dir, ent, seg, st.dir_bits, low_bits, st.kept_entries, n_slots, n_ent, tau_probe};
  }
};

namespace god {
// ss: the reference is still arriving from the host (SeqStream), else null
void build_index(const Params& P, const uint8_t* ref, const uint64_t* ref_offsets, uint32_t n_refs,
                 const god_cutoff& cut, god_index* ix, cudaStream_t st, const SeqStream* ss = nullptr);
void index_count(const god_index* ix, const uint64_t* hashes, uint64_t n, uint32_t* counts, cudaStream_t st);
void index_dump(const god_index* ix, uint64_t* hash, uint32_t* pos, uint8_t* strand, cudaStream_t st);
// returns total anchors; writes anchors only if total <= cap; anchor read ids are rid_base + the
// read's index in this call (batched callers pass the batch's first read)
uint64_t seed_reads(const god_index* ix, const uint8_t* reads, const uint64_t* offsets, uint32_t n_reads,
                    god_phase_mode mode, uint8_t* phases, uint32_t t, god_anchor* anchors, uint64_t* anchor_offsets,
                    uint64_t cap, cudaStream_t st, uint32_t rid_base = 0);
// location voting on the anchors of seed_reads (vote.cu); returns the number of voted locations and
// writes them (CSR by read) only if that is <= cap
uint64_t vote_reads(const god_index* ix, const uint8_t* reads, const uint64_t* roff, uint32_t n_reads,
                    const uint8_t* phases, const god_anchor* anchors, const uint64_t* aoff, const god_vote_params& vp,
                    god_vote* out, uint64_t* out_off, uint64_t cap, cudaStream_t st);
// containment search over reference batches (contain.cu); ref_off on the device and the host
void contain(const Params& P, const uint8_t* refs, const uint64_t* ref_off, const uint64_t* ref_off_host,
             uint32_t n_refs, const god_cutoff& cut, const uint8_t* reads, const uint64_t* roff, uint32_t n_reads,
             uint32_t t, const god_vote_params& vp, uint64_t batch_bases, uint32_t min_reads, uint32_t cov_num,
             uint32_t cov_den, uint64_t* mreads, uint64_t* mbases, uint8_t* accepted, cudaStream_t st);
// seed-comparison harness (harness.cu); pairs of <= harness_max_len() bases
void seed_harness(const Params& P, const uint8_t* a, const uint8_t* b, const uint64_t* off, uint32_t n,
                  uint64_t* ed, uint64_t* matches, uint64_t* totals, uint32_t* god_phase, cudaStream_t st);
uint32_t harness_max_len();
void harness_accepted(const uint64_t* ed, const uint64_t* mm, const uint64_t* tt, uint32_t n, const uint64_t* E,
                      uint32_t nE, uint64_t* acc, cudaStream_t st);
void sparsify(const Params& P, const uint8_t* seq, const uint64_t* offsets, uint32_t n, const uint8_t* phases,
              uint64_t* packed, uint64_t* nmask, uint64_t* out_offsets, uint64_t* counts, uint64_t cap_words,
              uint64_t* needed_host, cudaStream_t st);
}  // namespace god
