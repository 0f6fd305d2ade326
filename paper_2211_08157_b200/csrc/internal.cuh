// internal.cuh — cross-file declarations of libgod (kernels are in extract.cu, index.cu, seed.cu).
#pragma once
#include "common.cuh"

namespace god {

// One extraction job = one (sequence, phase) pair: the patterned sequence PQ_s of P:300 (s = 0
// and a global position base for the reference).  Its k-mer starts occupy the global
// position range [kb[j], kb[j] + nk] of the extraction index space; the last slot is a separator
// (a window barrier) so that no window ever spans two jobs.
struct Job {
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
  uint64_t* job_off = nullptr;  // optional: [n_jobs + 1] record offset per job
  uint64_t n = 0;               // records written (host)
  uint64_t cap = 0;
  uint32_t* cnt = nullptr;      // optional probe results (seeding)
  uint32_t* beg = nullptr;
};

// Run the fused sparsify + minimizer kernel over device jobs (kb = exclusive scan of nk + 1,
// total_pos = kb[n_jobs]).  Allocates rec arrays from `scr` (capacity grown on demand), fills
// rec.n (synchronizes once to read the count).
void run_extract(const Params& P, const uint8_t* seq, uint64_t seq_bytes, const Job* jobs, const uint64_t* kb,
                 uint32_t n_jobs, uint64_t total_pos, bool want_job, bool want_job_off, Records& rec, cudaStream_t st,
                 Scratch& scr, uint64_t cap_hint, const char* tag = "k_extract");
// Specialised register-resident kernel (extract2.cu) for x == 1 patterns of period 1 or 2 and
// (k, w) in {(21,11), (19,19), (15,10)}; returns false if not applicable.
bool run_extract2(const Params& P, const uint8_t* seq, uint64_t seq_bytes, const Job* jobs, uint32_t n_jobs,
                  bool want_job, bool want_job_off, Records& rec, cudaStream_t st, Scratch& scr,
                  uint64_t cap_hint, const char* tag);

// Build jobs for n sequences: phase from `phases` (nullable -> 0) or, if p_all != 0, one job per
// (sequence, s) for s < p_all (job index = seq * p_all + s).  nk capped at kcap (0 = no cap).
// Returns device jobs, kb (exclusive scan of nk+1) and total positions.
struct JobSet {
  Job* jobs = nullptr;
  uint64_t* kb = nullptr;
  uint32_t n = 0;
  uint64_t total_pos = 0;
  uint64_t seq_bytes = 0;   // offsets[n_seqs]: bytes of the sequence buffer
};
JobSet make_jobs(const Params& P, const uint64_t* offsets, uint32_t n_seqs, const uint8_t* phases, uint32_t p_all,
                 uint32_t kcap, bool global_pos, cudaStream_t st, Scratch& scr);

// ------------------------------------------------------------------------------------ index
// Device view of the seed index (P:286 (3): key = hash, value = sorted start locations).
// dir[s] (s < 2^B, plus dir[2^B] = n_kept): first kept entry whose hash has top-B bits >= s.
// ent_key[e] = (low (2k-B) hash bits) << 1 | strand; ent_pos[e] = global start position.
struct IndexView {
  const uint32_t* dir;
  const uint32_t* ent_key;
  const uint32_t* ent_pos;
  uint32_t dir_bits;
  uint32_t low_bits;     // 2k - B
  uint64_t n_kept;
};

// [begin, end) of the kept entries whose hash == h ("examines the presence of the extracted
// minimizers (their hash values) in the seed index"): directory slot = top B bits, then a binary
// search on the low bits inside the slot (entries are in (hash, pos) order).
__device__ __forceinline__ uint2 probe_range(const IndexView& v, uint64_t h) {
  const uint64_t slot = h >> v.low_bits;
  const uint32_t key = (uint32_t)(h & ((1ull << v.low_bits) - 1));
  const uint32_t lo = __ldg(v.dir + slot), hi = __ldg(v.dir + slot + 1);
  // lower bound by binary search, then a linear scan over the (usually single) matching entries:
  // measured faster than a second binary search (most hashes occur once; slots hold ~2 entries)
  uint32_t a = lo, b = hi;
  while (a < b) {
    const uint32_t mid = (a + b) >> 1;
    if ((__ldg(v.ent_key + mid) >> 1) < key) a = mid + 1;
    else b = mid;
  }
  uint32_t e = a;
  while (e < hi && (__ldg(v.ent_key + e) >> 1) == key) ++e;
  return make_uint2(a, e);
}

}  // namespace god

struct god_index {
  god::Params P;
  god_index_stats st;
  uint32_t* dir = nullptr;
  uint32_t* ent_key = nullptr;
  uint32_t* ent_pos = nullptr;
  cudaStream_t st_alloc = 0;
  god::IndexView view() const {
    return god::IndexView{dir, ent_key, ent_pos, st.dir_bits, (uint32_t)(2 * P.k) - st.dir_bits, st.kept_entries};
  }
};

namespace god {
void build_index(const Params& P, const uint8_t* ref, const uint64_t* ref_offsets, uint32_t n_refs,
                 const god_cutoff& cut, god_index* ix, cudaStream_t st);
void index_count(const god_index* ix, const uint64_t* hashes, uint64_t n, uint32_t* counts, cudaStream_t st);
void index_dump(const god_index* ix, uint64_t* hash, uint32_t* pos, uint8_t* strand, cudaStream_t st);
// returns total anchors; writes anchors only if total <= cap
uint64_t seed_reads(const god_index* ix, const uint8_t* reads, const uint64_t* offsets, uint32_t n_reads,
                    god_phase_mode mode, uint8_t* phases, uint32_t t, god_anchor* anchors, uint64_t* anchor_offsets,
                    uint64_t cap, cudaStream_t st);
void sparsify(const Params& P, const uint8_t* seq, const uint64_t* offsets, uint32_t n, const uint8_t* phases,
              uint64_t* packed, uint64_t* nmask, uint64_t* out_offsets, uint64_t* counts, uint64_t cap_words,
              uint64_t* needed_host, cudaStream_t st);
}  // namespace god
