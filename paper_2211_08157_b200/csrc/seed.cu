// seed.cu — stage 4: pattern alignment (phase selection) and compressed seeding.
//
// Pipeline (kernels S1-S4), all reads in one batch:
//   S1  extraction (extract.cu) over the (read, s) jobs for s < p, each capped to the first
//       KCAP k-mer starts ("limit the number of calculated minimizers in each PQ_s"):
//       records at k-mer index <= KCAP - w are exactly the first minimizers of the full PQ_s
//   S2  one thread per read: c = min(t, min_s |M_s|), score_s = sum over the first c records of
//       occ(hash) (index probes), a = argmax (smallest s on ties).  Reads whose capped prefix gave
//       fewer than t exact records for some phase (N-dense prefixes) are recomputed uncapped.
//   S3  the minimizers of PQ_a: reused from S1 when the read's phase-a job was complete
//       (every short read), else extracted again over (read, a_r) jobs and probed
//   S4  anchors from the probe results: fast path (all reads from S1) = 8-lane groups per read
//       (counts, scan over reads, write); general path = gather into read order, scan, write
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include "internal.cuh"

namespace god {

struct SeedSources {
  const uint64_t* hz[3];
  const uint32_t* pos[3];
  const uint64_t* off[3];   // first record of each job ...
  const uint64_t* end[3];   // ... and one past its last (job-aligned extraction places jobs tile by tile)
  const uint32_t* cnt[3];   // probe result per record: number of kept entries with its hash
  const uint32_t* beg[3];   // ... and the first of them
};

namespace {

// flags in a probe's count word (k_anchor_count<true>)
constexpr uint32_t CNT_INL = 0x80000000u, CNT_STRAND = 0x40000000u, CNT_MASK = 0x3FFFFFFFu;

__global__ void k_phase(const uint32_t* __restrict__ occ, const Job* __restrict__ jobs, const uint64_t* __restrict__ job_off,
                        const uint64_t* __restrict__ job_end,
                        const uint64_t* __restrict__ hz, const uint32_t* __restrict__ pos, const uint32_t* __restrict__ ids,
                        uint32_t n_reads, uint32_t p, uint32_t t, uint32_t w, uint32_t kcap, Pattern pat, int k,
                        uint8_t* phases, uint32_t* redo, uint32_t* n_redo, uint64_t* acount) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_reads; i += gridDim.x * blockDim.x) {
    const uint32_t r = ids ? ids[i] : i;
    uint64_t nmin = ~0ull;
    bool fallback = false;
    for (uint32_t s = 0; s < p; s++) {
      const uint64_t j = (uint64_t)i * p + s;
      const Job jb = jobs[j];
      uint64_t c = job_end[j] - job_off[j];
      if (kcap) {
        const uint64_t ninc = included_count(pat, jb.len, s);
        const uint64_t nk_full = ninc >= (uint64_t)k ? ninc - k + 1 : 0;
        if (nk_full > jb.nk) {  // truncated: only records with k-mer index <= nk - w are exact
          uint64_t safe = 0;
          if (jb.nk >= w) {
            const uint64_t lim = orig_of(pat, jb.nk - w, s);
            for (uint64_t q = job_off[j]; q < job_end[j] && pos[q] <= lim; q++) ++safe;
          }
          if (safe < t) fallback = true;
          c = safe;
        }
      }
      nmin = c < nmin ? c : nmin;
    }
    if (fallback) {
      redo[atomicAdd(n_redo, 1u)] = r;
      continue;
    }
    const uint64_t c = nmin < t ? nmin : t;
    uint64_t best = 0;
    uint32_t a = 0;
    for (uint32_t s = 0; s < p; s++) {
      const uint64_t j = (uint64_t)i * p + s;
      uint64_t sc = 0;
      for (uint64_t q = 0; q < c; q++) sc += occ[job_off[j] + q] & CNT_MASK;  // occ(h) of the q-th minimizer
      if (s == 0 || sc > best) { best = sc; a = s; }
    }
    phases[r] = (uint8_t)a;
    if (acount) {  // anchors of the read if PQ_a's records are this phase job's (the S4 fast path)
      const uint64_t j = (uint64_t)i * p + a;
      uint64_t na = 0;
      for (uint64_t q = job_off[j]; q < job_end[j]; q++) na += occ[q] & CNT_MASK;
      acount[r] = na;
    }
  }
}

// jobs for an explicit read list: (ids[i], s) for s < p
__global__ void k_make_jobs_ids(Params P, const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ ids,
                                uint32_t n, uint32_t p, Job* jobs, uint64_t* nkp1) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < (uint64_t)n * p; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = ids[j / p];
    const uint32_t s = (uint32_t)(j % p);
    Job jb;
    jb.seq_off = offsets[r];
    jb.len = offsets[r + 1] - offsets[r];
    jb.pos_base = 0;
    jb.phase = s;
    const uint64_t ninc = included_count(P.pat, jb.len, s);
    jb.nk = (uint32_t)(ninc >= (uint64_t)P.k ? ninc - P.k + 1 : 0);
    jobs[j] = jb;
    nkp1[j] = (uint64_t)jb.nk + 1;
  }
}

// developer check (GOD_DEBUG_JOBS): every job's record range lies inside the records
__global__ void k_check_jobs(const uint64_t* job_off, const uint64_t* job_end, uint64_t nj, uint64_t n,
                             unsigned long long* bad) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nj; j += (uint64_t)gridDim.x * blockDim.x)
    if (job_off[j] > job_end[j] || job_end[j] > n) atomicMin(bad, (unsigned long long)j);
}

// one probe per thread, one thread per record, large grid: the probe is a chain of two dependent
// random accesses (directory slot, entries) and is bound by HBM random-access bandwidth; many
// resident warps hide the latency better than a persistent loop with per-thread ILP (measured).
// INL (the index holds < 2^30 entries, so counts leave the top bits of cnt free): a record whose hash
// has ONE kept entry that its slot record holds gets cnt = 1 | CNT_INL | strand << 30 and beg = the
// entry's position — its anchor needs no access to `ent` (CNT_MASK strips the flags).
template <bool INL>
__global__ void k_anchor_count(IndexView v, const uint64_t* __restrict__ hz, uint64_t n, uint32_t* cnt, uint32_t* beg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t one = ~0ull;
    const uint2 rg = probe_range(v, hz[i] & ((1ull << 63) - 1), INL ? &one : nullptr);
    if (INL && rg.y - rg.x == 1 && one != ~0ull) {
      cnt[i] = 1u | CNT_INL | (((uint32_t)one & 1u) ? CNT_STRAND : 0u);
      beg[i] = (uint32_t)(one >> 32);
    } else {
      cnt[i] = rg.y - rg.x;
      beg[i] = rg.x;
    }
  }
}

// S4 fast path (every read's PQ_a records are its phase-a job of S1, each <= ~40 records): a group
// of 8 lanes per read sums its records' probe counts, and after the scan writes its anchors (each
// lane one record at a time, offsets by a group scan), so no read-ordered copy of the records is made.
#ifndef GOD_AW_MINB
#define GOD_AW_MINB 8  // measured (human): 5 -> 2.84 ms, 6 -> 2.46, 8 -> 2.33 (32 registers, 72 B spilled); 16-lane groups 3.41
#endif
#ifndef GOD_RG
#define GOD_RG 8
#endif
constexpr int RG = GOD_RG;
__global__ void k_read_anchor_counts1(const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ job_off,
                                      const uint64_t* __restrict__ job_end,
                                      const uint8_t* __restrict__ phases, uint32_t p, uint32_t n_reads, uint64_t* out) {
  const uint32_t l = threadIdx.x & (RG - 1);
  for (uint64_t g = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / RG; g < n_reads;
       g += (uint64_t)gridDim.x * blockDim.x / RG) {
    const uint32_t r = (uint32_t)g;
    const uint64_t j = (uint64_t)r * p + (phases ? phases[r] : 0u);
    const uint64_t b = job_off[j], e = job_end[j];
    uint64_t acc = 0;
    for (uint64_t q = b + l; q < e; q += RG) acc += cnt[q] & CNT_MASK;
#pragma unroll
    for (int d = RG / 2; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d, RG);
    if (l == 0) out[r] = acc;
  }
}
// The group's 8 lanes share the chunk's anchors evenly (anchor a of the chunk -> lane a mod 8, its
// record found from the lanes' inclusive counts by shuffles), two anchors per lane per round with both
// entry loads issued before either store: the writer is bound by the latency of the dependent entry
// reads, not by their number (measured: without them 1.74 ms, with them 3.45 ms whether 87 M or 40 M
// of them go to DRAM), so what counts is how many are in flight — and a frequent hash's run of entries
// is read by 8 lanes side by side instead of one lane in sequence.
template <bool A16>  // A16: out is 16-B aligned -> one 128-bit store per anchor
__global__ void __launch_bounds__(256, GOD_AW_MINB) k_anchor_write1(IndexView v, const uint64_t* __restrict__ hz, const uint32_t* __restrict__ pos,
                                const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ beg,
                                const uint64_t* __restrict__ job_off, const uint64_t* __restrict__ job_end,
                                const uint8_t* __restrict__ phases, uint32_t p,
                                uint32_t n_reads, const uint64_t* __restrict__ aoff, god_anchor* out,
                                uint32_t rid_base) {
  const uint32_t l = threadIdx.x & (RG - 1);
  static_assert(RG == 8 || RG == 16, "group mask");
  const uint32_t gm = RG == 8 ? 0xFFu << (threadIdx.x & 24u) : 0xFFFFu << (threadIdx.x & 16u);  // the lanes of this group
  for (uint64_t g = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / RG; g < n_reads;
       g += (uint64_t)gridDim.x * blockDim.x / RG) {
    const uint32_t r = (uint32_t)g;
    // the read's phase and the record ranges of all its phase jobs are loaded together (lane s holds
    // job s), then the chosen one is taken by shuffle: one dependent round trip less per read
    const uint32_t a_ph = phases ? phases[r] : 0u;
    uint64_t b, e;
    if (p <= (uint32_t)RG) {
      const uint64_t jl = (uint64_t)r * p + (l < p ? l : 0u);
      const uint64_t bl = job_off[jl], el = job_end[jl];
      b = __shfl_sync(gm, bl, a_ph, RG);
      e = __shfl_sync(gm, el, a_ph, RG);
    } else {
      const uint64_t j = (uint64_t)r * p + a_ph;
      b = job_off[j];
      e = job_end[j];
    }
    GOD_DCHECK(b <= e, "anchor writer: job record range");
    uint64_t o = aoff[r];
    for (uint64_t q0 = b; q0 < e; q0 += RG) {  // uniform trip count within the group
      const uint64_t q = q0 + l;
      // all four record fields at once (not the count first): a shorter dependent chain per read
      const uint32_t craw = q < e ? cnt[q] : 0u;
      const uint32_t bg0 = q < e ? beg[q] : 0u, qp0 = q < e ? pos[q] : 0u;
      const uint32_t qz0 = q < e ? (uint32_t)(hz[q] >> 63) : 0u;
      const uint32_t c = craw & CNT_MASK;
      uint32_t incl = c;
#pragma unroll
      for (int d = 1; d < RG; d <<= 1) {
        const uint32_t y = __shfl_up_sync(gm, incl, d, RG);
        if (l >= (uint32_t)d) incl += y;
      }
      const uint32_t tot = __shfl_sync(gm, incl, RG - 1, RG);
      uint32_t bg = 0, qp = 0, fl = 0;  // fl: bit 0 read strand, bit 1 entry strand (inline), bit 2 inline
      if (c) {
        bg = bg0;
        qp = qp0;
        fl = qz0 | ((craw >> 30) << 1);
        GOD_DCHECK(((craw & CNT_INL) || (uint64_t)bg + c <= v.n_ent) && o + incl <= aoff[n_reads],
                   "anchor writer: entry and anchor ranges");
      }
      const uint32_t excl = incl - c;
      uint32_t inc8[RG];
#pragma unroll
      for (int jl = 0; jl < RG; jl++) inc8[jl] = __shfl_sync(gm, incl, jl, RG);
      for (uint32_t a0 = 0; a0 < tot; a0 += 2 * RG) {  // uniform within the group
        uint64_t en[2];
        uint32_t rp[2], rf[2];
#pragma unroll
        for (int u = 0; u < 2; u++) {
          const uint32_t a = a0 + u * RG + l;
          uint32_t rec = 0;
#pragma unroll
          for (int jl = 0; jl < RG - 1; jl++) rec += inc8[jl] <= a;  // the record holding anchor a
          const uint32_t rb = __shfl_sync(gm, bg, rec, RG), rx = __shfl_sync(gm, excl, rec, RG);
          rp[u] = __shfl_sync(gm, qp, rec, RG);
          rf[u] = __shfl_sync(gm, fl, rec, RG);
          en[u] = 0;
          if (a < tot) {
            // the entry came with the probe (its slot record holds it), else read it
            if (rf[u] & 4u) en[u] = ((uint64_t)rb << 32) | ((rf[u] >> 1) & 1u);
            else
#ifdef GOD_DBG_NO_ENT
              en[u] = (uint64_t)rb + (a - rx);
#else
              en[u] = __ldg(v.ent + rb + (a - rx));
#endif
          }
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
          const uint32_t a = a0 + u * RG + l;
          if (a < tot) {
            const uint64_t oo = o + a;
            if (A16) {
              reinterpret_cast<uint4*>(out)[oo] =
                  make_uint4((uint32_t)(en[u] >> 32), rp[u], rid_base + r, ((uint32_t)en[u] & 1u) ^ (rf[u] & 1u));
            } else {
              god_anchor an;
              an.ref_pos = (uint32_t)(en[u] >> 32);
              an.read_pos = rp[u];
              an.read_id = rid_base + r;
              an.strand = ((uint32_t)en[u] & 1u) ^ (rf[u] & 1u);
              out[oo] = an;
            }
          }
        }
      }
      o += tot;
    }
  }
}

// one thread per read minimizer: its anchors are the kept entries [beg, beg + cnt)
__global__ void k_anchor_write(IndexView v, const uint32_t* __restrict__ pos, const uint32_t* __restrict__ rid,
                               const uint64_t* __restrict__ hz, uint64_t n, const uint64_t* __restrict__ aoff,
                               const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ beg,
                               const uint8_t* __restrict__ inl, god_anchor* out, uint32_t rid_base) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = cnt[i];
    if (!c) continue;
    const uint32_t qz = (uint32_t)(hz[i] >> 63), qpos = pos[i], r = rid_base + rid[i], b = beg[i];
    const uint32_t fl = inl[i];  // bit 1: the entry came with the probe (b = its position, bit 0 = its strand)
    uint64_t o = aoff[i];
    if (fl & 2u) {
      god_anchor an;
      an.ref_pos = b;
      an.read_pos = qpos;
      an.read_id = r;
      an.strand = (fl & 1u) ^ qz;
      out[o] = an;
      continue;
    }
    for (uint32_t e = b; e < b + c; e++, o++) {
      god_anchor an;
      const uint64_t en = __ldg(v.ent + e);
      an.ref_pos = (uint32_t)(en >> 32);
      an.read_pos = qpos;
      an.read_id = r;
      an.strand = ((uint32_t)en & 1u) ^ qz;
      out[o] = an;
    }
  }
}

// source of each read's PQ_a minimizers (see seed_reads); reads with src == 2 are already set
__global__ void k_seed_plan(Pattern pat, int k, uint32_t n_reads, uint32_t p, const uint8_t* __restrict__ phases,
                            const Job* __restrict__ jobs1, const uint64_t* __restrict__ offsets, uint8_t* src,
                            uint32_t* srcj, uint32_t* list3, uint32_t* n3) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_reads; r += gridDim.x * blockDim.x) {
    if (src[r] == 2) continue;
    if (jobs1) {
      const uint32_t a = phases[r];
      const uint64_t j = (uint64_t)r * p + a;
      const uint64_t len = offsets[r + 1] - offsets[r];
      const uint64_t ninc = included_count(pat, len, a);
      const uint64_t nk_full = ninc >= (uint64_t)k ? ninc - k + 1 : 0;
      if (jobs1[j].nk == nk_full) {
        src[r] = 1;
        srcj[r] = (uint32_t)j;
        continue;
      }
    }
    list3[atomicAdd(n3, 1u)] = r;
  }
}

__global__ void k_redo_src(uint32_t nr, uint32_t p, const uint32_t* __restrict__ redo, const uint8_t* __restrict__ phases,
                           uint8_t* src, uint32_t* srcj) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += gridDim.x * blockDim.x) {
    const uint32_t r = redo[i];
    src[r] = 2;
    srcj[r] = i * p + phases[r];
  }
}

__global__ void k_iota_src3(uint32_t n, uint8_t* src, uint32_t* srcj) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    src[r] = 3;
    srcj[r] = r;
  }
}

// jobs (list3[i], phase a) for the reads that need a dedicated extraction
__global__ void k_make_jobs_sel(Params P, const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ list3,
                                uint32_t n3, const uint8_t* __restrict__ phases, Job* jobs, uint64_t* nkp1, uint8_t* src,
                                uint32_t* srcj) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n3; i += gridDim.x * blockDim.x) {
    const uint32_t r = list3[i];
    Job jb;
    jb.seq_off = offsets[r];
    jb.len = offsets[r + 1] - offsets[r];
    jb.pos_base = 0;
    jb.phase = phases[r];
    const uint64_t ninc = included_count(P.pat, jb.len, jb.phase);
    jb.nk = (uint32_t)(ninc >= (uint64_t)P.k ? ninc - P.k + 1 : 0);
    jobs[i] = jb;
    nkp1[i] = (uint64_t)jb.nk + 1;
    src[r] = 3;
    srcj[r] = i;
  }
}

__global__ void k_seed_counts(SeedSources S, uint32_t n_reads, const uint8_t* __restrict__ src,
                              const uint32_t* __restrict__ srcj, uint64_t* cntr) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_reads; r += gridDim.x * blockDim.x) {
    const int s = src[r] - 1;
    const uint32_t j = srcj[r];
    cntr[r] = s >= 0 ? S.end[s][j] - S.off[s][j] : 0;
  }
}

// 8 threads per read copy its records into the read-ordered arrays
__global__ void k_seed_gather(SeedSources S, uint32_t n_reads, const uint8_t* __restrict__ src,
                              const uint32_t* __restrict__ srcj, const uint64_t* __restrict__ roff, uint64_t* hz,
                              uint32_t* qpos, uint32_t* rid, uint32_t* cnt, uint32_t* beg, uint8_t* inl) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < (uint64_t)n_reads * 8;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(g >> 3), l = (uint32_t)(g & 7);
    const int s = src[r] - 1;
    if (s < 0) continue;
    const uint64_t b = S.off[s][srcj[r]], o = roff[r], c = roff[r + 1] - o;
    for (uint64_t q = l; q < c; q += 8) {
      hz[o + q] = S.hz[s][b + q];
      qpos[o + q] = S.pos[s][b + q];
      rid[o + q] = r;
      const uint32_t craw = S.cnt[s][b + q];
      cnt[o + q] = craw & CNT_MASK;   // clean counts for the scan; the inline flags go beside them
      inl[o + q] = (uint8_t)(craw >> 30);
      beg[o + q] = S.beg[s][b + q];
    }
  }
}

__global__ void k_read_anchor_offsets(const uint64_t* __restrict__ job_off, const uint64_t* __restrict__ aoff,
                                      uint64_t n_rec, const uint64_t* total, uint32_t n_reads, uint64_t* out) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r <= n_reads; r += gridDim.x * blockDim.x) {
    const uint64_t q = job_off[r];
    out[r] = q < n_rec ? aoff[q] : *total;
  }
}
}  // namespace

// probe every record once: (count, first) of the kept entries with its hash
static void probe_all(const IndexView& v, Records& rec, cudaStream_t st, Scratch& scr) {
  rec.cnt = scr.alloc<uint32_t>(rec.n);
  rec.beg = scr.alloc<uint32_t>(rec.n);
  if (rec.n) {
    prof_add_units("k_probe", rec.n);  // probes (records looked up) for the stage-4 roofline
    // the count word's top bits carry the inline-entry flags only when no count can reach them
    if (v.n_ent < (1ull << 30))
      GOD_LAUNCH("k_probe", k_anchor_count<true>, grid_for(rec.n, 256), 256, 0, st, v, rec.hz, rec.n, rec.cnt, rec.beg);
    else
      GOD_LAUNCH("k_probe", k_anchor_count<false>, grid_for(rec.n, 256), 256, 0, st, v, rec.hz, rec.n, rec.cnt, rec.beg);
  }
}

uint64_t seed_reads(const god_index* ix, const uint8_t* reads, const uint64_t* offsets, uint32_t n_reads,
                    god_phase_mode mode, uint8_t* phases, uint32_t t, god_anchor* anchors, uint64_t* anchor_offsets,
                    uint64_t cap, cudaStream_t st, uint32_t rid_base) {
  NvtxRange nvtx("stage 4: phase selection + seeding");
  Scratch scr(st);
  const Params& P = ix->P;
  const uint32_t p = P.pat.p;
  const IndexView v = ix->view();
  if (n_reads == 0) {
    GOD_CUDA(cudaMemsetAsync(anchor_offsets, 0, sizeof(uint64_t), st));
    return 0;
  }
  // Where each read's PQ_a minimizers come from: 1 = the capped phase extraction (its phase-a job
  // was not truncated, so it holds all of PQ_a's minimizers), 2 = the uncapped phase re-extraction
  // (fallback reads), 3 = a dedicated extraction of PQ_a (long reads, GIVEN mode, p = 1).
  uint8_t* src = scr.alloc<uint8_t>(n_reads);
  uint32_t* srcj = scr.alloc<uint32_t>(n_reads);
  GOD_CUDA(cudaMemsetAsync(src, 0, n_reads, st));
  // ---------------- S1/S2: pattern alignment
  bool have_phase_records = false;
  bool counted = false;  // k_phase wrote each read's phase-a anchor count into anchor_offsets
  uint32_t nr = 0;
  Records rec1, rec2, rec3;
  JobSet js1;
  if (mode == GOD_PHASE_SELECT) {
    if (p == 1) {
      GOD_CUDA(cudaMemsetAsync(phases, 0, n_reads, st));
    } else {
      const uint32_t kcap = (t + 1) * (uint32_t)P.w + (uint32_t)P.w;
      js1 = make_jobs(P, offsets, n_reads, nullptr, p, kcap, false, st, scr);
      run_extract(P, reads, js1.seq_bytes, js1.jobs, js1.kb, js1.n, js1.total_pos, false, true, rec1, st, scr,
                  js1.total_pos / (uint64_t)(P.w + 1) * 2 + js1.total_pos / 8 + 4096, "extract_phase", js1.x2p(), ORDER_JOB);
      if (getenv("GOD_DEBUG_JOBS")) {
        unsigned long long* bad = scr.alloc<unsigned long long>(1);
        GOD_CUDA(cudaMemsetAsync(bad, 0xFF, 8, st));
        GOD_LAUNCH("k_check_jobs", k_check_jobs, grid_for(js1.n, 256), 256, 0, st, rec1.job_off, rec1.job_end, js1.n,
                   rec1.n, bad);
        unsigned long long hb = 0;
        uint64_t h2[2] = {0, 0};
        GOD_CUDA(cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost));
        if (hb != ~0ull) {
          GOD_CUDA(cudaMemcpy(&h2[0], rec1.job_off + hb, 8, cudaMemcpyDeviceToHost));
          GOD_CUDA(cudaMemcpy(&h2[1], rec1.job_end + hb, 8, cudaMemcpyDeviceToHost));
        }
        fprintf(stderr, "[jobs] n_jobs=%u n=%llu max_jb=%llu first_bad=%lld off=%llu end=%llu\n", js1.n,
                (unsigned long long)rec1.n, (unsigned long long)js1.x2.max_job_blocks,
                hb == ~0ull ? -1ll : (long long)hb, (unsigned long long)h2[0], (unsigned long long)h2[1]);
      }
      uint32_t* redo = scr.alloc<uint32_t>(n_reads);
      uint32_t* n_redo = scr.alloc<uint32_t>(1);
      GOD_CUDA(cudaMemsetAsync(n_redo, 0, sizeof(uint32_t), st));
      probe_all(v, rec1, st, scr);
      GOD_LAUNCH("k_phase", k_phase, grid_for(n_reads, 128), 128, 0, st, rec1.cnt, js1.jobs, rec1.job_off, rec1.job_end,
                 rec1.hz,
                 rec1.pos, nullptr, n_reads, p, t, P.w, kcap, P.pat, P.k, phases, redo, n_redo, anchor_offsets);
      counted = true;
      nr = d2h_scalar(n_redo, st);
      if (nr) {  // uncapped phase selection for reads whose capped prefix was not enough
        Job* jobs2 = scr.alloc<Job>((uint64_t)nr * p);
        uint64_t* kb2 = scr.alloc<uint64_t>((uint64_t)nr * p + 1);
        uint64_t* tot2 = scr.alloc<uint64_t>(1);
        GOD_LAUNCH("k_make_jobs_ids", k_make_jobs_ids, grid_for((uint64_t)nr * p, 256), 256, 0, st, P, offsets, redo,
                   nr, p, jobs2, kb2);
        scan_exclusive_u64(kb2, kb2, (uint64_t)nr * p, tot2, st, scr, "scan_seed_jobs");
        GOD_CUDA(cudaMemcpyAsync(kb2 + (uint64_t)nr * p, tot2, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
        const uint64_t tp2 = d2h_scalar(tot2, st);
        run_extract(P, reads, js1.seq_bytes, jobs2, kb2, nr * p, tp2, false, true, rec2, st, scr, tp2 / 4 + 4096,
                    "extract_phase_redo", nullptr, ORDER_JOB);
        uint32_t* n_redo2 = scr.alloc<uint32_t>(1);
        GOD_CUDA(cudaMemsetAsync(n_redo2, 0, sizeof(uint32_t), st));
        probe_all(v, rec2, st, scr);
        GOD_LAUNCH("k_phase", k_phase, grid_for(nr, 128), 128, 0, st, rec2.cnt, jobs2, rec2.job_off, rec2.job_end,
                   rec2.hz, rec2.pos,
                   redo, nr, p, t, P.w, 0, P.pat, P.k, phases, redo, n_redo2, nullptr);
        GOD_LAUNCH("k_redo_src", k_redo_src, grid_for(nr, 256), 256, 0, st, nr, p, redo, phases, src, srcj);
      }
      have_phase_records = true;
    }
  }
  // ---------------- S3: minimizers of PQ_a (reused from the phase extraction when complete)
  uint32_t* list3 = scr.alloc<uint32_t>(n_reads);
  uint32_t* n3 = scr.alloc<uint32_t>(1);
  GOD_CUDA(cudaMemsetAsync(n3, 0, sizeof(uint32_t), st));
  GOD_LAUNCH("k_seed_plan", k_seed_plan, grid_for(n_reads, 256), 256, 0, st, P.pat, P.k, n_reads, p, phases,
             have_phase_records ? js1.jobs : nullptr, offsets, src, srcj, list3, n3);
  const uint32_t h3 = d2h_scalar(n3, st);
  if (h3) {
    if (h3 == n_reads) {  // every read: phase-a jobs in read order
      JobSet js3 = make_jobs(P, offsets, n_reads, phases, 0, 0, false, st, scr);
      run_extract(P, reads, js3.seq_bytes, js3.jobs, js3.kb, js3.n, js3.total_pos, false, true, rec3, st, scr,
                  js3.total_pos / (uint64_t)(P.w + 1) * 2 + js3.total_pos / 8 + 4096, "extract_seed", js3.x2p(), ORDER_JOB);
      GOD_LAUNCH("k_iota_src3", k_iota_src3, grid_for(n_reads, 256), 256, 0, st, n_reads, src, srcj);
    } else {
      Job* jobs3 = scr.alloc<Job>(h3);
      uint64_t* kb3 = scr.alloc<uint64_t>((uint64_t)h3 + 1);
      uint64_t* tot3 = scr.alloc<uint64_t>(1);
      GOD_LAUNCH("k_make_jobs_sel", k_make_jobs_sel, grid_for(h3, 256), 256, 0, st, P, offsets, list3, h3, phases,
                 jobs3, kb3, src, srcj);
      scan_exclusive_u64(kb3, kb3, h3, tot3, st, scr, "scan_seed_jobs");
      GOD_CUDA(cudaMemcpyAsync(kb3 + h3, tot3, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
      const uint64_t tp3 = d2h_scalar(tot3, st);
      uint64_t bytes = 0;
      d2h_small(&bytes, offsets + n_reads, sizeof(uint64_t), st);
      GOD_CUDA(cudaStreamSynchronize(st));
      run_extract(P, reads, bytes, jobs3, kb3, h3, tp3, false, true, rec3, st, scr, tp3 / 4 + 4096, "extract_seed", nullptr, ORDER_JOB);
    }
  }
  if (h3) probe_all(v, rec3, st, scr);
  // ---------------- S4 fast path: every read's PQ_a records are one job of one extraction, (a) its
  // phase-a job of S1 (short reads in SELECT mode), or (b) its job of the dedicated extraction when
  // that covered every read in read order (p = 1, GIVEN mode, long reads).  Long reads too: 8 lanes
  // walk a read's thousands of records in chunks, which is less even than the general path's thread
  // per record but saves its copy of every record into read order (measured: HiFi 10.4 -> 8.5 ms per
  // step, ONT 8.1 -> 6.8 ms, the writer itself 0.4 -> 1.4 ms on ONT's 100 kbp tail)
  auto fast_path = [&](const Records& rc, const uint8_t* ph, uint32_t pp, bool have_counts) -> uint64_t {
    uint64_t* total = scr.alloc<uint64_t>(1);
    if (!have_counts)
      GOD_LAUNCH("k_read_anchor_counts", k_read_anchor_counts1, grid_for((uint64_t)n_reads * RG, 256), 256, 0, st,
                 rc.cnt, rc.job_off, rc.job_end, ph, pp, n_reads, anchor_offsets);
    scan_exclusive_u64(anchor_offsets, anchor_offsets, n_reads, total, st, scr, "scan_read_anchors");
    GOD_CUDA(cudaMemcpyAsync(anchor_offsets + n_reads, total, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    const uint64_t tot = d2h_scalar(total, st);
    if (tot <= cap) {
      if ((reinterpret_cast<uintptr_t>(anchors) & 15u) == 0)
        GOD_LAUNCH("k_anchor_write", k_anchor_write1<true>, grid_for((uint64_t)n_reads * RG, 256), 256, 0, st, v,
                   rc.hz, rc.pos, rc.cnt, rc.beg, rc.job_off, rc.job_end, ph, pp, n_reads, anchor_offsets, anchors,
                   rid_base);
      else
        GOD_LAUNCH("k_anchor_write", k_anchor_write1<false>, grid_for((uint64_t)n_reads * RG, 256), 256, 0, st, v,
                   rc.hz, rc.pos, rc.cnt, rc.beg, rc.job_off, rc.job_end, ph, pp, n_reads, anchor_offsets, anchors,
                   rid_base);
    }
    return tot;
  };
  if (have_phase_records && nr == 0 && h3 == 0) return fast_path(rec1, phases, p, counted);
  // (GOD_SEED_GENERAL: test hook, forces the general path below)
  if (h3 == n_reads && nr == 0 && !getenv("GOD_SEED_GENERAL"))
    return fast_path(rec3, nullptr, 1, false);  // one job per read, in read order
  SeedSources S{};
  S.hz[0] = rec1.hz; S.pos[0] = rec1.pos; S.off[0] = rec1.job_off; S.cnt[0] = rec1.cnt; S.beg[0] = rec1.beg;
  S.hz[1] = rec2.hz; S.pos[1] = rec2.pos; S.off[1] = rec2.job_off; S.cnt[1] = rec2.cnt; S.beg[1] = rec2.beg;
  S.hz[2] = rec3.hz; S.pos[2] = rec3.pos; S.off[2] = rec3.job_off; S.cnt[2] = rec3.cnt; S.beg[2] = rec3.beg;
  S.end[0] = rec1.job_end; S.end[1] = rec2.job_end; S.end[2] = rec3.job_end;
  // per-read record counts -> offsets -> one contiguous record array in read order
  uint64_t* roff = scr.alloc<uint64_t>((uint64_t)n_reads + 1);
  uint64_t* rtot = scr.alloc<uint64_t>(1);
  GOD_LAUNCH("k_seed_counts", k_seed_counts, grid_for(n_reads, 256), 256, 0, st, S, n_reads, src, srcj, roff);
  scan_exclusive_u64(roff, roff, n_reads, rtot, st, scr, "scan_read_records");
  GOD_CUDA(cudaMemcpyAsync(roff + n_reads, rtot, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  const uint64_t n = d2h_scalar(rtot, st);
  uint64_t* hz = scr.alloc<uint64_t>(n);
  uint32_t* qpos = scr.alloc<uint32_t>(n);
  uint32_t* rid = scr.alloc<uint32_t>(n);
  uint32_t* cnt = scr.alloc<uint32_t>(n);
  uint32_t* beg = scr.alloc<uint32_t>(n);
  uint8_t* inl = scr.alloc<uint8_t>(n);
  GOD_LAUNCH("k_seed_gather", k_seed_gather, grid_for((uint64_t)n_reads * 8, 256), 256, 0, st, S, n_reads, src, srcj,
             roff, hz, qpos, rid, cnt, beg, inl);
  // ---------------- S4: anchors (every read minimizer was probed once, right after its extraction)
  uint64_t* aoff = scr.alloc<uint64_t>(n);
  uint64_t* total = scr.alloc<uint64_t>(1);
  scan_exclusive_u32_to_u64(cnt, aoff, n, total, st, scr, "scan_anchors");
  GOD_LAUNCH("k_read_anchor_offsets", k_read_anchor_offsets, grid_for((uint64_t)n_reads + 1, 256), 256, 0, st, roff,
             aoff, n, total, n_reads, anchor_offsets);
  const uint64_t tot = d2h_scalar(total, st);
  if (tot <= cap && n)
    GOD_LAUNCH("k_anchor_write", k_anchor_write, grid_for(n, 256), 256, 0, st, v, qpos, rid, hz, n, aoff, cnt, beg,
               inl, anchors, rid_base);
  return tot;
}

}  // namespace god
