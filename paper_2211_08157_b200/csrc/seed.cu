// seed.cu — stage 4: pattern alignment (phase selection) and compressed seeding.
//
// Pipeline (kernels S1-S4), all reads in one batch:
//   S1  extraction (extract.cu) over the (read, s) jobs for s < p, each capped to the first
//       KCAP k-mer starts ("limit the number of calculated minimizers in each PQ_s"):
//       records at k-mer index <= KCAP - w are exactly the first minimizers of the full PQ_s
//   S2  one thread per read: c = min(t, min_s |M_s|), score_s = sum over the first c records of
//       occ(hash) (index probes), a = argmax (smallest s on ties).  Reads whose capped prefix gave
//       fewer than t exact records for some phase (N-dense prefixes) are recomputed uncapped.
//   S3  extraction over the (read, a_r) jobs -> all minimizers of PQ_a
//   S4  per record: probe -> anchor count; exclusive scan; probe again -> write anchors
#include "internal.cuh"

namespace god {

namespace {

__global__ void k_phase(IndexView v, const Job* __restrict__ jobs, const uint64_t* __restrict__ job_off,
                        const uint64_t* __restrict__ hz, const uint32_t* __restrict__ pos, const uint32_t* __restrict__ ids,
                        uint32_t n_reads, uint32_t p, uint32_t t, uint32_t w, uint32_t kcap, Pattern pat, int k,
                        uint8_t* phases, uint32_t* redo, uint32_t* n_redo) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_reads; i += gridDim.x * blockDim.x) {
    const uint32_t r = ids ? ids[i] : i;
    uint64_t nmin = ~0ull;
    bool fallback = false;
    for (uint32_t s = 0; s < p; s++) {
      const uint64_t j = (uint64_t)i * p + s;
      const Job jb = jobs[j];
      uint64_t c = job_off[j + 1] - job_off[j];
      if (kcap) {
        const uint64_t ninc = included_count(pat, jb.len, s);
        const uint64_t nk_full = ninc >= (uint64_t)k ? ninc - k + 1 : 0;
        if (nk_full > jb.nk) {  // truncated: only records with k-mer index <= nk - w are exact
          uint64_t safe = 0;
          if (jb.nk >= w) {
            const uint64_t lim = orig_of(pat, jb.nk - w, s);
            for (uint64_t q = job_off[j]; q < job_off[j + 1] && pos[q] <= lim; q++) ++safe;
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
      for (uint64_t q = 0; q < c; q++) {
        const uint2 rg = probe_range(v, hz[job_off[j] + q] & ((1ull << 63) - 1));
        sc += rg.y - rg.x;
      }
      if (s == 0 || sc > best) { best = sc; a = s; }
    }
    phases[r] = (uint8_t)a;
  }
}

__global__ void k_gather_offsets(const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ ids, uint32_t n,
                                 uint64_t* seq_off, uint64_t* seq_len) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    seq_off[i] = offsets[ids[i]];
    seq_len[i] = offsets[ids[i] + 1] - offsets[ids[i]];
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

__global__ void k_anchor_count(IndexView v, const uint64_t* __restrict__ hz, uint64_t n, uint32_t* cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 rg = probe_range(v, hz[i] & ((1ull << 63) - 1));
    cnt[i] = rg.y - rg.x;
  }
}

__global__ void k_anchor_write(IndexView v, const uint64_t* __restrict__ hz, const uint32_t* __restrict__ pos,
                               const uint32_t* __restrict__ job, uint64_t n, const uint64_t* __restrict__ aoff,
                               god_anchor* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = hz[i];
    const uint2 rg = probe_range(v, h & ((1ull << 63) - 1));
    uint64_t o = aoff[i];
    const uint32_t qz = (uint32_t)(h >> 63), qpos = pos[i], rid = job[i];
    for (uint32_t e = rg.x; e < rg.y; e++, o++) {
      god_anchor an;
      an.ref_pos = __ldg(v.ent_pos + e);
      an.read_pos = qpos;
      an.read_id = rid;
      an.strand = (__ldg(v.ent_key + e) & 1u) ^ qz;
      out[o] = an;
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

uint64_t seed_reads(const god_index* ix, const uint8_t* reads, const uint64_t* offsets, uint32_t n_reads,
                    god_phase_mode mode, uint8_t* phases, uint32_t t, god_anchor* anchors, uint64_t* anchor_offsets,
                    uint64_t cap, cudaStream_t st) {
  Scratch scr(st);
  const Params& P = ix->P;
  const uint32_t p = P.pat.p;
  const IndexView v = ix->view();
  if (n_reads == 0) {
    GOD_CUDA(cudaMemsetAsync(anchor_offsets, 0, sizeof(uint64_t), st));
    return 0;
  }
  // ---------------- S1/S2: pattern alignment
  if (mode == GOD_PHASE_SELECT) {
    if (p == 1) {
      GOD_CUDA(cudaMemsetAsync(phases, 0, n_reads, st));
    } else {
      const uint32_t kcap = (t + 1) * (uint32_t)P.w + (uint32_t)P.w;
      JobSet js = make_jobs(P, offsets, n_reads, nullptr, p, kcap, false, st, scr);
      const uint64_t js_bytes = js.seq_bytes;
      Records rec;
      run_extract(P, reads, js.seq_bytes, js.jobs, js.kb, js.n, js.total_pos, false, true, rec, st, scr,
                  js.total_pos / (uint64_t)(P.w + 1) * 2 + js.total_pos / 8 + 4096, "extract_phase");
      uint32_t* redo = scr.alloc<uint32_t>(n_reads);
      uint32_t* n_redo = scr.alloc<uint32_t>(1);
      GOD_CUDA(cudaMemsetAsync(n_redo, 0, sizeof(uint32_t), st));
      GOD_LAUNCH("k_phase", k_phase, grid_for(n_reads, 128), 128, 0, st, v, js.jobs, rec.job_off, rec.hz, rec.pos, nullptr, n_reads, p, t,
                                                      P.w, kcap, P.pat, P.k, phases, redo, n_redo);
      const uint32_t nr = d2h_scalar(n_redo, st);
      if (nr) {  // uncapped phase selection for reads whose capped prefix was not enough
        Job* jobs2 = scr.alloc<Job>((uint64_t)nr * p);
        uint64_t* kb2 = scr.alloc<uint64_t>((uint64_t)nr * p + 1);
        uint64_t* tot2 = scr.alloc<uint64_t>(1);
        GOD_LAUNCH("k_make_jobs_ids", k_make_jobs_ids, grid_for((uint64_t)nr * p, 256), 256, 0, st, P, offsets, redo, nr, p, jobs2, kb2);
        scan_exclusive_u64(kb2, kb2, (uint64_t)nr * p, tot2, st, scr);
        GOD_CUDA(cudaMemcpyAsync(kb2 + (uint64_t)nr * p, tot2, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
        const uint64_t tp2 = d2h_scalar(tot2, st);
        Records rec2;
        run_extract(P, reads, js_bytes, jobs2, kb2, nr * p, tp2, false, true, rec2, st, scr, tp2 / 4 + 4096, "extract_phase_redo");
        uint32_t* n_redo2 = scr.alloc<uint32_t>(1);
        GOD_CUDA(cudaMemsetAsync(n_redo2, 0, sizeof(uint32_t), st));
        GOD_LAUNCH("k_phase", k_phase, grid_for(nr, 128), 128, 0, st, v, jobs2, rec2.job_off, rec2.hz, rec2.pos, redo, nr, p, t, P.w, 0,
                                                   P.pat, P.k, phases, redo, n_redo2);
      }
    }
  }
  // ---------------- S3: minimizers of PQ_a
  JobSet js = make_jobs(P, offsets, n_reads, phases, 0, 0, false, st, scr);
  Records rec;
  run_extract(P, reads, js.seq_bytes, js.jobs, js.kb, js.n, js.total_pos, true, true, rec, st, scr,
              js.total_pos / (uint64_t)(P.w + 1) * 2 + js.total_pos / 8 + 4096, "extract_seed");
  // ---------------- S4: probes -> anchors
  const uint64_t n = rec.n;
  uint32_t* cnt = scr.alloc<uint32_t>(n);
  uint64_t* aoff = scr.alloc<uint64_t>(n);
  uint64_t* total = scr.alloc<uint64_t>(1);
  if (n) {
    GOD_LAUNCH("k_anchor_count", k_anchor_count, grid_for(n, 256), 256, 0, st, v, rec.hz, n, cnt);
  }
  scan_exclusive_u32_to_u64(cnt, aoff, n, total, st, scr);
  GOD_LAUNCH("k_read_anchor_offsets", k_read_anchor_offsets, grid_for((uint64_t)n_reads + 1, 256), 256, 0, st, rec.job_off, aoff, n, total, n_reads,
                                                                             anchor_offsets);
  const uint64_t tot = d2h_scalar(total, st);
  if (tot <= cap && n) {
    GOD_LAUNCH("k_anchor_write", k_anchor_write, grid_for(n, 256), 256, 0, st, v, rec.hz, rec.pos, rec.job, n, aoff, anchors);
  }
  return tot;
}

}  // namespace god
