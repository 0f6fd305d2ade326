// extract.cu — fused sparsify + double-strand (w,k)-minimizer extraction (stages 1+2 of the hot path).
//
// PAPER.md: P:286 (1)-(3) (diet pattern -> patterned sequence -> minimizers, start locations in
// original coordinates), P:294 (double-strand (w,k)-minimizer), P:300/P:308 (PQ_s, PQ_a),
// P:370 (2-bit encoding, Wang hash, an N terminates the computation).  Readings: DESIGN.md §2.
//
// Design (kernel K1): the extraction index space is the concatenation over jobs
// of [k-mer starts of the job, one separator].  A CTA owns a tile of T consecutive positions
// plus a (w-1) halo on each side.  (1) Each thread rolls the canonical k-mer over a contiguous
// chunk of the extended tile directly from the ASCII bytes (the pattern is applied on the fly
// via the orig() map, so the sparsified string is never materialised) and writes
// H = hash + 1 (0 = barrier: N-spanning k-mer, separator or outside; ~0 = palindrome) to SMEM.
// (2) Window minima by van Herk/Gil-Werman (prefix/suffix minima over blocks of w), then the
// sliding MAX of the window minima the same way: position j is a minimizer iff
// H[j] == max_{windows W containing j} min(W)  (all ties kept; windows crossing a barrier have
// min 0 and never select).  Runs shorter than w (partial window) are fixed up directly.
// (3) Ordered compaction: block scan + decoupled look-back across tiles, so records come out in
// position order (per job: the order the oracle and god_minimizers define).
#include "internal.cuh"

namespace god {

namespace {
constexpr int EX_NT = 256;
constexpr int EX_CPT = 8;
constexpr int EX_T = EX_NT * EX_CPT;  // interior positions per tile
constexpr uint64_t H_PAL = ~0ull;

struct ExArgs {
  Params P;
  const uint8_t* seq;
  const Job* jobs;
  const uint64_t* kb;
  uint32_t n_jobs;
  uint64_t total_pos;
  uint64_t* status;
  uint32_t* tile_ctr;
  uint64_t* out_hz;
  uint32_t* out_pos;
  uint32_t* out_job;
  uint64_t* job_off;
  uint64_t cap;
  uint64_t* total_out;
};

// largest j in [lo, hi] with kb[j] <= g  (kb ascending, kb[lo] <= g)
__device__ __forceinline__ uint32_t find_job(const uint64_t* kb, uint32_t lo, uint32_t hi, uint64_t g) {
  while (lo < hi) {
    uint32_t mid = lo + (hi - lo + 1) / 2;
    if (kb[mid] <= g) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(EX_NT) k_extract(ExArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int w = a.P.w, k = a.P.k;
  const int E = EX_T + 2 * (w - 1);
  uint64_t* H = reinterpret_cast<uint64_t*>(smem);
  uint64_t* PF = H + E;
  uint64_t* SF = PF + E;
  uint64_t* WM = SF + E;
  uint32_t* JX = reinterpret_cast<uint32_t*>(WM + E);  // job index | (1<<31 if first position of job)
  uint8_t* Z = reinterpret_cast<uint8_t*>(JX + E);
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_j0, s_j1;
  __shared__ uint32_t warp_cnt[EX_NT / 32];
  __shared__ uint64_t s_base;

  const int tid = threadIdx.x;
  if (tid == 0) {
    uint32_t t = atomicAdd(a.tile_ctr, 1u);
    s_tile = t;
    int64_t g0 = (int64_t)t * EX_T - (w - 1);
    uint64_t gfirst = g0 < 0 ? 0 : (uint64_t)g0;
    uint64_t glast = (uint64_t)t * EX_T + EX_T + (w - 1);
    if (glast >= a.total_pos) glast = a.total_pos ? a.total_pos - 1 : 0;
    s_j0 = find_job(a.kb, 0, a.n_jobs - 1, gfirst);
    s_j1 = find_job(a.kb, s_j0, a.n_jobs - 1, glast);
  }
  __syncthreads();
  const uint64_t tile = s_tile;
  const int64_t g0 = (int64_t)tile * EX_T - (w - 1);  // global index of extended position 0
  const uint32_t j0 = s_j0, j1 = s_j1;
  const Pattern& pat = a.P.pat;
  const uint64_t kmask = a.P.kmask;
  const int rshift = 2 * (k - 1);

  // ---------------------------------------------------------------- (1) hashes
  {
    const int per = (E + EX_NT - 1) / EX_NT;
    int e = tid * per;
    const int eend = min(E, e + per);
    int64_t g = g0 + e;
    uint32_t J = j0;
    bool have_job = false;
    while (e < eend) {
      if (g < 0 || (uint64_t)g >= a.total_pos) {
        H[e] = 0; JX[e] = 0; Z[e] = 0;
        ++e; ++g;
        continue;
      }
      if (!have_job) { J = find_job(a.kb, j0, j1, (uint64_t)g); have_job = true; }
      while (J + 1 < a.n_jobs && a.kb[J + 1] <= (uint64_t)g) ++J;
      const Job jb = a.jobs[J];
      const uint64_t local = (uint64_t)g - a.kb[J];
      const uint32_t first_flag = local == 0 ? 0x80000000u : 0u;
      if (local >= jb.nk) {  // separator
        H[e] = 0; JX[e] = J | first_flag; Z[e] = 0;
        ++e; ++g;
        continue;
      }
      const int cnt = (int)min((uint64_t)(eend - e), (uint64_t)jb.nk - local);
      // roll over included bases local .. local + cnt + k - 2
      uint32_t r = (uint32_t)(local % pat.x);
      uint64_t o = orig_of(pat, local, jb.phase);
      const uint8_t* s = a.seq + jb.seq_off;
      uint64_t fwd = 0, rev = 0;
      int nv = 0;
      const int nb = cnt + k - 1;
      for (int i = 0; i < nb; i++) {
        uint32_t c = base_code(__ldg(s + o));
        o += pat.gap[r];
        r = (r + 1 == pat.x) ? 0 : r + 1;
        if (c > 3) { nv = 0; c = 0; } else { ++nv; }
        fwd = ((fwd << 2) | c) & kmask;
        rev = (rev >> 2) | ((uint64_t)(3 - c) << rshift);
        if (i >= k - 1) {
          const int ee = e + i - (k - 1);
          uint64_t h = 0;
          uint8_t z = 0;
          if (nv >= k) {
            if (fwd == rev) h = H_PAL;
            else {
              z = fwd > rev;
              h = wang_hash(z ? rev : fwd, kmask) + 1;
            }
          }
          H[ee] = h; Z[ee] = z;
          JX[ee] = J | ((local + (uint64_t)(i - (k - 1)) == 0) ? 0x80000000u : 0u);
        }
      }
      e += cnt; g += cnt;
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- (2) window minima (van Herk)
  const int nblk = (E + w - 1) / w;
  for (int b = tid; b < nblk; b += EX_NT) {
    const int s0 = b * w, s1 = min(s0 + w, E);
    uint64_t m = ~0ull;
    for (int e = s0; e < s1; e++) { m = min(m, H[e]); PF[e] = m; }
    m = ~0ull;
    for (int e = s1 - 1; e >= s0; e--) { m = min(m, H[e]); SF[e] = m; }
  }
  __syncthreads();
  const int NA = E - w + 1;  // window starts a in [0, NA): window [a, a+w-1]
  for (int x = tid; x < NA; x += EX_NT) WM[x] = (x % w == 0) ? SF[x] : min(SF[x], PF[x + w - 1]);
  __syncthreads();
  const int nblk2 = (NA + w - 1) / w;
  for (int b = tid; b < nblk2; b += EX_NT) {
    const int s0 = b * w, s1 = min(s0 + w, NA);
    uint64_t m = 0;
    for (int e = s0; e < s1; e++) { m = max(m, WM[e]); PF[e] = m; }
    m = 0;
    for (int e = s1 - 1; e >= s0; e--) { m = max(m, WM[e]); SF[e] = m; }
  }
  __syncthreads();

  // ---------------------------------------------------------------- (3) select + ordered compaction
  const int e_begin = (w - 1) + tid * EX_CPT;
  uint32_t selmask = 0;
#pragma unroll
  for (int i = 0; i < EX_CPT; i++) {
    const int e = e_begin + i;
    const uint64_t h = H[e];
    if (h == 0 || h == H_PAL) continue;
    const int x = e - (w - 1);  // first window start covering e
    const uint64_t mm = (x % w == 0) ? SF[x] : max(SF[x], PF[x + w - 1]);
    bool sel = (h == mm);
    if (mm == 0) {  // run shorter than w: one partial window = the whole run (reading O6)
      int lo = e, hi = e;
      while (lo - 1 >= 0 && H[lo - 1] != 0) --lo;
      while (hi + 1 < E && H[hi + 1] != 0) ++hi;
      uint64_t m = ~0ull;
      for (int q = lo; q <= hi; q++) if (H[q] != H_PAL) m = min(m, H[q]);
      sel = (h == m);
    }
    if (sel) selmask |= 1u << i;
  }
  const uint32_t cnt = __popc(selmask);
  const int lane = tid & 31, wid = tid >> 5;
  uint32_t incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) warp_cnt[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t ws = lane < EX_NT / 32 ? warp_cnt[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, ws, d);
      if (lane >= d) ws += y;
    }
    if (lane < EX_NT / 32) warp_cnt[lane] = ws;
    if (lane == EX_NT / 32 - 1) {
      uint64_t base = lb_exclusive(a.status, tile, ws);
      s_base = base;
      const uint64_t ntiles = (a.total_pos + EX_T - 1) / EX_T;
      if (tile == ntiles - 1) *a.total_out = base + ws;
    }
  }
  __syncthreads();
  uint64_t idx = s_base + (wid ? warp_cnt[wid - 1] : 0) + incl - cnt;
  const uint64_t tile_g0 = tile * EX_T;
#pragma unroll
  for (int i = 0; i < EX_CPT; i++) {
    const int e = e_begin + i;
    const uint64_t g = tile_g0 + (uint64_t)tid * EX_CPT + i;
    if (g >= a.total_pos) break;
    const uint32_t jx = JX[e];
    const uint32_t J = jx & 0x7FFFFFFFu;
    if ((jx & 0x80000000u) && a.job_off) a.job_off[J] = idx;
    if (selmask & (1u << i)) {
      if (idx < a.cap) {
        const Job jb = a.jobs[J];
        const uint64_t local = g - a.kb[J];
        a.out_hz[idx] = (H[e] - 1) | ((uint64_t)Z[e] << 63);
        a.out_pos[idx] = (uint32_t)(jb.pos_base + orig_of(pat, local, jb.phase));
        if (a.out_job) a.out_job[idx] = J;
      }
      ++idx;
    }
  }
}

// ---------------------------------------------------------------------------------- job building
// kb[j]: the generic layout's nk + 1 (one separator per job), or with x2 the specialised kernel's
// padded count (nk rounded up to a multiple of w, >= w) and cw[j] its 16-base code words; nk_sum
// accumulates the k-mer starts (x2 only)
__global__ void k_make_jobs(Params P, const uint64_t* offsets, uint32_t n_seqs, const uint8_t* phases, uint32_t p_all,
                            uint32_t kcap, int global_pos, Job* jobs, uint64_t* nkp1, int x2, uint64_t* cw,
                            unsigned long long* nk_sum) {
  const uint64_t nj = p_all ? (uint64_t)n_seqs * p_all : n_seqs;
  uint64_t acc = 0, mxb = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nj; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j32 = (uint32_t)j;  // nj < 2^31 (make_jobs)
    const uint64_t sidx = p_all ? j32 / p_all : j32;
    const uint32_t s = p_all ? j32 % p_all : (phases ? phases[sidx] : 0u);
    Job jb;
    jb.seq_off = offsets[sidx];
    jb.len = offsets[sidx + 1] - offsets[sidx];
    jb.pos_base = global_pos ? jb.seq_off : 0;
    jb.phase = s;
    const uint64_t ninc = included_count(P.pat, jb.len, s);
    uint64_t nk = ninc >= (uint64_t)P.k ? ninc - P.k + 1 : 0;
    if (kcap && nk > kcap) nk = kcap;
    jb.nk = (uint32_t)nk;
    jobs[j] = jb;
    if (x2) {
      const uint32_t W = (uint32_t)P.w, nk32 = (uint32_t)nk;  // nk fits 32 bits (Job::nk)
      const uint32_t blocks = nk32 ? (nk32 - 1) / W + 1 : 1u;  // ceil(nk / W)
      nkp1[j] = (uint64_t)blocks * W;
      cw[j] = nk ? (nk + P.k - 1 + 15) / 16 : 0;
      acc += nk;
      mxb = max(mxb, (uint64_t)blocks);
    } else {
      nkp1[j] = nk + 1;
    }
  }
  if (x2) {
    for (int d = 16; d; d >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, d);
      mxb = max(mxb, __shfl_xor_sync(0xffffffffu, mxb, d));
    }
    // one atomic per CTA on each of the two words (a per-warp atomic on one global word serialises:
    // 625 k of them for the 20 M read jobs of the human step)
    __shared__ unsigned long long s_mx, s_acc;
    if (threadIdx.x == 0) { s_mx = 0; s_acc = 0; }
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && mxb) atomicMax(&s_mx, (unsigned long long)mxb);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&s_acc, (unsigned long long)acc);
    __syncthreads();
    if (threadIdx.x == 0 && s_mx) atomicMax(nk_sum + 1, s_mx);
    if (threadIdx.x == 0 && s_acc) atomicAdd(nk_sum, s_acc);
  }
}
}  // namespace

JobSet make_jobs(const Params& P, const uint64_t* offsets, uint32_t n_seqs, const uint8_t* phases, uint32_t p_all,
                 uint32_t kcap, bool global_pos, cudaStream_t st, Scratch& scr) {
  JobSet js;
  const uint64_t nj = p_all ? (uint64_t)n_seqs * p_all : n_seqs;
  GOD_REQUIRE(nj < 0x7FFFFFFFull, "too many (sequence, phase) jobs");
  js.n = (uint32_t)nj;
  js.jobs = scr.alloc<Job>(nj);
  if (nj && x2_supported(P)) {  // the specialised kernel's layout in the same pass (no generic layout)
    uint64_t* kb = scr.alloc<uint64_t>(nj + 1);
    uint64_t* cw = scr.alloc<uint64_t>(nj + 1);
    uint64_t* tot = scr.alloc<uint64_t>(4);
    GOD_CUDA(cudaMemsetAsync(tot + 2, 0, 2 * sizeof(uint64_t), st));
    GOD_LAUNCH("k_make_jobs", k_make_jobs, grid_for(nj, 256), 256, 0, st, P, offsets, n_seqs, phases, p_all, kcap,
               global_pos, js.jobs, kb, 1, cw, reinterpret_cast<unsigned long long*>(tot + 2));
    scan_exclusive_u64(kb, kb, nj, tot, st, scr, "scan_jobs");
    scan_exclusive_u64(cw, cw, nj, tot + 1, st, scr, "scan_jobs");
    GOD_CUDA(cudaMemcpyAsync(kb + nj, tot, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    GOD_CUDA(cudaMemcpyAsync(cw + nj, tot + 1, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    uint64_t h[5] = {0, 0, 0, 0, 0};
    d2h_small(h, tot, 4 * sizeof(uint64_t), st);
    d2h_small(&h[4], offsets + n_seqs, sizeof(uint64_t), st);
    js.x2.kb = kb;
    js.x2.cw = cw;
    js.x2.total_pos = h[0];
    js.x2.nk_sum = h[2];
    js.x2.max_job_blocks = h[3];
    js.total_pos = h[2] + nj;  // the generic layout's size (cap estimates)
    js.seq_bytes = h[4];
    return js;
  }
  js.kb = scr.alloc<uint64_t>(nj + 1);
  uint64_t* tot = scr.alloc<uint64_t>(1);
  if (nj) {
    GOD_LAUNCH("k_make_jobs", k_make_jobs, grid_for(nj, 256), 256, 0, st, P, offsets, n_seqs, phases, p_all, kcap,
               global_pos, js.jobs, js.kb, 0, nullptr, nullptr);
  }
  scan_exclusive_u64(js.kb, js.kb, nj, tot, st, scr, "scan_jobs");
  GOD_CUDA(cudaMemcpyAsync(js.kb + nj, tot, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  uint64_t h[2] = {0, 0};
  d2h_small(&h[0], tot, sizeof(uint64_t), st);
  d2h_small(&h[1], offsets + n_seqs, sizeof(uint64_t), st);
  js.total_pos = h[0];
  js.seq_bytes = h[1];
  return js;
}

void run_extract(const Params& P, const uint8_t* seq, uint64_t seq_bytes, const Job* jobs, const uint64_t* kb,
                 uint32_t n_jobs, uint64_t total_pos, bool want_job, bool want_job_off, Records& rec, cudaStream_t st,
                 Scratch& scr, uint64_t cap_hint, const char* tag, const X2Layout* x2, RecOrder order,
                 const SeqStream* ss) {
  rec.n = 0;
  if (run_extract2(P, seq, seq_bytes, jobs, n_jobs, want_job, want_job_off, rec, st, scr, cap_hint, tag, x2, order, ss))
    return;
  if (ss) ss->wait_all(st);  // the generic kernel reads the whole buffer
  if (n_jobs == 0 || total_pos == 0) {
    rec.cap = 1;
    rec.hz = scr.alloc<uint64_t>(1);
    rec.pos = scr.alloc<uint32_t>(1);
    if (want_job) rec.job = scr.alloc<uint32_t>(1);
    if (want_job_off) {
      rec.job_off = scr.alloc<uint64_t>(n_jobs + 1);
      rec.job_end = rec.job_off + 1;
      GOD_CUDA(cudaMemsetAsync(rec.job_off, 0, (n_jobs + 1) * sizeof(uint64_t), st));
    }
    return;
  }
  const uint64_t ntiles = (total_pos + EX_T - 1) / EX_T;
  GOD_REQUIRE(ntiles < 0x7FFFFFFFull, "input too large for one extraction launch");
  prof_add_units(tag, total_pos - n_jobs);  // kb = exclusive scan of nk + 1 (one separator per job)
  const int E = EX_T + 2 * (P.w - 1);
  const size_t smem = (size_t)E * (4 * sizeof(uint64_t) + sizeof(uint32_t) + 1);
  static DeviceOnce attr_once;
  attr_once.run([] { GOD_CUDA(cudaFuncSetAttribute(k_extract, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); });
  uint64_t cap = cap_hint ? cap_hint : total_pos;
  if (cap > total_pos) cap = total_pos;
  uint64_t* status = scr.alloc<uint64_t>(ntiles);
  uint32_t* ctr = scr.alloc<uint32_t>(1);
  uint64_t* dtotal = scr.alloc<uint64_t>(1);
  if (want_job_off) {
    rec.job_off = scr.alloc<uint64_t>(n_jobs + 1);
    rec.job_end = rec.job_off + 1;  // position order: a job ends where the next begins
  }
  for (int attempt = 0; attempt < 2; attempt++) {
    rec.cap = cap;
    rec.hz = scr.alloc<uint64_t>(cap);
    rec.pos = scr.alloc<uint32_t>(cap);
    rec.job = want_job ? scr.alloc<uint32_t>(cap) : nullptr;
    GOD_CUDA(cudaMemsetAsync(status, 0, ntiles * sizeof(uint64_t), st));
    GOD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
    ExArgs a{P, seq, jobs, kb, n_jobs, total_pos, status, ctr, rec.hz, rec.pos, rec.job, rec.job_off, cap, dtotal};
    GOD_LAUNCH(tag, k_extract, (unsigned)ntiles, EX_NT, smem, st, a);
    uint64_t n = d2h_scalar(dtotal, st);
    if (n <= cap) {
      rec.n = n;
      if (want_job_off) GOD_CUDA(cudaMemcpyAsync(rec.job_off + n_jobs, dtotal, sizeof(uint64_t),
                                                 cudaMemcpyDeviceToDevice, st));
      return;
    }
    cap = n;  // grow and rerun (rare: only when the density estimate was too low)
  }
  GOD_REQUIRE(false, "extraction capacity retry failed");
}

}  // namespace god
