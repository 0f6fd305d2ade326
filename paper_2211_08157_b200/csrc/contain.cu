// contain.cu — desk-scale containment search, built from
// the hot path: for each batch of reference sequences (<= batch_bases bases, "-I") the index
// is built on the fly (stages 1-3), every read is phase-selected, seeded and voted against it
// (stages 4 + location voting), and the reads' voted locations are accumulated per reference
// sequence.  Readings C1-C4: DESIGN.md §2 / include/god.h.
#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace god {
namespace {

constexpr unsigned FULLM = 0xffffffffu;

// the batch sequence containing global (batch-relative) position x: largest i with off[i] <= x
__device__ __forceinline__ uint32_t seq_of(const uint64_t* __restrict__ off, uint32_t nb, uint64_t x) {
  uint32_t lo = 0, hi = nb - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// C2/C3: per read, the distinct batch sequences its voted locations fall in (by ref_lo); every
// (read, sequence) pair adds one read and the read's length.  Warp-aggregated: lanes whose current
// sequence is equal combine their contributions before one atomic.
__global__ void k_contain_accum(const god_vote* __restrict__ v, const uint64_t* __restrict__ vo, uint32_t n_reads,
                                const uint64_t* __restrict__ roff, const uint64_t* __restrict__ off, uint32_t nb,
                                uint32_t b0, unsigned long long* __restrict__ mreads,
                                unsigned long long* __restrict__ mbases) {
  const int lane = threadIdx.x & 31;
  for (uint32_t r0 = blockIdx.x * blockDim.x; r0 < n_reads; r0 += gridDim.x * blockDim.x) {  // warp-uniform
    const uint32_t r = r0 + threadIdx.x;
    uint64_t j0 = 0, j1 = 0;
    uint32_t L = 0;
    if (r < n_reads) {
      j0 = vo[r];
      j1 = vo[r + 1];
      L = (uint32_t)(roff[r + 1] - roff[r]);
    }
    for (uint64_t j = j0;; ++j) {
      const bool live = j < j1;
      if (!__any_sync(FULLM, live)) break;
      uint32_t t = 0xffffffffu;
      if (live) {
        t = seq_of(off, nb, v[j].ref_lo);
        for (uint64_t u = j0; u < j; ++u)
          if (seq_of(off, nb, v[u].ref_lo) == t) { t = 0xffffffffu; break; }  // already counted for this read
      }
      const uint32_t m = __match_any_sync(FULLM, t);
      if (t != 0xffffffffu) {
        const uint32_t lo16 = __reduce_add_sync(m, L & 0xFFFFu), hi16 = __reduce_add_sync(m, L >> 16);
        if (lane == __ffs(m) - 1) {
          atomicAdd(mreads + b0 + t, (unsigned long long)__popc(m));
          atomicAdd(mbases + b0 + t, (unsigned long long)lo16 + ((unsigned long long)hi16 << 16));
        }
      }
    }
  }
}

// C4: accepted iff mapped_reads >= min_reads and mapped_bases * cov_den >= cov_num * len
__global__ void k_contain_accept(const uint64_t* __restrict__ mreads, const uint64_t* __restrict__ mbases,
                                 const uint64_t* __restrict__ ref_off, uint32_t n_refs, uint32_t min_reads,
                                 uint32_t cov_num, uint32_t cov_den, uint8_t* __restrict__ acc) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_refs; i += gridDim.x * blockDim.x) {
    const uint64_t len = ref_off[i + 1] - ref_off[i];
    const unsigned __int128 lhs = (unsigned __int128)mbases[i] * cov_den;
    const unsigned __int128 rhs = (unsigned __int128)cov_num * len;
    acc[i] = (uint8_t)(mreads[i] >= min_reads && lhs >= rhs);
  }
}

template <class T>
struct DevBuf {  // grow-only stream-ordered buffer
  T* p = nullptr;
  uint64_t cap = 0;
  cudaStream_t st;
  explicit DevBuf(cudaStream_t s) : st(s) {}
  void need(uint64_t n) {
    if (n <= cap && p) return;
    if (p) cudaFreeAsync(p, st);
    cap = std::max<uint64_t>(n, 1) + n / 8;
    GOD_CUDA(cudaMallocAsync((void**)&p, cap * sizeof(T), st));
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

}  // namespace

void contain(const Params& P, const uint8_t* refs, const uint64_t* ref_off, const uint64_t* ref_off_host,
             uint32_t n_refs, const god_cutoff& cut, const uint8_t* reads, const uint64_t* roff, uint32_t n_reads,
             uint32_t t, const god_vote_params& vp, uint64_t batch_bases, uint32_t min_reads, uint32_t cov_num,
             uint32_t cov_den, uint64_t* mreads, uint64_t* mbases, uint8_t* accepted, cudaStream_t st) {
  GOD_CUDA(cudaMemsetAsync(mreads, 0, n_refs * sizeof(uint64_t), st));
  GOD_CUDA(cudaMemsetAsync(mbases, 0, n_refs * sizeof(uint64_t), st));
  DevBuf<uint64_t> off_b(st), aoff(st), vo(st);
  DevBuf<uint8_t> ph(st);
  DevBuf<god_anchor> an(st);
  DevBuf<god_vote> vv(st);
  aoff.need((uint64_t)n_reads + 1);
  vo.need((uint64_t)n_reads + 1);
  ph.need(n_reads ? n_reads : 1);
  std::vector<uint64_t> hoff;
  const int nsm = num_sms();
  uint32_t b0 = 0;
  while (b0 < n_refs) {
    // C1: consecutive sequences while the batch holds <= batch_bases bases (0: one batch)
    uint32_t b1 = b0 + 1;
    if (!batch_bases) b1 = n_refs;
    else
      while (b1 < n_refs && ref_off_host[b1 + 1] - ref_off_host[b0] <= batch_bases) ++b1;
    const uint32_t nb = b1 - b0;
    GOD_REQUIRE(ref_off_host[b1] - ref_off_host[b0] < (1ull << 32), "a batch must hold < 2^32 bases");
    hoff.resize(nb + 1);
    for (uint32_t i = 0; i <= nb; i++) hoff[i] = ref_off_host[b0 + i] - ref_off_host[b0];
    off_b.need(nb + 1);
    GOD_CUDA(cudaMemcpyAsync(off_b.p, hoff.data(), (nb + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    god_index ix;
    build_index(P, refs + ref_off_host[b0], off_b.p, nb, cut, &ix, st);
    // C2: phase selection + seeding (retried in GIVEN mode with a larger buffer if it did not fit)
    uint64_t na = seed_reads(&ix, reads, roff, n_reads, GOD_PHASE_SELECT, ph.p, t, an.p, aoff.p, an.cap, st);
    if (na > an.cap) {
      an.need(na);
      na = seed_reads(&ix, reads, roff, n_reads, GOD_PHASE_GIVEN, ph.p, t, an.p, aoff.p, an.cap, st);
    }
    uint64_t nv = vote_reads(&ix, reads, roff, n_reads, ph.p, an.p, aoff.p, vp, vv.p, vo.p, vv.cap, st);
    if (nv > vv.cap) {
      vv.need(nv);
      nv = vote_reads(&ix, reads, roff, n_reads, ph.p, an.p, aoff.p, vp, vv.p, vo.p, vv.cap, st);
    }
    if (n_reads)
      GOD_LAUNCH("k_contain_accum", k_contain_accum, std::min<unsigned>(grid_for(n_reads, 256), nsm * 8u), 256, 0, st,
                 vv.p, vo.p, n_reads, roff, off_b.p, nb, b0, (unsigned long long*)mreads,
                 (unsigned long long*)mbases);
    if (ix.dir) cudaFreeAsync(ix.dir, st);
    if (ix.ent) cudaFreeAsync(ix.ent, st);
    if (ix.seg) cudaFreeAsync(ix.seg, st);
    ix.dir = nullptr; ix.ent = nullptr; ix.seg = nullptr;
    b0 = b1;
  }
  if (n_refs)
    GOD_LAUNCH("k_contain_accept", k_contain_accept, grid_for(n_refs, 256), 256, 0, st, mreads, mbases, ref_off, n_refs,
               min_reads, cov_num, cov_den, accepted);
  GOD_CUDA(cudaStreamSynchronize(st));
}

}  // namespace god
