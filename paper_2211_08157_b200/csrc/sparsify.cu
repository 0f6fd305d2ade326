// sparsify.cu — stage 1 as a standalone parity export (god_sparsify).  The index and seeding paths
// never materialise the sparsified string: extract.cu applies the pattern on the fly.
//
// P:282 (PR/PQ = the non-zero elements of the repeated pattern times the sequence), P:286 (1)-(2),
// P:300 (PQ_s shifted by s).  Reading O3: keep original j iff j >= s and P[(j - s) mod p] = 1.
#include "internal.cuh"

namespace god {

namespace {
__global__ void k_sp_counts(Pattern pat, const uint64_t* __restrict__ offsets, const uint8_t* __restrict__ phases,
                            uint32_t n, uint64_t* counts, uint64_t* words) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t c = included_count(pat, offsets[i + 1] - offsets[i], phases ? phases[i] : 0u);
    counts[i] = c;
    words[i] = (c + 31) / 32;
  }
}

// one thread per output word: 32 kept bases -> 2-bit codes + N bits
__global__ void k_sp_pack(Pattern pat, const uint8_t* __restrict__ seq, const uint64_t* __restrict__ offsets,
                          const uint8_t* __restrict__ phases, uint32_t n, const uint64_t* __restrict__ woff,
                          const uint64_t* __restrict__ counts, uint64_t total_words, uint64_t* packed, uint64_t* nmask) {
  for (uint64_t wi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; wi < total_words;
       wi += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = n - 1;  // sequence = largest i with woff[i] <= wi
    while (lo < hi) {
      uint32_t mid = lo + (hi - lo + 1) / 2;
      if (woff[mid] <= wi) lo = mid;
      else hi = mid - 1;
    }
    const uint32_t i = lo;
    const uint32_t s = phases ? phases[i] : 0u;
    const uint64_t q0 = (wi - woff[i]) * 32;
    const uint64_t cnt = counts[i];
    const uint8_t* src = seq + offsets[i];
    uint64_t word = 0, nm = 0;
    uint64_t o = orig_of(pat, q0, s);
    uint32_t r = (uint32_t)(q0 % pat.x);
    for (uint32_t b = 0; b < 32 && q0 + b < cnt; b++) {
      const uint32_t c = base_code(src[o]);
      o += pat.gap[r];
      r = (r + 1 == pat.x) ? 0 : r + 1;
      if (c > 3) nm |= 1ull << b;
      else word |= (uint64_t)c << (2 * b);
    }
    packed[wi] = word;
    nmask[wi] = nm;
  }
}
}  // namespace

void sparsify(const Params& P, const uint8_t* seq, const uint64_t* offsets, uint32_t n, const uint8_t* phases,
              uint64_t* packed, uint64_t* nmask, uint64_t* out_offsets, uint64_t* counts, uint64_t cap_words,
              uint64_t* needed_host, cudaStream_t st) {
  Scratch scr(st);
  uint64_t* words = scr.alloc<uint64_t>(n);
  uint64_t* tot = scr.alloc<uint64_t>(1);
  if (n) {
    GOD_LAUNCH("k_sp_counts", k_sp_counts, grid_for(n, 256), 256, 0, st, P.pat, offsets, phases, n, counts, words);
  }
  scan_exclusive_u64(words, out_offsets, n, tot, st, scr);
  GOD_CUDA(cudaMemcpyAsync(out_offsets + n, tot, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  const uint64_t total = d2h_scalar(tot, st);
  *needed_host = total;
  if (total > cap_words) throw Fail{GOD_ETRUNC};
  if (total) {
    GOD_LAUNCH("k_sp_pack", k_sp_pack, grid_for(total, 256), 256, 0, st, P.pat, seq, offsets, phases, n, out_offsets, counts, total, packed,
                                                    nmask);
  }
}

}  // namespace god
