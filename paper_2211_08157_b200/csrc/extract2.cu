// extract2.cu — K1 v2: register-resident fused sparsify + minimizer extraction (stages 1+2).
//
// Same definitions as extract.cu (P:282/P:286/P:294/P:300/P:370; readings O1-O6 of DESIGN.md §2),
// specialised at compile time for the hot configurations: k, w and patterns with exactly one '1'
// (period PS = 1: "1"; PS = 2: "10"/"01").  Everything else runs the generic kernel (extract.cu).
//
// Layout.  Each job's k-mer starts are padded to a multiple of W positions (the pad slots are
// window barriers), so a W-block never straddles two jobs; each job's patterned bases are packed
// 16 per u32 word, MSB-first, starting on a fresh word.  A CTA of 256 threads owns 256 W-blocks
// (thread t = block t); blocks 0 and 255 are halo (computed, not emitted), so consecutive tiles
// overlap by two blocks.
//   A. sparsify: the tile's code words are built once in SMEM straight from the ASCII bytes
//      (PRMT gathers the included bytes, SIMD 2-bit encode, an IMAD packs 4 codes, a 256-entry
//      SMEM table of expected letters detects any non-ACGT byte exactly).
//   B. per thread: its W k-mers are extracted from a funnel-aligned window of the code words
//      (fwd) and of its reverse complement (rev); canonical = min, strand = fwd > rev; masked Wang
//      hash; key = top 31 hash bits + 1 (0 = barrier, ~0 = palindrome).
//   C. selection in registers on 32-bit keys (van Herk/Gil-Werman): block prefix/suffix minima,
//      window minima (next block's prefix minima by shuffle), block prefix/suffix maxima of the
//      window minima, MM = max over the windows containing the position (previous block's suffix
//      maxima by shuffle); candidate iff key == MM.  Keys are monotone in the hash, so every true
//      minimizer is a candidate; a candidate can be false only if two candidates closer than w
//      share a key but not a hash — checked exactly after compaction.
//   D. exact slow path for the whole tile (64-bit hashes in SMEM, direct window rule incl. partial
//      windows) when the tile has an N, a run shorter than w, or such a key tie.
//   E. ordered compaction: staged in SMEM, tile offset by decoupled look-back, coalesced copy.
#include "internal.cuh"

namespace god {

namespace {

constexpr int X2_NT = 256;
constexpr int X2_OUT_BLOCKS = X2_NT - 2;

struct X2Args {
  const uint8_t* seq;
  uint64_t seq_bytes;
  const Job* jobs;
  const uint64_t* kb;   // padded position base per job (multiple of W), [n_jobs + 1]
  const uint64_t* cw;   // code-word base per job, [n_jobs + 1]
  uint32_t n_jobs;
  uint64_t total_blocks;
  uint32_t one0;        // offset of the single '1' of the pattern
  uint32_t key_shift;   // key = (hash >> key_shift) + 1
  uint64_t* status;
  uint32_t* tile_ctr;
  uint64_t* out_hz;
  uint32_t* out_pos;
  uint32_t* out_job;
  uint64_t* job_off;
  uint64_t cap;
  uint64_t* total_out;
};

__device__ __forceinline__ uint32_t find_job_le(const uint64_t* arr, uint32_t lo, uint32_t hi, uint64_t g) {
  // largest j in [lo, hi] with arr[j] <= g  (arr ascending, arr[lo] <= g)
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo + 1) / 2;
    if (arr[mid] <= g) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <int NW>
__device__ __forceinline__ uint32_t word_at(const uint32_t (&w)[NW], int i) {
  return i < NW ? w[i] : 0u;
}

// bits [S, S+LEN) of the MSB-first bit string held in w[], right-aligned (LEN <= 56).  Called
// from fully unrolled loops, so S is a compile-time constant after inlining (no local memory).
template <int NW>
__device__ __forceinline__ uint64_t ext_bits(const uint32_t (&w)[NW], const int S, const int LEN) {
  const int w0 = S >> 5, off = S & 31;
  const uint64_t hi64 = ((uint64_t)word_at(w, w0) << 32) | word_at(w, w0 + 1);
  const uint64_t v = off ? (hi64 << off) | (word_at(w, w0 + 2) >> (32 - off)) : hi64;
  return v >> (64 - LEN);
}

__device__ __forceinline__ uint32_t rev2(uint32_t x) {  // reverse the 16 2-bit fields of x
  const uint32_t y = __brev(x);
  return ((y >> 1) & 0x55555555u) | ((y & 0x55555555u) << 1);
}

template <int K>
__device__ __forceinline__ uint64_t wang_hash_k(uint64_t key) {
  constexpr uint64_t mask = (K >= 32) ? ~0ull : ((1ull << (2 * K)) - 1);
  key = (~key + (key << 21)) & mask;
  key = key ^ (key >> 24);
  key = (key * 265ull) & mask;
  key = key ^ (key >> 14);
  key = (key * 21ull) & mask;
  key = key ^ (key >> 28);
  key = (key + (key << 31)) & mask;
  return key;
}

struct X2Shared {
  uint32_t j0, j1;
  uint64_t cw_lo, cw_hi;
  uint32_t any_n, slow, tie;
  uint64_t base;
  uint32_t warp_cnt[X2_NT / 32];
  uint32_t tile;
};

template <int K, int W, int PS>
struct X2Cfg {
  static constexpr int NB = W + K - 1;                 // bases in a thread's window
  static constexpr int NWIN = (2 * NB + 31) / 32;       // aligned window words
  static constexpr int NLOAD = (30 + 2 * NB + 31) / 32; // words loaded before alignment
  static constexpr int POS = X2_NT * W;                 // positions per tile (incl. halo blocks)
  // code words the tile can touch: every block's window, plus one partial word per job (<= 256 jobs)
  static constexpr int MAXWORDS = (POS + X2_NT * (K - 1) + 15) / 16 + X2_NT + 8;
};

// ---------------------------------------------------------------------------------------------
template <int K, int W, int PS>
__global__ void __launch_bounds__(X2_NT, 1) k_extract2(X2Args a) {
  using C = X2Cfg<K, W, PS>;
  constexpr int NB = C::NB, NWIN = C::NWIN, NLOAD = C::NLOAD, POS = C::POS;
  extern __shared__ __align__(16) unsigned char x2_smem[];
  // layout: lut[256] | codes[MAXWORDS] | nmask[MAXWORDS] | xchg[2][8][W] | stage (12 B x POS, or 8 B x POS H64)
  uint32_t* lut = reinterpret_cast<uint32_t*>(x2_smem);
  uint32_t* codes = lut + 256;
  uint32_t* nmask = codes + C::MAXWORDS;
  uint32_t* xchg = nmask + C::MAXWORDS;                     // [2][8][W]
  uint64_t* st_hz = reinterpret_cast<uint64_t*>(xchg + 2 * 8 * W + 2);  // 8-aligned (W*16 even)
  uint32_t* st_pos = reinterpret_cast<uint32_t*>(st_hz + POS);
  uint16_t* st_e = reinterpret_cast<uint16_t*>(st_pos + POS);
  uint64_t* H64 = st_hz;  // slow path alias (POS entries)
  __shared__ X2Shared sh;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // ---- tile id (dynamic, in launch order -> look-back safe) and job range
  if (tid == 0) {
    const uint32_t t = atomicAdd(a.tile_ctr, 1u);
    sh.tile = t;
    const int64_t b_first = (int64_t)t * X2_OUT_BLOCKS - 1;
    const int64_t b_last = (int64_t)t * X2_OUT_BLOCKS + X2_NT - 2;
    const uint64_t gfirst = b_first < 0 ? 0 : (uint64_t)b_first * W;
    uint64_t glast = (uint64_t)(b_last < 0 ? 0 : b_last) * W;
    const uint64_t gmax = a.total_blocks * W - 1;
    if (glast > gmax) glast = gmax;
    sh.j0 = find_job_le(a.kb, 0, a.n_jobs - 1, gfirst);
    sh.j1 = find_job_le(a.kb, sh.j0, a.n_jobs - 1, glast);
    sh.any_n = 0; sh.slow = 0; sh.tie = 0;
  }
  // expected-letter table: for 4 MSB-first codes pk, bytes "ACGT"[c_i], base 0 in byte 0
  {
    const uint32_t pk = tid;
    const uint32_t L4 = 0x54474341u;  // 'A','C','G','T'
    uint32_t e = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const uint32_t c = (pk >> (6 - 2 * i)) & 3u;
      e |= ((L4 >> (8 * c)) & 0xFFu) << (8 * i);
    }
    lut[tid] = e;
  }
  __syncthreads();
  const uint32_t tile = sh.tile;
  const uint32_t j0 = sh.j0, j1 = sh.j1;

  // ---- my block
  const int64_t myb = (int64_t)tile * X2_OUT_BLOCKS - 1 + tid;
  const bool blk_in = myb >= 0 && (uint64_t)myb < a.total_blocks;
  uint32_t J = j0;
  uint64_t l0 = 0;
  uint32_t nk = 0;
  if (blk_in) {
    const uint64_t g = (uint64_t)myb * W;
    J = find_job_le(a.kb, j0, j1, g);
    l0 = g - a.kb[J];
    nk = a.jobs[J].nk;
  }
  // tile code-word range (from the first and last blocks' jobs)
  if (tid == 0) {
    uint64_t lo;
    const int64_t bf = (int64_t)tile * X2_OUT_BLOCKS - 1;
    if (bf < 0) lo = a.cw[0];
    else {
      const uint64_t g = (uint64_t)bf * W;
      lo = a.cw[j0] + (g - a.kb[j0]) / 16;
    }
    sh.cw_lo = lo;
    // end: the last block's window, within its job
    const int64_t bl = (int64_t)tile * X2_OUT_BLOCKS + X2_NT - 2;
    uint64_t gl = (uint64_t)(bl < 0 ? 0 : bl) * W;
    const uint64_t gmax = a.total_blocks * W - 1;
    if (gl > gmax) gl = gmax;
    const uint64_t ll = gl - a.kb[j1];
    uint64_t hi = a.cw[j1] + (ll + NB + 15) / 16 + 1;
    if (hi > a.cw[j1 + 1]) hi = a.cw[j1 + 1];
    sh.cw_hi = hi < lo ? lo : hi;
  }
  __syncthreads();
  const uint64_t cw_lo = sh.cw_lo;
  uint64_t cw_hi = sh.cw_hi;
  if (cw_hi > cw_lo + C::MAXWORDS) cw_hi = cw_lo + C::MAXWORDS;  // cannot happen for 256 blocks; guard
  const int nwords = (int)(cw_hi - cw_lo);

  // ---------------------------------------------------------------- A. sparsify into SMEM
  {
    uint32_t my_n = 0;
    uint32_t Jw = j0;
    for (int wi = tid; wi < nwords; wi += X2_NT) {
      uint32_t word = 0, nm = 0;
      {
        const uint64_t gw = cw_lo + wi;
        Jw = find_job_le(a.cw, Jw, j1, gw);
        while (Jw < j1 && a.cw[Jw + 1] <= gw) ++Jw;
        const Job jb = a.jobs[Jw];
        const uint64_t ncode = jb.nk ? (uint64_t)jb.nk + K - 1 : 0;
        const uint64_t q0 = (gw - a.cw[Jw]) * 16;
        if (q0 < ncode) {
          const int nb = (int)min((uint64_t)16, ncode - q0);
          const uint64_t A = jb.seq_off + jb.phase + a.one0 + (uint64_t)PS * q0;
          const uint64_t Aa = A & ~3ull;
          const uint32_t d8 = (uint32_t)(A - Aa) * 8;
          constexpr int NL = 4 * PS + 1;
          uint32_t w[NL];
#pragma unroll
          for (int i = 0; i < NL; i++) {
            const uint64_t ad = Aa + 4ull * i;
            w[i] = ad + 4 <= a.seq_bytes ? __ldg(reinterpret_cast<const uint32_t*>(a.seq + ad))
                                         : 0u;
            if (ad + 4 > a.seq_bytes && ad < a.seq_bytes) {  // ragged tail of the buffer
              uint32_t v = 0;
              for (uint64_t q = ad; q < a.seq_bytes; q++) v |= (uint32_t)a.seq[q] << (8 * (q - ad));
              w[i] = v;
            }
          }
          uint32_t t4[4];
#pragma unroll
          for (int g = 0; g < 4; g++) {
            uint32_t x;
            if constexpr (PS == 1) {
              x = __funnelshift_r(w[g], w[g + 1], d8);
            } else {
              const uint32_t lo = __funnelshift_r(w[2 * g], w[2 * g + 1], d8);
              const uint32_t hi = __funnelshift_r(w[2 * g + 1], w[2 * g + 2], d8);
              x = __byte_perm(lo, hi, 0x6420);
            }
            const uint32_t c = ((x >> 1) ^ (x >> 2)) & 0x03030303u;
            const uint32_t t = c * 0x40100401u;  // top byte = the 4 codes, MSB-first
            uint32_t bad = (x & 0xDFDFDFDFu) ^ lut[t >> 24];
            const int valid_here = nb - 4 * g;  // bases of this group that exist
            if (valid_here < 4) bad = valid_here <= 0 ? 0u : (bad & (0xFFFFFFFFu >> (8 * (4 - valid_here))));
            if (bad) {
#pragma unroll
              for (int i = 0; i < 4; i++)
                if ((bad >> (8 * i)) & 0xFFu) nm |= 1u << (15 - (4 * g + i));
            }
            t4[g] = t;
          }
          const uint32_t u = __byte_perm(t4[1], t4[0], 0x7300);
          const uint32_t v = __byte_perm(t4[3], t4[2], 0x0073);
          word = __byte_perm(u, v, 0x3254);
          if (nb < 16) word &= 0xFFFFFFFFu << (32 - 2 * nb);
        }
      }
      codes[wi] = word;
      nmask[wi] = nm;
      my_n |= nm;
    }
    if (__syncthreads_or(my_n != 0)) {
      if (tid == 0) sh.any_n = 1;
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- B. k-mers and hashes
  const bool blk_has_kmers = blk_in && l0 < nk;
  uint32_t win[NWIN];
  {
    const uint64_t gwb = a.cw[J] + l0 / 16;
    const int wbase = (int)(gwb - cw_lo);
    const uint32_t off = (uint32_t)(l0 % 16) * 2;
    uint32_t raw[NLOAD + 1];
#pragma unroll
    for (int i = 0; i <= NLOAD; i++) {
      const int idx = wbase + i;
      raw[i] = (blk_has_kmers && idx >= 0 && idx < C::MAXWORDS) ? codes[idx] : 0u;
    }
#pragma unroll
    for (int i = 0; i < NWIN; i++) win[i] = __funnelshift_l(raw[i + 1], raw[i], off);
  }
  uint32_t rcw[NWIN];
#pragma unroll
  for (int i = 0; i < NWIN; i++) rcw[i] = ~rev2(win[NWIN - 1 - i]);
  constexpr int PADB = 32 * NWIN - 2 * NB;

  uint64_t hz[W];     // hash | strand << 63
  uint32_t key[W];
  uint32_t palmask = 0;
  const uint32_t ks = a.key_shift;
#pragma unroll
  for (int i = 0; i < W; i++) {
    const uint64_t fwd = ext_bits(win, 2 * i, 2 * K);
    const uint64_t rev = ext_bits(rcw, PADB + 2 * (NB - i - K), 2 * K);
    const bool z = fwd > rev;
    const uint64_t h = wang_hash_k<K>(z ? rev : fwd);
    hz[i] = h | ((uint64_t)z << 63);
    uint32_t kk = (uint32_t)(h >> ks) + 1u;
    if constexpr ((K & 1) == 0) {
      if (fwd == rev) { kk = 0xFFFFFFFFu; palmask |= 1u << i; }
    }
    key[i] = (blk_has_kmers && l0 + i < nk) ? kk : 0u;
  }

  // ---------------------------------------------------------------- C. selection on keys
  uint32_t selmask = 0;
  bool need_slow = false;
  if (!sh.any_n) {
    uint32_t PF[W], SF[W];
    PF[0] = key[0];
#pragma unroll
    for (int i = 1; i < W; i++) PF[i] = min(PF[i - 1], key[i]);
    SF[W - 1] = key[W - 1];
#pragma unroll
    for (int i = W - 2; i >= 0; i--) SF[i] = min(SF[i + 1], key[i]);
    // next block's prefix minima
    uint32_t* xpf = xchg;            // [8][W]
    uint32_t* xsf = xchg + 8 * W;    // [8][W]
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < W; i++) xpf[wid * W + i] = PF[i];
    }
    __syncthreads();
    uint32_t nPF[W];
#pragma unroll
    for (int i = 0; i < W; i++) {
      uint32_t v = __shfl_down_sync(0xffffffffu, PF[i], 1);
      if (lane == 31) v = (wid < 7) ? xpf[(wid + 1) * W + i] : 0u;
      nPF[i] = v;
    }
    uint32_t WM[W];
    WM[0] = SF[0];
#pragma unroll
    for (int i = 1; i < W; i++) WM[i] = min(SF[i], nPF[i - 1]);
    uint32_t PX[W], SX[W];
    PX[0] = WM[0];
#pragma unroll
    for (int i = 1; i < W; i++) PX[i] = max(PX[i - 1], WM[i]);
    SX[W - 1] = WM[W - 1];
#pragma unroll
    for (int i = W - 2; i >= 0; i--) SX[i] = max(SX[i + 1], WM[i]);
    if (lane == 31) {
#pragma unroll
      for (int i = 0; i < W; i++) xsf[wid * W + i] = SX[i];
    }
    __syncthreads();
    uint32_t pSX[W];
#pragma unroll
    for (int i = 0; i < W; i++) {
      uint32_t v = __shfl_up_sync(0xffffffffu, SX[i], 1);
      if (lane == 0) v = (wid > 0) ? xsf[(wid - 1) * W + i] : 0u;
      pSX[i] = v;
    }
#pragma unroll
    for (int o = 0; o < W; o++) {
      const uint32_t mm = (o == W - 1) ? PX[W - 1] : max(pSX[o + 1], PX[o]);
      const uint32_t k = key[o];
      bool s = (k == mm) && k != 0u;
      if constexpr ((K & 1) == 0) s = s && k != 0xFFFFFFFFu;
      if (k != 0u && mm == 0u) need_slow = true;  // run shorter than w: partial-window rule
      if (s) selmask |= 1u << o;
    }
    if (tid == 0 || tid == X2_NT - 1) need_slow = false;  // halo blocks are not emitted
  }
  if (__syncthreads_or(need_slow)) {
    if (tid == 0) sh.slow = 1;
  }
  __syncthreads();

  // ---------------------------------------------------------------- D. exact slow path
  auto slow_path = [&]() {
    // 64-bit H (hash+1; 0 barrier; ~0 palindrome) for every position of the tile, exact N handling
#pragma unroll
    for (int i = 0; i < W; i++) {
      uint64_t hv = 0;
      if (blk_has_kmers && l0 + i < nk) {
        const uint64_t q = l0 + i;  // k-mer start (patterned index) in job J
        // N bits for bases q .. q+K-1
        const uint64_t gwq = a.cw[J] + q / 16;
        const int wb = (int)(gwq - cw_lo);
        const uint32_t o = (uint32_t)(q % 16);
        bool anyn = false;
        for (int b = 0; b < K; b++) {
          const int wi2 = wb + (int)((o + b) / 16);
          const uint32_t bit = 15 - ((o + b) % 16);
          if (wi2 >= 0 && wi2 < C::MAXWORDS && ((nmask[wi2] >> bit) & 1u)) anyn = true;
        }
        if (!anyn) hv = ((palmask >> i) & 1u) ? ~0ull : (hz[i] & ~(1ull << 63)) + 1;
      }
      H64[tid * W + i] = hv;
    }
    __syncthreads();
    uint32_t m = 0;
    if (tid > 0 && tid < X2_NT - 1) {
      for (int i = 0; i < W; i++) {
        const int j = tid * W + i;
        const uint64_t hj = H64[j];
        if (hj == 0 || hj == ~0ull) continue;
        int lo = j, hi = j;
        while (lo > j - (W - 1) && H64[lo - 1] != 0) --lo;
        while (hi < j + (W - 1) && H64[hi + 1] != 0) ++hi;
        bool s = false;
        if (hi - lo + 1 < W) {  // the whole run is one partial window
          uint64_t mn = ~0ull;
          for (int q = lo; q <= hi; q++)
            if (H64[q] != ~0ull) mn = min(mn, H64[q]);
          s = (hj == mn);
        } else {
          const int a0 = max(lo, j - (W - 1)), a1 = min(j, hi - (W - 1));
          for (int st = a0; st <= a1 && !s; st++) {
            uint64_t mn = ~0ull;
            for (int q = st; q < st + W; q++)
              if (H64[q] != ~0ull) mn = min(mn, H64[q]);
            s = (hj == mn);
          }
        }
        if (s) m |= 1u << i;
      }
    }
    selmask = m;
    __syncthreads();
  };
  if (sh.any_n || sh.slow) slow_path();
  if (tid == 0 || tid == X2_NT - 1 || !blk_in) selmask = 0;

  // ---------------------------------------------------------------- E. compaction (staged)
  auto stage_records = [&]() -> uint32_t {
    const uint32_t cnt = __popc(selmask);
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane == 31) sh.warp_cnt[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      uint32_t ws = lane < X2_NT / 32 ? sh.warp_cnt[lane] : 0u;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, ws, d);
        if (lane >= d) ws += y;
      }
      if (lane < X2_NT / 32) sh.warp_cnt[lane] = ws;
    }
    __syncthreads();
    uint32_t idx = (wid ? sh.warp_cnt[wid - 1] : 0u) + incl - cnt;
    const uint32_t first = idx;
    const Job jb = a.jobs[J];
#pragma unroll
    for (int i = 0; i < W; i++) {
      if (selmask & (1u << i)) {
        st_hz[idx] = hz[i];
        st_pos[idx] = (uint32_t)(jb.pos_base + jb.phase + a.one0 + (uint64_t)PS * (l0 + i));
        st_e[idx] = (uint16_t)(tid * W + i);
        ++idx;
      }
    }
    return first;
  };
  uint32_t my_first = stage_records();
  __syncthreads();
  uint32_t tile_cnt = sh.warp_cnt[X2_NT / 32 - 1];
  // exactness check of the 31-bit keys: candidates closer than w with equal keys and different hashes
  if (!sh.any_n && !sh.slow && a.key_shift > 0) {
    bool tie = false;
    for (uint32_t r = tid; r < tile_cnt; r += X2_NT) {
      const uint64_t hr = st_hz[r] & ~(1ull << 63);
      const uint32_t kr = (uint32_t)(hr >> ks);
      const int er = st_e[r];
      for (uint32_t q = r + 1; q < tile_cnt; q++) {
        if (st_e[q] - er >= W) break;
        const uint64_t hq = st_hz[q] & ~(1ull << 63);
        if ((uint32_t)(hq >> ks) == kr && hq != hr) tie = true;
      }
    }
    if (__syncthreads_or(tie)) {
      // recompute exactly (the H64 alias overwrites the staging area)
      slow_path();
      if (tid == 0 || tid == X2_NT - 1 || !blk_in) selmask = 0;
      my_first = stage_records();
      __syncthreads();
      tile_cnt = sh.warp_cnt[X2_NT / 32 - 1];
    }
  }
  // tile offset (decoupled look-back in tile order)
  if (tid == 0) {
    const uint64_t base = lb_exclusive(a.status, tile, tile_cnt);
    sh.base = base;
    const uint64_t ntiles = (a.total_blocks + X2_OUT_BLOCKS - 1) / X2_OUT_BLOCKS;
    if (tile == ntiles - 1) *a.total_out = base + tile_cnt;
  }
  __syncthreads();
  const uint64_t base = sh.base;
  if (a.job_off && blk_in && tid > 0 && tid < X2_NT - 1 && l0 == 0) a.job_off[J] = base + my_first;
  for (uint32_t r = tid; r < tile_cnt; r += X2_NT) {
    const uint64_t gi = base + r;
    if (gi < a.cap) {
      a.out_hz[gi] = st_hz[r];
      a.out_pos[gi] = st_pos[r];
    }
  }
  if (a.out_job) {
    // job of each staged record: recover from its tile position (block -> job), rare enough per record
    for (uint32_t r = tid; r < tile_cnt; r += X2_NT) {
      const uint64_t gi = base + r;
      if (gi < a.cap) {
        const int e = st_e[r];
        const uint64_t g = ((uint64_t)tile * X2_OUT_BLOCKS - 1) * W + e;
        a.out_job[gi] = find_job_le(a.kb, j0, j1, g);
      }
    }
  }
}

// padded position bases (multiple of W) and code-word bases per job
__global__ void k_x2_sizes(const Job* __restrict__ jobs, uint32_t n, int K, int W, uint64_t* kb, uint64_t* cw) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint64_t nk = jobs[j].nk;
    kb[j] = (nk + 1 + W - 1) / W * W;
    const uint64_t ncode = nk ? nk + K - 1 : 0;
    cw[j] = (ncode + 15) / 16;
  }
}

template <int K, int W, int PS>
size_t x2_smem_bytes() {
  using C = X2Cfg<K, W, PS>;
  return (size_t)(256 + 2 * C::MAXWORDS + 2 * 8 * W + 2) * 4 + (size_t)C::POS * (8 + 4 + 2) + 16;
}

template <int K, int W, int PS>
void launch_x2(const X2Args& a, uint64_t ntiles, cudaStream_t st, const char* tag) {
  static bool attr = false;
  const size_t smem = x2_smem_bytes<K, W, PS>();
  if (!attr) {
    GOD_CUDA(cudaFuncSetAttribute(k_extract2<K, W, PS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  GOD_LAUNCH(tag, (k_extract2<K, W, PS>), (unsigned)ntiles, X2_NT, smem, st, a);
}

}  // namespace

// Returns false if no specialised kernel exists for these parameters (caller uses the generic one).
bool run_extract2(const Params& P, const uint8_t* seq, uint64_t seq_bytes, const Job* jobs, uint32_t n_jobs,
                  bool want_job, bool want_job_off, Records& rec, cudaStream_t st, Scratch& scr,
                  uint64_t cap_hint, const char* tag) {
  if (P.pat.x != 1 || (P.pat.p != 1 && P.pat.p != 2)) return false;
  const int K = P.k, W = P.w, PS = (int)P.pat.p;
  auto supported = [&](int k, int w) { return K == k && W == w; };
  if (!(supported(21, 11) || supported(19, 19) || supported(15, 10))) return false;
  if (getenv("GOD_DISABLE_X2")) return false;
  rec.n = 0;
  if (n_jobs == 0) return false;
  // padded layouts
  uint64_t* kb = scr.alloc<uint64_t>(n_jobs + 1);
  uint64_t* cw = scr.alloc<uint64_t>(n_jobs + 1);
  uint64_t* tot = scr.alloc<uint64_t>(2);
  GOD_LAUNCH("k_x2_sizes", k_x2_sizes, grid_for(n_jobs, 256), 256, 0, st, jobs, n_jobs, K, W, kb, cw);
  scan_exclusive_u64(kb, kb, n_jobs, tot, st, scr);
  scan_exclusive_u64(cw, cw, n_jobs, tot + 1, st, scr);
  GOD_CUDA(cudaMemcpyAsync(kb + n_jobs, tot, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  GOD_CUDA(cudaMemcpyAsync(cw + n_jobs, tot + 1, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  uint64_t htot[2];
  GOD_CUDA(cudaMemcpyAsync(htot, tot, sizeof(htot), cudaMemcpyDeviceToHost, st));
  GOD_CUDA(cudaStreamSynchronize(st));
  const uint64_t total_pos = htot[0];
  const uint64_t total_blocks = total_pos / W;
  const uint64_t ntiles = (total_blocks + X2_OUT_BLOCKS - 1) / X2_OUT_BLOCKS;
  GOD_REQUIRE(ntiles < 0x7FFFFFFFull, "input too large for one extraction launch");
  uint64_t cap = cap_hint ? cap_hint : total_pos;
  if (cap > total_pos) cap = total_pos;
  if (cap == 0) cap = 1;
  uint64_t* status = scr.alloc<uint64_t>(ntiles);
  uint32_t* ctr = scr.alloc<uint32_t>(1);
  uint64_t* dtotal = scr.alloc<uint64_t>(1);
  if (want_job_off) rec.job_off = scr.alloc<uint64_t>(n_jobs + 1);
  const char* dbg = getenv("GOD_DEBUG_KEYBITS");  // test hook: coarser keys force the exact tie path
  uint32_t key_shift = 2 * K > 31 ? 2 * K - 31 : 0;
  if (dbg) {
    const int kbits = atoi(dbg);
    if (kbits > 0 && kbits < 2 * K) key_shift = 2 * K - kbits;
  }
  for (int attempt = 0; attempt < 2; attempt++) {
    rec.cap = cap;
    rec.hz = scr.alloc<uint64_t>(cap);
    rec.pos = scr.alloc<uint32_t>(cap);
    rec.job = want_job ? scr.alloc<uint32_t>(cap) : nullptr;
    GOD_CUDA(cudaMemsetAsync(status, 0, ntiles * sizeof(uint64_t), st));
    GOD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
    X2Args a{seq, seq_bytes, jobs, kb, cw, n_jobs, total_blocks, P.pat.one[0], key_shift, status, ctr,
             rec.hz, rec.pos, rec.job, rec.job_off, cap, dtotal};
    if (ntiles) {
      if (K == 21 && W == 11) {
        if (PS == 2) launch_x2<21, 11, 2>(a, ntiles, st, tag);
        else launch_x2<21, 11, 1>(a, ntiles, st, tag);
      } else if (K == 19 && W == 19) {
        if (PS == 2) launch_x2<19, 19, 2>(a, ntiles, st, tag);
        else launch_x2<19, 19, 1>(a, ntiles, st, tag);
      } else {
        if (PS == 2) launch_x2<15, 10, 2>(a, ntiles, st, tag);
        else launch_x2<15, 10, 1>(a, ntiles, st, tag);
      }
    } else {
      GOD_CUDA(cudaMemsetAsync(dtotal, 0, sizeof(uint64_t), st));
    }
    const uint64_t n = d2h_scalar(dtotal, st);
    if (n <= cap) {
      rec.n = n;
      if (want_job_off)
        GOD_CUDA(cudaMemcpyAsync(rec.job_off + n_jobs, dtotal, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
      return true;
    }
    cap = n;
  }
  GOD_REQUIRE(false, "extraction capacity retry failed");
  return true;
}

}  // namespace god
