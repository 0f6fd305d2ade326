// extract2.cu — K1 v2: register-resident fused sparsify + minimizer extraction (stages 1+2).
//
// Same definitions as extract.cu (P:282/P:286/P:294/P:300/P:370; readings O1-O6 of DESIGN.md §2),
// specialised at compile time for the hot configurations: k, w and patterns with exactly one '1' of
// period <= 3 ("1", "10"/"01", "100"/"010"/"001") or whose x ones come first ("110", "1110").  Everything else
// runs the generic kernel (extract.cu).
//
// Layout.  Each job's k-mer starts are padded to a multiple of W positions (the pad slots are
// window barriers), so a W-block never straddles two jobs; each job's patterned bases are packed
// 16 per u32 word, MSB-first, starting on a fresh word.  A tile of X2_NT = 128 threads owns 128
// W-blocks (thread t = block t); blocks 0 and 127 are halo (computed, not emitted), so consecutive
// tiles overlap by two blocks.  CTAs are persistent (occupancy x SMs) and take tiles in order.
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
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include "internal.cuh"

namespace god {

namespace {

constexpr int X2_NT = 128;
constexpr int X2_OUT_BLOCKS = X2_NT - 2;
// Staging capacity (selected records per tile) of the deferred copy-out.  Minimizer density is
// ~2/(w+1), i.e. ~17% of a tile's positions; a tile with more (all-ties runs: homopolymers, tandem
// repeats) is written out at once instead, after a synchronous look-back.
constexpr int X2_CAP = 384;
constexpr uint32_t X2_FLUSHED = 0xFFFFFFFFu;  // pending-count marker: the tile was written out already
// resident CTAs per SM the register allocation is sized for (SMEM allows 7): 7 for w <= 11 (72
// registers, no spills), 6 for w = 19 (more registers per W-block)
template <int W>
constexpr int x2_minb() { return W >= 16 ? 6 : 7; }

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
  uint32_t dbg_flags;      // developer toggles (GOD_X2_DBG): 1 = unordered output, 2 = no tie check
  uint32_t* dbg_counts;    // [0] tiles on the slow path, [1] tiles with a key tie
  const struct X2Desc* desc;  // [ntiles] per-tile descriptors (k_x2_tile_desc)
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

// The masked Wang hash (O5).  The shift-add steps are written as the equal multiplications
// (~x + (x << 21) = x (2^21 - 1) - 1 and x + (x << 31) = x (2^31 + 1) mod 2^64), which the compiler
// issues on the FMA pipe (IMAD) instead of the integer ALU pipe that the rest of K1 saturates.
template <int K>
__device__ __forceinline__ uint64_t wang_hash_k(uint64_t key) {
  constexpr uint64_t mask = (K >= 32) ? ~0ull : ((1ull << (2 * K)) - 1);
  key = (key * ((1ull << 21) - 1) - 1ull) & mask;
  key = key ^ (key >> 24);
  key = (key * 265ull) & mask;
  key = key ^ (key >> 14);
  key = (key * 21ull) & mask;
  key = key ^ (key >> 28);
  key = (key * ((1ull << 31) + 1)) & mask;
  return key;
}

// per-tile descriptor, precomputed by k_x2_tile_desc so that a CTA never walks a dependent chain
// of global loads (tile -> jobs -> code-word range) while its other warps wait at a barrier
struct __align__(16) X2Desc {
  uint32_t j0, j1, simple, safe;  // safe: every byte the tile may read is inside the buffer
  uint64_t cw_lo, cw_hi;
};

struct X2Tile {  // per-tile scalars, in SMEM
  uint32_t tile, j0, j1, simple, safe, any_n, slow, cnt;
  uint64_t cw_lo, cw_hi;
};

template <int K, int W, int PP, int PX>
struct X2Cfg {
  static_assert(X2_NT * W < 4096, "staged record index must fit 12 bits (block info packing)");
  static constexpr int NB = W + K - 1;                 // bases in a thread's window
  static constexpr int NWIN = (2 * NB + 31) / 32;       // aligned window words
  static constexpr int NLOAD = (30 + 2 * NB + 31) / 32; // words loaded before alignment
  static constexpr int POS = X2_NT * W;                 // positions per tile (incl. the two halo blocks)
  static constexpr int MAXWORDS = (POS + X2_NT * (K - 1) + 15) / 16 + X2_NT + 8;
  // SMEM layout (bytes)
  static constexpr size_t O_LUT = 0;
  static constexpr size_t O_CODES = O_LUT + 256 * 4;
  static constexpr size_t O_NMASK = O_CODES + (size_t)MAXWORDS * 4;
  static constexpr size_t O_XCHG = O_NMASK + (size_t)MAXWORDS * 4;
  static constexpr size_t O_HZ = (O_XCHG + 2 * (X2_NT / 32) * W * 4 + 15) / 16 * 16;  // [POS] hz, this tile
  static constexpr size_t O_SHZ = O_HZ + (size_t)POS * 8;         // [2][X2_CAP] staged hz of the selected
  static constexpr size_t O_SE = O_SHZ + 2 * (size_t)X2_CAP * 8;  // [2][X2_CAP] staged: e | key16 << 16
  static constexpr size_t O_BI = O_SE + 2 * (size_t)X2_CAP * 4;   // block info [2][2][NT]
  static constexpr size_t SMEM = (O_BI + 2 * 2 * X2_NT * 4 + 15) / 16 * 16;
};

// (pack16 gathers the included bytes with compile-time byte-permutations)
// *nm gets the N bits (bit 15 - b for base b).  nb = bases that exist (<= 16).
// Pattern geometry: period PP with ones at offsets 0..PX-1 (x = 1 patterns may be rotated: their
// single one's offset is added to the job base).  Included base q of a job lies at byte offset
// (q / PX) * PP + q % PX.
__host__ __device__ constexpr int pat_off(int PP, int PX, int q) { return (q / PX) * PP + q % PX; }
// byte offset, relative to base q0 (q0 % PX == R0), of base q0 + b
__host__ __device__ constexpr int pat_rel(int PP, int PX, int R0, int b) {
  return pat_off(PP, PX, R0 + b) - pat_off(PP, PX, R0);
}
template <int PP, int PX>
constexpr int pack_words() {  // u32 words loaded per 16 bases (incl. the alignment shift)
  int mx = 0;
  for (int r = 0; r < PX; r++) mx = pat_rel(PP, PX, r, 15) > mx ? pat_rel(PP, PX, r, 15) : mx;
  return (mx + 3) / 4 + 2;
}
// selector of __byte_perm gathering bases 4g..4g+3 from aligned words (a, a+1), a = rel(4g) / 4
template <int PP, int PX, int R0, int G>
constexpr uint32_t pack_sel() {
  const int a4 = (pat_rel(PP, PX, R0, 4 * G) / 4) * 4;
  uint32_t sel = 0;
  for (int i = 0; i < 4; i++) sel |= (uint32_t)(pat_rel(PP, PX, R0, 4 * G + i) - a4) << (4 * i);
  return sel;
}
// byte offset of base 4G + i relative to the aligned start of base 4G (period 3: 0, 3, 6, 9)
template <int PP, int PX, int R0, int G>
constexpr int pack_off(int i) {
  return pat_rel(PP, PX, R0, 4 * G + i) - (pat_rel(PP, PX, R0, 4 * G) / 4) * 4;
}

// 16 patterned bases (MSB-first 2-bit codes) from the ASCII bytes, base 0 at byte A (its job-relative
// index has residue R0 mod PX); *nm gets the N bits (bit 15 - b for base b).  nb = bases that exist.
template <int PP, int PX, int R0, bool CHECKED>
__device__ __forceinline__ uint32_t pack16(const uint8_t* seq, uint64_t seq_bytes, uint64_t A, int nb,
                                           const uint32_t* lut, uint32_t* nm) {
  // words aligned in the ADDRESS space (the caller's buffer may start anywhere, e.g. a tensor slice);
  // the first word may begin up to 3 bytes before byte A (inside the allocation: allocations are
  // aligned), and the tile descriptor's end margin covers the last one
  const uintptr_t pA = reinterpret_cast<uintptr_t>(seq + A);
  const uintptr_t pa = pA & ~(uintptr_t)3;
  const uint32_t d8 = (uint32_t)(pA - pa) * 8;
  constexpr int NL = pack_words<PP, PX>();
  uint32_t w[NL];
  const uint32_t* src = reinterpret_cast<const uint32_t*>(pa);
#pragma unroll
  for (int i = 0; i < NL; i++) {
    if constexpr (CHECKED) {
      const int64_t ad = (int64_t)(pa - reinterpret_cast<uintptr_t>(seq)) + 4ll * i;  // relative to seq
      uint32_t v = 0;
      if (ad >= 0 && (uint64_t)ad + 4 <= seq_bytes) v = __ldg(src + i);
      else
        for (int64_t q = ad < 0 ? 0 : ad; q < ad + 4 && (uint64_t)q < seq_bytes; q++)
          v |= (uint32_t)seq[q] << (8 * (q - ad));
      w[i] = v;
    } else {
      w[i] = __ldg(src + i);
    }
  }
  uint32_t t4[4];
  uint32_t bad_any = 0, badw[4];
  auto gather = [&](auto gc) -> uint32_t {
    constexpr int G = decltype(gc)::value;
    constexpr int a = pat_rel(PP, PX, R0, 4 * G) / 4;
    constexpr uint32_t sel = pack_sel<PP, PX, R0, G>();
    const uint32_t lo = __funnelshift_r(w[a], w[a + 1], d8);
    if constexpr (sel == 0x3210u) return lo;  // four consecutive bytes
    const uint32_t hi = __funnelshift_r(w[a + 1], w[a + 2], d8);
    if constexpr (pack_off<PP, PX, R0, G>(3) < 8) {
      return __byte_perm(lo, hi, sel);
    } else {  // period 3: bases at 0, 3, 6 from (lo, hi), the fourth (offset 8..11) from the next word
      static_assert(pack_off<PP, PX, R0, G>(2) < 8 && pack_off<PP, PX, R0, G>(3) < 12, "byte gather span");
      const uint32_t hi2 = __funnelshift_r(w[a + 2], w[a + 3], d8);
      const uint32_t t = __byte_perm(lo, hi, sel & 0x0FFFu);
      return __byte_perm(t, hi2, 0x0210u | ((uint32_t)(4 + pack_off<PP, PX, R0, G>(3) - 8) << 12));
    }
  };
  const uint32_t xs[4] = {gather(std::integral_constant<int, 0>()), gather(std::integral_constant<int, 1>()),
                          gather(std::integral_constant<int, 2>()), gather(std::integral_constant<int, 3>())};
#pragma unroll
  for (int g = 0; g < 4; g++) {
    const uint32_t x = xs[g];
    const uint32_t c = ((x >> 1) ^ (x >> 2)) & 0x03030303u;  // A0 C1 G2 T3 (either case)
    const uint32_t t = c * 0x40100401u;                       // top byte = the 4 codes, MSB-first
    badw[g] = (x & 0xDFDFDFDFu) ^ lut[t >> 24];              // nonzero byte <=> not A/C/G/T
    bad_any |= badw[g];
    t4[g] = t;
  }
  uint32_t word = __byte_perm(__byte_perm(t4[1], t4[0], 0x7300), __byte_perm(t4[3], t4[2], 0x0073), 0x3254);
  if (nb < 16) word &= 0xFFFFFFFFu << (32 - 2 * nb);
  uint32_t n = 0;
  if (bad_any) {
#pragma unroll
    for (int g = 0; g < 4; g++)
#pragma unroll
      for (int i = 0; i < 4; i++)
        if (((badw[g] >> (8 * i)) & 0xFFu) && 4 * g + i < nb) n |= 1u << (15 - (4 * g + i));
  }
  *nm = n;
  return word;
}

// code word at job-relative base q0 (a multiple of 16) of the job whose base 0 is byte A0
template <int PP, int PX, bool CHECKED>
__device__ __forceinline__ uint32_t pack_word(const uint8_t* seq, uint64_t seq_bytes, uint64_t A0, uint64_t q0, int nb,
                                              const uint32_t* lut, uint32_t* nm) {
  const uint32_t r0 = (uint32_t)(q0 % PX);
  const uint64_t A = A0 + (q0 / PX) * PP + r0;
  if constexpr (PX == 1) {
    return pack16<PP, PX, 0, CHECKED>(seq, seq_bytes, A, nb, lut, nm);
  } else if constexpr (PX == 2) {
    return r0 ? pack16<PP, PX, 1, CHECKED>(seq, seq_bytes, A, nb, lut, nm)
              : pack16<PP, PX, 0, CHECKED>(seq, seq_bytes, A, nb, lut, nm);
  } else {
    static_assert(PX == 3, "patterns with up to 3 leading ones");
    return r0 == 0 ? pack16<PP, PX, 0, CHECKED>(seq, seq_bytes, A, nb, lut, nm)
         : r0 == 1 ? pack16<PP, PX, 1, CHECKED>(seq, seq_bytes, A, nb, lut, nm)
                   : pack16<PP, PX, 2, CHECKED>(seq, seq_bytes, A, nb, lut, nm);
  }
}
// original-coordinate distance from base q to base q + i, with r = q % PX
template <int PP, int PX>
__device__ __forceinline__ uint32_t pat_delta(uint32_t r, uint32_t i) {
  return ((r + i) / PX) * PP + (r + i) % PX - r;
}

// deferred decoupled look-back: publish the aggregate as soon as it is known ...
__device__ __forceinline__ void lb_publish(uint64_t* status, uint64_t tile, uint64_t local) {
  lb_store(&status[tile], (tile == 0 ? LB_INC : LB_AGG) | local);
}
// ... and resolve the exclusive prefix later (whole warp), publishing the inclusive prefix
__device__ inline uint64_t lb_resolve_warp(uint64_t* status, uint64_t tile, uint64_t local) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) return 0;
  uint64_t excl = 0;
  int64_t j = (int64_t)tile - 1 - lane;
  while (true) {
    uint64_t s = j >= 0 ? lb_load(&status[j]) : (LB_INC | 0ull);
    while (__any_sync(0xffffffffu, (s & ~LB_VAL) == 0)) {
      if ((s & ~LB_VAL) == 0) s = lb_load(&status[j]);
    }
    const uint32_t inc = __ballot_sync(0xffffffffu, (s & ~LB_VAL) == LB_INC);
    const int first = inc ? __ffs(inc) - 1 : 32;
    uint64_t v = lane <= first ? (s & LB_VAL) : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc) break;
    j -= 32;
  }
  if (lane == 0) lb_store(&status[tile], LB_INC | (excl + local));
  return excl;
}

// ---------------------------------------------------------------------------------------------
// Persistent CTAs: each grabs tiles in order (atomic counter), computes a tile, publishes its
// record count, and only then resolves the PREVIOUS tile's output offset and writes its records,
// so the look-back never stalls the CTA on a tile that other CTAs are still computing.
template <int K, int W, int PP, int PX>
__global__ void __launch_bounds__(X2_NT, x2_minb<W>()) k_extract2(X2Args a) {
  using C = X2Cfg<K, W, PP, PX>;
  constexpr int NB = C::NB, NWIN = C::NWIN, NLOAD = C::NLOAD, POS = C::POS;
  constexpr int NWARP = X2_NT / 32;
  extern __shared__ __align__(16) unsigned char x2_smem[];
  uint32_t* lut = reinterpret_cast<uint32_t*>(x2_smem + C::O_LUT);
  uint32_t* codes = reinterpret_cast<uint32_t*>(x2_smem + C::O_CODES);
  uint32_t* nmask = reinterpret_cast<uint32_t*>(x2_smem + C::O_NMASK);
  uint32_t* xpf = reinterpret_cast<uint32_t*>(x2_smem + C::O_XCHG);
  uint32_t* xsf = xpf + NWARP * W;
  uint64_t* HZ = reinterpret_cast<uint64_t*>(x2_smem + C::O_HZ);     // [POS]
  uint64_t* SHZ = reinterpret_cast<uint64_t*>(x2_smem + C::O_SHZ);   // [2][X2_CAP]
  uint32_t* SE = reinterpret_cast<uint32_t*>(x2_smem + C::O_SE);     // [2][X2_CAP]
  // block info [2][2][NT]: pos base | first staged record (12 bits) + job start flag << 12 +
  // job - j0 << 13 (8 bits) + first k-mer index mod x << 21
  uint32_t* BI = reinterpret_cast<uint32_t*>(x2_smem + C::O_BI);
  __shared__ uint32_t s_bj0[2];  // j0 of the tile staged in each buffer
  __shared__ uint64_t s_ovf_base;
  __shared__ X2Tile T;
  __shared__ uint64_t skb[X2_NT + 2], scw[X2_NT + 2];
  __shared__ uint64_t sjb[X2_NT + 2];  // per job of the tile: byte address of its first patterned base
  __shared__ uint32_t sjn[X2_NT + 2];  // ... its k-mer count n_k
  __shared__ uint32_t sjp[X2_NT + 2];  // ... its output position base (pos_base + phase + one0)
  __shared__ uint8_t swj[(X2Cfg<K, W, PP, PX>::MAXWORDS + 3) / 4 * 4];  // code word -> job (relative)
  __shared__ uint32_t sjob[X2_NT];
  __shared__ uint32_t warp_cnt[NWARP];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t ntiles = (a.total_blocks + X2_OUT_BLOCKS - 1) / X2_OUT_BLOCKS;
  {  // expected-letter table: for 4 MSB-first codes pk, bytes "ACGT"[c_i], base 0 in byte 0
    const uint32_t L4 = 0x54474341u;
    for (int pk = tid; pk < 256; pk += X2_NT) {
      uint32_t e = 0;
#pragma unroll
      for (int i = 0; i < 4; i++) e |= ((L4 >> (8 * ((pk >> (6 - 2 * i)) & 3u))) & 0xFFu) << (8 * i);
      lut[pk] = e;
    }
  }
  const uint32_t ks = a.key_shift;
  int buf = 0;

  // write the staged records of a finished tile: warp 0 alone resolves its output offset (decoupled
  // look-back) and copies the records out, overlapped with the other warps' sparsify of the next tile
  auto flush_warp0 = [&](uint64_t tile, uint32_t cnt, int b) {
    uint64_t base;
    if (a.dbg_flags & 1u) base = lane == 0 ? atomicAdd((unsigned long long*)&a.status[ntiles], (unsigned long long)cnt) : 0;
    else base = lb_resolve_warp(a.status, tile, cnt);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (lane == 0 && tile == ntiles - 1) *a.total_out = base + cnt;
    const uint64_t* hzb = SHZ + (size_t)b * X2_CAP;
    const uint32_t* se = SE + (size_t)b * X2_CAP;
    const uint32_t* bpb = BI + (size_t)b * 2 * X2_NT;
    const uint32_t* binf = bpb + X2_NT;
    const uint32_t bj0 = s_bj0[b];
    if (a.job_off)
      for (int t = lane; t < X2_NT; t += 32) {
        const uint32_t f = binf[t];
        if ((f >> 12) & 1u) a.job_off[bj0 + ((f >> 13) & 0xFFu)] = base + (f & 0xFFFu);
      }
    for (uint32_t r = lane; r < cnt; r += 32) {
      const uint64_t gi = base + r;
      if (gi < a.cap) {
        const int e = se[r] & 0xFFFFu;
        const int blk = e / W;
        a.out_hz[gi] = hzb[r];
        a.out_pos[gi] = bpb[blk] + pat_delta<PP, PX>((binf[blk] >> 21) & 3u, (uint32_t)(e - blk * W));
        if (a.out_job) a.out_job[gi] = bj0 + ((binf[blk] >> 13) & 0xFFu);
      }
    }
  };

  // Warp roles per iteration (tile u): warps 1..3 claim the tile (thread SETUP_TID claims tiles in
  // order from an atomic counter, one ahead, with the descriptor prefetched), load its job bases
  // and sparsify it into SMEM (A), synchronising among themselves with named barrier 1; meanwhile
  // warp 0 finishes tile u-2 (look-back + copy-out from the staging buffer that tile u will reuse).
  // Then all four warps compute (B-E) and tile u's count is published.
  constexpr int SETUP_TID = 32;
  uint32_t next_t = 0;
  X2Desc nd{};
  if (tid == SETUP_TID) {
    next_t = atomicAdd(a.tile_ctr, 1u);
    if (next_t < ntiles) nd = a.desc[next_t];
  }
  int64_t pend_old = -1, pend_new = -1;
  uint32_t cnt_old = 0, cnt_new = 0;
  while (true) {
    if (wid == 0) {
      if (pend_old >= 0 && cnt_old != X2_FLUSHED) flush_warp0((uint64_t)pend_old, cnt_old, buf);
    } else {
      if (tid == SETUP_TID) {
        T.tile = next_t < ntiles ? next_t : 0xFFFFFFFFu;
        if (next_t < ntiles) {
          T.j0 = nd.j0; T.j1 = nd.j1;
          T.cw_lo = nd.cw_lo; T.cw_hi = nd.cw_hi;
          T.simple = nd.simple;
          T.safe = nd.safe;
          T.any_n = 0; T.slow = 0;
          next_t = atomicAdd(a.tile_ctr, 1u);
          if (next_t < ntiles) nd = a.desc[next_t];
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(X2_NT - 32) : "memory");
      if (T.tile != 0xFFFFFFFFu) {
        const uint32_t j0 = T.j0, nj = T.j1 - T.j0 + 1;
        const uint64_t cw_lo = T.cw_lo;
        const int nwords = (int)(T.cw_hi - cw_lo);
        const int t1 = tid - 32, nt1 = X2_NT - 32;
        // the tile's job bases in SMEM (a tile spans <= NT + 1 jobs: every job owns >= 1 block)
        for (uint32_t q = t1; q <= nj; q += nt1) {
          skb[q] = a.kb[j0 + q];
          scw[q] = a.cw[j0 + q];
          if (q < nj) {
            const Job jq = a.jobs[j0 + q];
            sjb[q] = jq.seq_off + jq.phase + a.one0;
            sjn[q] = jq.nk;
            sjp[q] = (uint32_t)(jq.pos_base + jq.phase + a.one0);
          }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(X2_NT - 32) : "memory");
        if (!T.simple) {  // code word -> job, filled job by job
          for (uint32_t q = t1; q < nj; q += nt1) {
            const int64_t w0 = (int64_t)scw[q] - (int64_t)cw_lo, w1 = (int64_t)scw[q + 1] - (int64_t)cw_lo;
            for (int64_t wi = w0 < 0 ? 0 : w0; wi < w1 && wi < nwords; wi++) swj[wi] = (uint8_t)q;
          }
          asm volatile("bar.sync 1, %0;" ::"r"(X2_NT - 32) : "memory");
        }
        // ---------------------------------------------------------- A. sparsify into SMEM
        uint32_t my_n = 0;
        if (T.simple) {
          const Job jb = a.jobs[j0];
          const uint64_t w0 = cw_lo - scw[0];
          const uint32_t ncode = jb.nk ? jb.nk + K - 1 : 0;
          const uint64_t A0 = jb.seq_off + jb.phase + a.one0;
          for (int wi = t1; wi < nwords; wi += nt1) {
            const uint64_t q0 = (w0 + wi) * 16;
            uint32_t nm = 0, word = 0;
            if (q0 < ncode) word = pack_word<PP, PX, false>(a.seq, a.seq_bytes, A0, q0,
                                                            (int)min((uint64_t)16, ncode - q0), lut, &nm);
            codes[wi] = word;
            nmask[wi] = nm;
            my_n |= nm;
          }
        } else {
          const bool safe = T.safe;
          for (int wi = t1; wi < nwords; wi += nt1) {
            const uint32_t Jw = swj[wi];
            const uint64_t nkq = sjn[Jw];
            const uint64_t ncode = nkq ? nkq + K - 1 : 0;
            const uint64_t q0 = (cw_lo + wi - scw[Jw]) * 16;
            uint32_t nm = 0, word = 0;
            if (q0 < ncode) {
              const int nb = (int)min((uint64_t)16, ncode - q0);
              word = safe ? pack_word<PP, PX, false>(a.seq, a.seq_bytes, sjb[Jw], q0, nb, lut, &nm)
                          : pack_word<PP, PX, true>(a.seq, a.seq_bytes, sjb[Jw], q0, nb, lut, &nm);
            }
            codes[wi] = word;
            nmask[wi] = nm;
            my_n |= nm;
          }
        }
        if (my_n) T.any_n = 1;
      }
    }
    __syncthreads();
    const uint32_t tile = T.tile;
    if (tile == 0xFFFFFFFFu) break;
    const uint32_t j0 = T.j0, j1 = T.j1;
    const uint64_t cw_lo = T.cw_lo;
    const uint32_t nj = j1 - j0 + 1;

    // ---- my block: job J, first k-mer index l0
    const int64_t myb = (int64_t)tile * X2_OUT_BLOCKS - 1 + tid;
    const bool blk_in = myb >= 0 && (uint64_t)myb < a.total_blocks;
    uint32_t J = j0, l0 = 0, nk = 0;
    if (blk_in) {
      const uint64_t g = (uint64_t)myb * W;
      J = (j0 == j1) ? j0 : j0 + find_job_le(skb, 0, nj - 1, g);
      l0 = (uint32_t)(g - skb[J - j0]);
      nk = sjn[J - j0];
    }
    sjob[tid] = blk_in ? J : 0xFFFFFFFFu;  // block -> job (job boundaries are window barriers)
    __syncthreads();

    // ------------------------------------------------------------ B. k-mers and hashes
    const bool blk_has_kmers = blk_in && l0 < nk;
    uint32_t win[NWIN];
    {
      const int wbase = (int)(scw[J - j0] + l0 / 16 - cw_lo);
      const uint32_t off = (l0 % 16) * 2;
      uint32_t raw[NLOAD + 1];
#pragma unroll
      for (int i = 0; i <= NLOAD; i++) {
        const int idx = wbase + i;
        raw[i] = (blk_has_kmers && idx < C::MAXWORDS) ? codes[idx] : 0u;
      }
#pragma unroll
      for (int i = 0; i < NWIN; i++) win[i] = __funnelshift_l(raw[i + 1], raw[i], off);
    }
    uint32_t rcw[NWIN];
#pragma unroll
    for (int i = 0; i < NWIN; i++) rcw[i] = ~rev2(win[NWIN - 1 - i]);
    constexpr int PADB = 32 * NWIN - 2 * NB;
    uint32_t key[W];
    uint32_t palmask = 0;
    const uint32_t nvalid = blk_has_kmers ? min((uint32_t)W, nk - l0) : 0u;
    // the first k-mer of the block is extracted, the others rolled: fwd gains the entering base
    // as its least significant digit, rev its complement as the most significant (O4)
    constexpr uint64_t KMASK = (K >= 32) ? ~0ull : ((1ull << (2 * K)) - 1);
    uint64_t fwd = ext_bits(win, 0, 2 * K);
    uint64_t rev = ext_bits(rcw, PADB + 2 * (NB - K), 2 * K);
#pragma unroll
    for (int i = 0; i < W; i++) {
      if (i > 0) {
        const uint64_t c = ext_bits(win, 2 * (i + K - 1), 2);
        fwd = ((fwd << 2) | c) & KMASK;
        rev = (rev >> 2) | ((c ^ 3ull) << (2 * K - 2));
      }
      const bool z = fwd > rev;
      const uint64_t h = wang_hash_k<K>(z ? rev : fwd);
      HZ[tid * W + i] = h | ((uint64_t)z << 63);
      uint32_t kk = (uint32_t)(h >> ks) + 1u;
      if constexpr ((K & 1) == 0) {
        if (fwd == rev) { kk = 0xFFFFFFFFu; palmask |= 1u << i; }
      }
      key[i] = (uint32_t)i < nvalid ? kk : 0u;
    }

    // ------------------------------------------------------------ C. selection on keys
    uint32_t selmask = 0;
    if (!T.any_n) {
      bool need_slow = false;
      uint32_t PF[W], SF[W];
      PF[0] = key[0];
#pragma unroll
      for (int i = 1; i < W; i++) PF[i] = min(PF[i - 1], key[i]);
      SF[W - 1] = key[W - 1];
#pragma unroll
      for (int i = W - 2; i >= 0; i--) SF[i] = min(SF[i + 1], key[i]);
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < W; i++) xpf[wid * W + i] = PF[i];
      }
      __syncthreads();
      uint32_t nPF[W];
#pragma unroll
      for (int i = 0; i < W; i++) nPF[i] = __shfl_down_sync(0xffffffffu, PF[i], 1);
      if (lane == 31) {
#pragma unroll
        for (int i = 0; i < W; i++) nPF[i] = (wid < NWARP - 1) ? xpf[(wid + 1) * W + i] : 0u;
      }
      // the next block starting another job: no window crosses into it (a job boundary is a barrier)
      if (tid + 1 < X2_NT && sjob[tid + 1] != J) {
#pragma unroll
        for (int i = 0; i < W; i++) nPF[i] = 0u;
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
      for (int i = 0; i < W; i++) pSX[i] = __shfl_up_sync(0xffffffffu, SX[i], 1);
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < W; i++) pSX[i] = (wid > 0) ? xsf[(wid - 1) * W + i] : 0u;
      }
#pragma unroll
      for (int o = 0; o < W; o++) {
        const uint32_t mm = (o == W - 1) ? PX[W - 1] : max(pSX[o + 1], PX[o]);
        const uint32_t k = key[o];
        bool s = (k == mm) && k != 0u;
        if constexpr ((K & 1) == 0) s = s && k != 0xFFFFFFFFu;
        need_slow |= (k != 0u) & (mm == 0u);  // a run shorter than w: partial-window rule
        if (s) selmask |= 1u << o;
      }
      if (tid == 0 || tid == X2_NT - 1) need_slow = false;  // halo blocks are not emitted
      if (__syncthreads_or(need_slow) && tid == 0) T.slow = 1;
    }
    __syncthreads();

    // ------------------------------------------------------------ D. exact slow path (whole tile)
    auto slow_path = [&]() {
      uint32_t zmask = 0;
#pragma unroll
      for (int i = 0; i < W; i++) zmask |= (uint32_t)(HZ[tid * W + i] >> 63) << i;
      uint64_t* H64 = HZ;  // hash+1, 0 barrier, ~0 palindrome
#pragma unroll
      for (int i = 0; i < W; i++) {
        uint64_t hv = 0;
        if ((uint32_t)i < nvalid) {
          const uint32_t q = l0 + i;
          const int wb = (int)(scw[J - j0] + q / 16 - cw_lo);
          const uint32_t o = q % 16;
          bool anyn = false;
          for (int bb = 0; bb < K; bb++) {
            const int wi2 = wb + (int)((o + bb) / 16);
            if (wi2 < C::MAXWORDS && ((nmask[wi2] >> (15 - ((o + bb) % 16))) & 1u)) anyn = true;
          }
          if (!anyn) hv = ((palmask >> i) & 1u) ? ~0ull : (HZ[tid * W + i] & ~(1ull << 63)) + 1;
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
          while (lo > j - (W - 1) && H64[lo - 1] != 0 && sjob[(lo - 1) / W] == J) --lo;
          while (hi < j + (W - 1) && H64[hi + 1] != 0 && sjob[(hi + 1) / W] == J) ++hi;
          bool s = false;
          if (hi - lo + 1 < W) {
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
      __syncthreads();
#pragma unroll
      for (int i = 0; i < W; i++)  // back to hash | strand (only selected entries matter)
        HZ[tid * W + i] = (H64[tid * W + i] - 1) | ((uint64_t)((zmask >> i) & 1u) << 63);
      selmask = m;
    };
    if (T.any_n || T.slow) {
      if (tid == 0 && a.dbg_counts) atomicAdd(&a.dbg_counts[0], 1u);
      slow_path();
    }
    if (tid == 0 || tid == X2_NT - 1 || !blk_in) selmask = 0;

    // ------------------------------------------------------------ E. compaction into staging[buf]
    uint32_t* se = SE + (size_t)buf * X2_CAP;
    uint64_t* shz = SHZ + (size_t)buf * X2_CAP;
    uint32_t* bi = BI + (size_t)buf * 2 * X2_NT;
    uint32_t my_idx0 = 0;
    auto compact = [&]() -> uint32_t {
      const uint32_t cnt = __popc(selmask);
      uint32_t incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
      }
      if (lane == 31) warp_cnt[wid] = incl;
      __syncthreads();
      uint32_t before = 0, total = 0;
#pragma unroll
      for (int q = 0; q < NWARP; q++) {
        const uint32_t c = warp_cnt[q];
        before += q < wid ? c : 0u;
        total += c;
      }
      uint32_t idx = before + incl - cnt;
      my_idx0 = idx;
      bi[tid] = sjp[J - j0] + (uint32_t)pat_off(PP, PX, (int)l0);
      bi[X2_NT + tid] = idx | ((blk_in && tid > 0 && tid < X2_NT - 1 && l0 == 0) ? 1u << 12 : 0u) | ((J - j0) << 13) |
                        ((l0 % PX) << 21);
      if (tid == 0) s_bj0[buf] = j0;
      uint32_t m = selmask;
      while (m) {
        const int i = __ffs(m) - 1;
        m &= m - 1;
        if (idx < (uint32_t)X2_CAP) {
          const uint64_t hv = HZ[tid * W + i];
          se[idx] = (uint32_t)(tid * W + i) | ((uint32_t)(hv >> ks) << 16);
          shz[idx] = hv;
        }
        ++idx;
      }
      __syncthreads();
      return total;
    };
    uint32_t cnt = compact();
    // exactness of the 31-bit keys: candidates closer than w with equal keys but different hashes
    if (cnt > (uint32_t)X2_CAP && !T.any_n && !T.slow) {
      // too many for the staging (and the tie check works on the staged list): exact selection
      slow_path();
      if (tid == 0 || tid == X2_NT - 1 || !blk_in) selmask = 0;
      cnt = compact();
    } else if (!T.any_n && !T.slow && ks > 0 && !(a.dbg_flags & 2u)) {
      bool tie = false;
      for (uint32_t r = tid; r < cnt; r += X2_NT) {
        const uint32_t vr = se[r];
        const int er = vr & 0xFFFFu;
        // later candidates within W positions: three independent SMEM loads per round
        for (uint32_t q = r + 1; q < cnt; q += 3) {
          uint32_t vq[3];
#pragma unroll
          for (int u = 0; u < 3; u++) vq[u] = q + u < cnt ? se[q + u] : 0xFFFFu;
          bool more = true;
#pragma unroll
          for (int u = 0; u < 3; u++) {
            if ((int)(vq[u] & 0xFFFFu) - er >= W) { more = false; break; }
            if ((vq[u] >> 16) == (vr >> 16)) {  // 16 key bits agree: compare the full keys and hashes
              const uint64_t hr = HZ[er] & ~(1ull << 63), hq = HZ[vq[u] & 0xFFFFu] & ~(1ull << 63);
              tie |= ((hq >> ks) == (hr >> ks)) & (hq != hr);
            }
          }
          if (!more) break;
        }
      }
      if (__syncthreads_or(tie)) {
        if (tid == 0 && a.dbg_counts) atomicAdd(&a.dbg_counts[1], 1u);
        slow_path();
        if (tid == 0 || tid == X2_NT - 1 || !blk_in) selmask = 0;
        cnt = compact();
      }
    }
    // publish this tile's count; its records leave two iterations later (warp 0, flush_warp0), or
    // now if they did not fit the staging
    if (tid == 0 && !(a.dbg_flags & 1u)) lb_publish(a.status, tile, cnt);
    if (cnt > (uint32_t)X2_CAP) {
      if (wid == 0) {
        uint64_t base;
        if (a.dbg_flags & 1u) base = lane == 0 ? atomicAdd((unsigned long long*)&a.status[ntiles], (unsigned long long)cnt) : 0;
        else base = lb_resolve_warp(a.status, tile, cnt);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (lane == 0) {
          s_ovf_base = base;
          if (tile == ntiles - 1) *a.total_out = base + cnt;
        }
      }
      __syncthreads();
      const uint64_t base = s_ovf_base;
      if (a.job_off && blk_in && tid > 0 && tid < X2_NT - 1 && l0 == 0) a.job_off[J] = base + my_idx0;
      uint32_t m = selmask, idx = my_idx0;
      const uint32_t pb = sjp[J - j0] + (uint32_t)pat_off(PP, PX, (int)l0);
      while (m) {
        const int i = __ffs(m) - 1;
        m &= m - 1;
        const uint64_t gi = base + idx;
        if (gi < a.cap) {
          a.out_hz[gi] = HZ[tid * W + i];
          a.out_pos[gi] = pb + pat_delta<PP, PX>(l0 % PX, (uint32_t)i);
          if (a.out_job) a.out_job[gi] = J;
        }
        ++idx;
      }
      cnt = X2_FLUSHED;
    }
    pend_old = pend_new;
    cnt_old = cnt_new;
    pend_new = tile;
    cnt_new = cnt;
    buf ^= 1;
    __syncthreads();
  }
  // pend_old was flushed in the last (tile-less) iteration; the newest tile is in buffer buf ^ 1
  if (pend_new >= 0 && cnt_new != X2_FLUSHED && wid == 0) flush_warp0((uint64_t)pend_new, cnt_new, buf ^ 1);
}

// per-tile descriptors: first and last job (binary searches over the padded bases), the tile's
// code-word range, and whether it is a single job whose bytes can be read unchecked
__global__ void k_x2_tile_desc(const uint64_t* __restrict__ kb, const uint64_t* __restrict__ cw,
                               const Job* __restrict__ jobs, uint32_t n_jobs, uint64_t total_blocks, int W, int NB,
                               int maxwords, int PP, int PX, uint32_t one0, uint64_t seq_bytes, uint64_t ntiles,
                               X2Desc* desc) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntiles; t += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t b_first = (int64_t)t * X2_OUT_BLOCKS - 1;
    const int64_t b_last = (int64_t)t * X2_OUT_BLOCKS + X2_NT - 2;
    const uint64_t gmax = total_blocks * W - 1;
    const uint64_t gfirst = b_first < 0 ? 0 : (uint64_t)b_first * W;
    uint64_t glast = (uint64_t)(b_last < 0 ? 0 : b_last) * W;
    if (glast > gmax) glast = gmax;
    const uint32_t j0 = find_job_le(kb, 0, n_jobs - 1, gfirst);
    const uint32_t j1 = find_job_le(kb, j0, n_jobs - 1, glast);
    const uint64_t lo = b_first < 0 ? cw[0] : cw[j0] + (gfirst - kb[j0]) / 16;
    uint64_t hi = cw[j1] + (glast - kb[j1] + NB + 15) / 16 + 1;
    if (hi > cw[j1 + 1]) hi = cw[j1 + 1];
    if (hi < lo) hi = lo;
    if (hi > lo + (uint64_t)maxwords) hi = lo + maxwords;
    const Job jb = jobs[j0];
    // bytes touched up to word hi: base 16 (hi - cw) at offset <= (q / x + 1) p, plus the load width
    const uint64_t last_byte = jb.seq_off + jb.phase + one0 + (16 * (hi - cw[j0]) / PX + 1) * PP + 48;
    // jobs are in sequence-buffer order: the tile's last bytes are those of job j1
    const Job jl = jobs[j1];
    const uint64_t last_l = jl.seq_off + jl.phase + one0 + (16 * (hi - cw[j1]) / PX + 1) * PP + 48;
    X2Desc d;
    d.j0 = j0;
    d.j1 = j1;
    d.simple = (j0 == j1) && last_byte <= seq_bytes;
    d.safe = last_l <= seq_bytes && last_byte <= seq_bytes;
    d.cw_lo = lo;
    d.cw_hi = hi;
    desc[t] = d;
  }
}

// padded position bases (multiple of W) and code-word bases per job
__global__ void k_x2_sizes(const Job* __restrict__ jobs, uint32_t n, int K, int W, uint64_t* kb, uint64_t* cw,
                           unsigned long long* nk_sum) {
  uint64_t acc = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint64_t nk = jobs[j].nk;
    kb[j] = (nk ? (nk + W - 1) / W : 1) * W;  // no separator: job boundaries are handled in-kernel
    const uint64_t ncode = nk ? nk + K - 1 : 0;
    cw[j] = (ncode + 15) / 16;
    acc += nk;
  }
  for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(nk_sum, (unsigned long long)acc);
}

template <int K, int W, int PP, int PX>
size_t x2_smem_bytes() {
  return X2Cfg<K, W, PP, PX>::SMEM;
}

template <int K, int W, int PP, int PX>
void launch_x2(const X2Args& a, uint64_t ntiles, cudaStream_t st, const char* tag) {
  static int grid = 0;
  const size_t smem = x2_smem_bytes<K, W, PP, PX>();
  if (!grid) {
    GOD_CUDA(cudaFuncSetAttribute(k_extract2<K, W, PP, PX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    GOD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_extract2<K, W, PP, PX>, X2_NT, smem));
    grid = (per_sm > 0 ? per_sm : 1) * num_sms();
  }
  const unsigned g = (unsigned)(ntiles < (uint64_t)grid ? ntiles : (uint64_t)grid);
  GOD_LAUNCH(tag, (k_extract2<K, W, PP, PX>), g, X2_NT, smem, st, a);
}

}  // namespace

bool x2_supported(const Params& P) {
  // patterns: x = 1 with p <= 3 (any rotation: "1", "10", "100"), or p = x + 1 <= 4 with the ones
  // first ("110", "1110")
  const int PP = (int)P.pat.p, PX = (int)P.pat.x;
  bool pat_ok = (PX == 1 && PP <= 3) || ((PX == 2 || PX == 3) && PP == PX + 1);
  if (PX >= 2)
    for (int i = 0; i < PX; i++) pat_ok = pat_ok && P.pat.one[i] == (uint32_t)i;
  if (!pat_ok) return false;
  const int K = P.k, W = P.w;
  auto supported = [&](int k, int w) { return K == k && W == w; };
  // the BASELINE configs (21,11), (19,19), (15,10) and the paper's containment search (19,16)
  if (!(supported(21, 11) || supported(19, 19) || supported(15, 10) || supported(19, 16))) return false;
  return !getenv("GOD_DISABLE_X2");
}

// Returns false if no specialised kernel exists for these parameters (caller uses the generic one).
bool run_extract2(const Params& P, const uint8_t* seq, uint64_t seq_bytes, const Job* jobs, uint32_t n_jobs,
                  bool want_job, bool want_job_off, Records& rec, cudaStream_t st, Scratch& scr,
                  uint64_t cap_hint, const char* tag, const X2Layout* x2) {
  if (!x2_supported(P)) return false;
  const int PP = (int)P.pat.p, PX = (int)P.pat.x;
  const int K = P.k, W = P.w;
  rec.n = 0;
  if (n_jobs == 0) return false;
  // padded layouts (built by make_jobs in the same pass as the jobs, else here)
  const uint64_t* kb;
  const uint64_t* cw;
  uint64_t total_pos, nk_sum;
  if (x2) {
    kb = x2->kb;
    cw = x2->cw;
    total_pos = x2->total_pos;
    nk_sum = x2->nk_sum;
  } else {
    uint64_t* kbw = scr.alloc<uint64_t>(n_jobs + 1);
    uint64_t* cww = scr.alloc<uint64_t>(n_jobs + 1);
    uint64_t* tot = scr.alloc<uint64_t>(3);
    GOD_CUDA(cudaMemsetAsync(tot + 2, 0, sizeof(uint64_t), st));
    GOD_LAUNCH("k_x2_sizes", k_x2_sizes, grid_for(n_jobs, 256), 256, 0, st, jobs, n_jobs, K, W, kbw, cww,
               reinterpret_cast<unsigned long long*>(tot + 2));
    scan_exclusive_u64(kbw, kbw, n_jobs, tot, st, scr, "scan_x2_jobs");
    scan_exclusive_u64(cww, cww, n_jobs, tot + 1, st, scr, "scan_x2_jobs");
    GOD_CUDA(cudaMemcpyAsync(kbw + n_jobs, tot, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    GOD_CUDA(cudaMemcpyAsync(cww + n_jobs, tot + 1, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    uint64_t htot[3];
    d2h_small(htot, tot, sizeof(htot), st);
    kb = kbw;
    cw = cww;
    total_pos = htot[0];
    nk_sum = htot[2];
  }
  prof_add_units(tag, nk_sum);
  const uint64_t total_blocks = total_pos / W;
  const uint64_t ntiles = (total_blocks + X2_OUT_BLOCKS - 1) / X2_OUT_BLOCKS;
  GOD_REQUIRE(ntiles < 0x7FFFFFFFull, "input too large for one extraction launch");
  uint64_t cap = cap_hint ? cap_hint : total_pos;
  if (cap > total_pos) cap = total_pos;
  if (cap == 0) cap = 1;
  uint64_t* status = scr.alloc<uint64_t>(ntiles + 1);
  X2Desc* desc = scr.alloc<X2Desc>(ntiles ? ntiles : 1);
  uint32_t* ctr = scr.alloc<uint32_t>(1);
  if (ntiles) {
    const int NB = W + K - 1;
    const int maxwords = (X2_NT * W + X2_NT * (K - 1) + 15) / 16 + X2_NT + 8;  // X2Cfg::MAXWORDS
    GOD_LAUNCH("k_x2_tile_desc", k_x2_tile_desc, grid_for(ntiles, 256), 256, 0, st, kb, cw, jobs, n_jobs, total_blocks,
               W, NB, maxwords, PP, PX, P.pat.one[0], seq_bytes, ntiles, desc);
  }
  uint64_t* dtotal = scr.alloc<uint64_t>(1);
  if (want_job_off) rec.job_off = scr.alloc<uint64_t>(n_jobs + 1);
  const char* dflag = getenv("GOD_X2_DBG");
  const uint32_t dbg_flags = dflag ? (uint32_t)atoi(dflag) : 0u;
  uint32_t* dbg_counts = nullptr;
  if (dflag) {
    dbg_counts = scr.alloc<uint32_t>(2);
    GOD_CUDA(cudaMemsetAsync(dbg_counts, 0, 8, st));
  }
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
    GOD_CUDA(cudaMemsetAsync(status, 0, (ntiles + 1) * sizeof(uint64_t), st));
    GOD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
    X2Args a{seq, seq_bytes, jobs, kb, cw, n_jobs, total_blocks, P.pat.one[0], key_shift, status, ctr,
             rec.hz, rec.pos, rec.job, rec.job_off, cap, dtotal, dbg_flags, dbg_counts, desc};
    if (ntiles) {
      auto by_pattern = [&](auto kc, auto wc) {
        constexpr int KK = decltype(kc)::value, WW = decltype(wc)::value;
        if (PX == 1 && PP == 1) launch_x2<KK, WW, 1, 1>(a, ntiles, st, tag);
        else if (PX == 1 && PP == 2) launch_x2<KK, WW, 2, 1>(a, ntiles, st, tag);
        else if (PX == 1) launch_x2<KK, WW, 3, 1>(a, ntiles, st, tag);
        else if (PX == 2) launch_x2<KK, WW, 3, 2>(a, ntiles, st, tag);
        else launch_x2<KK, WW, 4, 3>(a, ntiles, st, tag);
      };
      if (K == 21 && W == 11) by_pattern(std::integral_constant<int, 21>(), std::integral_constant<int, 11>());
      else if (K == 19 && W == 19) by_pattern(std::integral_constant<int, 19>(), std::integral_constant<int, 19>());
      else if (K == 19 && W == 16) by_pattern(std::integral_constant<int, 19>(), std::integral_constant<int, 16>());
      else by_pattern(std::integral_constant<int, 15>(), std::integral_constant<int, 10>());
    } else {
      GOD_CUDA(cudaMemsetAsync(dtotal, 0, sizeof(uint64_t), st));
    }
    const uint64_t n = d2h_scalar(dtotal, st);
    if (dbg_counts) {
      uint32_t hc[2];
      GOD_CUDA(cudaMemcpy(hc, dbg_counts, 8, cudaMemcpyDeviceToHost));
      fprintf(stderr, "[x2] %s tiles=%llu slow=%u tie=%u\n", tag, (unsigned long long)ntiles, hc[0], hc[1]);
    }
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
