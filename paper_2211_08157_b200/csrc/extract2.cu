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
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include "internal.cuh"

namespace god {

namespace {

// threads (= W-blocks) per tile.  Smaller CTAs mean more independent barrier domains per SM (the
// kernel's top stall is the CTA barrier) at the price of more halo blocks (2 per tile).
#ifndef X2_NT_DEF
#define X2_NT_DEF 128
#endif
constexpr int X2_NT = X2_NT_DEF;
constexpr int X2_OUT_BLOCKS = X2_NT - 2;
// unordered output staging (selected records per tile); density is ~2/(w+1), i.e. ~17% of a tile's
// positions: a tile with more (all-ties runs) writes its records directly
constexpr int X2_CAP = 4 * X2_NT;
// resident CTAs per SM the register allocation is sized for (SMEM allows 7): 7 for w <= 11 (72
// registers, no spills), 6 for w = 19 (more registers per W-block)
template <int W>
constexpr int x2_minb() { return (W >= 16 ? 5 : 7) * (128 / X2_NT); }

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
  uint64_t* job_end;    // aligned tiles: one past each job's last record (else null: job_off[j + 1])
  uint64_t cap;
  uint64_t* total_out;
  uint32_t dbg_flags;      // developer toggles (GOD_X2_DBG): 2 = no tie check
  uint32_t* dbg_counts;    // [0] tiles on the slow path, [1] tiles with a key tie
  const struct X2Desc* desc;  // [ntiles] per-tile descriptors (k_x2_tile_desc)
  uint32_t aligned;     // tiles are whole jobs (k_x2_tile_desc_aligned): no halo blocks
  uint64_t ntiles;
  uint32_t no_stage;    // developer toggle (GOD_X2_NO_STAGE): direct global loads in the sparsify stage
  // slotted output (position order without inter-CTA waiting): tile t writes its records at t * X2_CAP
  // and its count to tile_cnt[t]; a scan and k_x2_compact close the gaps.  A tile with more than X2_CAP
  // records sets *overflow (the caller then runs the look-back kernel instead)
  uint32_t* tile_cnt;
  uint32_t* overflow;
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

__device__ __forceinline__ uint32_t rev2(uint32_t x) {  // reverse the 16 2-bit fields of x
  const uint32_t y = __brev(x);
  return ((y >> 1) & 0x55555555u) | ((y & 0x55555555u) << 1);
}

// per-tile descriptor, precomputed by k_x2_tile_desc so that a CTA never walks a dependent chain
// of global loads (tile -> jobs -> code-word range) while its other warps wait at a barrier
struct __align__(16) X2Desc {
  uint32_t j0, j1, simple, safe;  // safe: every byte the tile may read is inside the buffer
  uint64_t cw_lo, cw_hi;
  uint64_t b0;                    // aligned tiles: first block (thread 0's), and the block count
  uint32_t nb, raw_len;           // raw_len: bytes a bulk copy stages for the tile (0: direct loads)
  uint64_t raw_lo;                // ... from this 16-B aligned global address
  uint64_t need;                  // the tile reads only bytes [0, need) of the sequence buffer (streamed input)
};
// bytes of the SMEM buffer the next tile's ASCII bytes are staged into (unordered K1)
constexpr uint32_t X2_RAW_CAP = 48 * X2_NT;
// the byte span [lo, hi) one job's code words [ws, we) load from (pack16: words aligned in the address
// space, pack_words of them from each word's first byte)
__device__ __forceinline__ void job_byte_span(uint64_t base, uint64_t ws, uint64_t we, int PP, int PX, int NL,
                                              uint64_t& lo, uint64_t& hi) {
  const uint64_t q0 = 16 * ws, q1 = 16 * (we - 1);
  lo = base + (q0 / PX) * PP + q0 % PX;
  hi = ((base + (q1 / PX) * PP + q1 % PX) & ~3ull) + 4ull * NL;
}
__device__ __forceinline__ int pack_words_rt(int PP, int PX) {
  int mx = 0;
  for (int r = 0; r < PX; r++) {
    const int q = r + 15;
    const int v = ((q / PX) * PP + q % PX) - ((r / PX) * PP + r % PX);
    mx = v > mx ? v : mx;
  }
  return (mx + 3) / 4 + 2;
}
// the tile's staged span if it fits X2_RAW_CAP and lies inside [seq, seq + seq_bytes) after 16-B alignment
__device__ __forceinline__ void raw_span(const uint8_t* seq, uint64_t seq_bytes, uint64_t lo, uint64_t hi,
                                         uint64_t& raw_lo, uint32_t& raw_len) {
  const uint64_t s0 = reinterpret_cast<uintptr_t>(seq);
  const uint64_t a = (s0 + lo) & ~15ull, b = (s0 + hi + 15) & ~15ull;
  raw_lo = a;
  raw_len = (a >= s0 && b <= s0 + seq_bytes && b - a <= X2_RAW_CAP && hi > lo) ? (uint32_t)(b - a) : 0u;
}

// bytes of the buffer a tile may touch: [0, need).  last_byte bounds every direct load (with its margin),
// sp_hi the staged span before its 16-B alignment in the address space; checked loads stop at seq_bytes
__device__ __forceinline__ uint64_t tile_need(uint64_t last_byte, uint64_t sp_hi, uint64_t seq_bytes) {
  const uint64_t n = last_byte > sp_hi + 16 ? last_byte : sp_hi + 16;
  return n < seq_bytes ? n : seq_bytes;
}

struct X2Tile {  // per-tile scalars, in SMEM
  uint32_t tile, j0, j1, simple, safe, slow, nb, raw_len;
  uint64_t cw_lo, cw_hi, b0, raw_lo;
};

template <int K, int W, int PP, int PX>
struct X2Cfg {
  static_assert(X2_NT * W < 65536, "staged tile-local record indices are 16-bit");
  static constexpr int NB = W + K - 1;                 // bases in a thread's window
  static constexpr int NWIN = (2 * NB + 31) / 32;       // aligned window words
  static constexpr int NLOAD = (30 + 2 * NB + 31) / 32; // words loaded before alignment
  static constexpr int POS = X2_NT * W;                 // positions per tile (incl. the two halo blocks)
  static constexpr int MAXWORDS = (POS + X2_NT * (K - 1) + 15) / 16 + X2_NT + 8;
  // SMEM layout (bytes)
  static constexpr size_t O_LUT = 0;
  static constexpr size_t O_CODES = O_LUT + 256 * 4;
  static constexpr size_t O_NMASK = O_CODES + (size_t)MAXWORDS * 4;
  static constexpr int WP = (W + 3) / 4 * 4;  // exchange row (16-B vectors)
  static constexpr size_t O_XCHG = (O_NMASK + (size_t)MAXWORDS * 4 + 15) / 16 * 16;
  static constexpr size_t O_STG = (O_XCHG + 2 * (X2_NT / 32) * WP * 4 + 15) / 16 * 16;  // [X2_CAP] indices
  static constexpr size_t O_HZ = O_STG + (size_t)X2_CAP * 2;                                  // [NHZ][POS] hz
  // ordered output keeps the previous tile's hashes until its look-back resolves (2 buffers)
  // unordered: one HZ buffer + the raw-byte staging buffer of the next tile; ordered: two HZ buffers
  static constexpr size_t O_RAW = O_HZ + (size_t)POS * 8;
  static constexpr size_t smem(bool ordered) {
    return ((ordered ? O_HZ + 2 * (size_t)POS * 8 : O_RAW + X2_RAW_CAP) + 15) / 16 * 16;
  }
};

// (pack16 gathers the included bytes with compile-time byte-permutations)
// *nm gets the N bits (bit 15 - b for base b).  nb = bases that exist (<= 16).
// Pattern geometry: period PP with ones at offsets 0..PX-1 (x = 1 patterns may be rotated: their
// single one's offset is added to the job base).  Included base q of a job lies at byte offset
// (q / PX) * PP + q % PX.
__host__ __device__ constexpr int pat_off(int PP, int PX, int q) { return (q / PX) * PP + q % PX; }
// the same for a runtime k-mer index (up to the sequence length: no int overflow past 2^31; the
// whole-config digest test caught human '1110' positions beyond 2.86 Gbp computed through int)
template <int PP, int PX>
__device__ __forceinline__ uint32_t pat_off_u(uint32_t q) {
  return (uint32_t)(((uint64_t)(q / PX)) * PP + q % PX);
}
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
// SMEM: the tile's bytes were staged by a bulk copy into sm (its first byte is the global address
// sm_base, 16-B aligned); the same aligned words are read from there
template <int PP, int PX, int R0, bool CHECKED, bool SMEM = false>
__device__ __forceinline__ uint32_t pack16(const uint8_t* seq, uint64_t seq_bytes, uint64_t A, int nb,
                                           const uint32_t* lut, uint32_t* nm, const uint32_t* sm = nullptr,
                                           uintptr_t sm_base = 0) {
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
    if constexpr (SMEM) {
      w[i] = sm[(pa - sm_base) / 4 + i];
    } else if constexpr (CHECKED) {
      const int64_t ad = (int64_t)(pa - reinterpret_cast<uintptr_t>(seq)) + 4ll * i;  // relative to seq
      uint32_t v = 0;
      if (ad >= 0 && (uint64_t)ad + 4 <= seq_bytes) v = __ldg(src + i);
      else
        for (int64_t q = ad < 0 ? 0 : ad; q < ad + 4 && (uint64_t)q < seq_bytes; q++)
          v |= (uint32_t)seq[q] << (8 * (q - ad));
      w[i] = v;
    } else {
#ifdef GOD_CHECKED
      {
        const int64_t ad = (int64_t)(pa - reinterpret_cast<uintptr_t>(seq)) + 4ll * i;
        if (ad < -3 || ad >= (int64_t)seq_bytes)
          printf("GOD_CHECKED detail: A=%llu ad=%lld i=%d NL=%d seq_bytes=%llu nb=%d block %u thread %u\n",
                 (unsigned long long)A, (long long)ad, i, NL, (unsigned long long)seq_bytes, nb, blockIdx.x, threadIdx.x);
      }
#endif
      GOD_DCHECK((int64_t)(pa - reinterpret_cast<uintptr_t>(seq)) + 4ll * i >= -3 &&
                     (int64_t)(pa - reinterpret_cast<uintptr_t>(seq)) + 4ll * i < (int64_t)seq_bytes,
                 "K1 unchecked sequence load inside the buffer");
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
template <int PP, int PX, bool CHECKED, bool SMEM = false>
__device__ __forceinline__ uint32_t pack_word(const uint8_t* seq, uint64_t seq_bytes, uint64_t A0, uint64_t q0, int nb,
                                              const uint32_t* lut, uint32_t* nm, const uint32_t* sm = nullptr,
                                              uintptr_t sm_base = 0) {
  const uint32_t r0 = (uint32_t)(q0 % PX);
  const uint64_t A = A0 + (q0 / PX) * PP + r0;
  if constexpr (PX == 1) {
    return pack16<PP, PX, 0, CHECKED, SMEM>(seq, seq_bytes, A, nb, lut, nm, sm, sm_base);
  } else if constexpr (PX == 2) {
    return r0 ? pack16<PP, PX, 1, CHECKED, SMEM>(seq, seq_bytes, A, nb, lut, nm, sm, sm_base)
              : pack16<PP, PX, 0, CHECKED, SMEM>(seq, seq_bytes, A, nb, lut, nm, sm, sm_base);
  } else {
    static_assert(PX == 3, "patterns with up to 3 leading ones");
    return r0 == 0 ? pack16<PP, PX, 0, CHECKED, SMEM>(seq, seq_bytes, A, nb, lut, nm, sm, sm_base)
         : r0 == 1 ? pack16<PP, PX, 1, CHECKED, SMEM>(seq, seq_bytes, A, nb, lut, nm, sm, sm_base)
                   : pack16<PP, PX, 2, CHECKED, SMEM>(seq, seq_bytes, A, nb, lut, nm, sm, sm_base);
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
// ... and resolve the exclusive prefix later (whole warp), publishing the inclusive prefix.
// The resident CTAs reach this point almost in lock-step (each resolves tile t after computing its
// next tile), so a tile's predecessors mostly carry aggregates, not inclusive prefixes, and the walk
// back spans the whole resident window (~600 tiles on 148 SMs).  LB_R rounds of 32 predecessors are
// therefore loaded at once: ~3 dependent L2 round trips instead of ~18 (measured on HiFi reads, whose
// long jobs need position order: extract_seed 19.2 -> see DESIGN.md §6).
constexpr int LB_R = 8;
__device__ inline uint64_t lb_resolve_warp(uint64_t* status, uint64_t tile, uint64_t local) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) return 0;
  uint64_t part = 0;  // this lane's share of the exclusive prefix
  int64_t j0 = (int64_t)tile - 1;
  bool done = false;
  while (!done) {
    uint64_t s[LB_R];
#pragma unroll
    for (int r = 0; r < LB_R; r++) {
      const int64_t j = j0 - 32 * r - lane;
      s[r] = j >= 0 ? lb_load(&status[j]) : (LB_INC | 0ull);
    }
#pragma unroll
    for (int r = 0; r < LB_R; r++) {
      if (done) break;
      const int64_t j = j0 - 32 * r - lane;
      while (__any_sync(0xffffffffu, (s[r] & ~LB_VAL) == 0)) {
        __nanosleep(32);  // back off: a spinning warp takes issue slots from the CTAs doing the work
        if ((s[r] & ~LB_VAL) == 0) s[r] = lb_load(&status[j]);
      }
      const uint32_t inc = __ballot_sync(0xffffffffu, (s[r] & ~LB_VAL) == LB_INC);
      const int first = inc ? __ffs(inc) - 1 : 32;
      if (lane <= first) part += s[r] & LB_VAL;
      done = inc != 0;
    }
    j0 -= 32 * LB_R;
  }
  uint64_t excl = part;
#pragma unroll
  for (int o = 16; o; o >>= 1) excl += __shfl_xor_sync(0xffffffffu, excl, o);
  if (lane == 0) lb_store(&status[tile], LB_INC | (excl + local));
  return excl;
}

// ---------------------------------------------------------------------------------------------
// Lean two-word arithmetic for B.  A k-mer / hash value of 2K bits is held as hi:lo with the top
// HB = 2K - 32 bits in hi (K = 21: 10 bits, K = 19: 6 bits) or, for 2K <= 32, in lo alone.  A
// multiplication by a 32-bit constant is one IMAD.WIDE.U32 plus one IMAD (the wide product's high
// word is the carry into hi); an xor-shift by s >= HB is one mask of hi, one funnel shift and one
// LOP3 (hi ^ hi >> s == hi).  Every step is reduced mod 2^2K as in O5.
template <int K>
struct KW {
  static constexpr int HB = 2 * K > 32 ? 2 * K - 32 : 0;
  static constexpr uint32_t HM = HB ? (1u << HB) - 1 : 0u;
  static constexpr uint32_t LM = 2 * K >= 32 ? 0xFFFFFFFFu : (1u << (2 * K)) - 1;
  static_assert(HB <= 14, "xor-shift steps assume hi has at most 14 bits");
};

template <int K>
__device__ __forceinline__ void wang_hash_2w(uint32_t& hi, uint32_t& lo) {
  if constexpr (KW<K>::HB > 0) {
    constexpr uint32_t HM = KW<K>::HM;
    auto mul = [&](uint32_t c) {
      const uint64_t p = (uint64_t)lo * c;
      hi = hi * c + (uint32_t)(p >> 32);
      lo = (uint32_t)p;
    };
    {  // x1 = (2^21 - 1) x - 1: the -1 rides in the wide multiply's 64-bit addend
      const uint64_t p = (uint64_t)lo * ((1u << 21) - 1) + ~0ull;
      hi = hi * ((1u << 21) - 1) + (uint32_t)(p >> 32);
      lo = (uint32_t)p;
    }
    hi &= HM; lo ^= __funnelshift_r(lo, hi, 24);   // x2 = x1 ^ x1 >> 24
    mul(265u);                                      // x3
    hi &= HM; lo ^= __funnelshift_r(lo, hi, 14);   // x4
    mul(21u);                                       // x5
    hi &= HM; lo ^= __funnelshift_r(lo, hi, 28);   // x6
    mul(0x80000001u);                               // H = (2^31 + 1) x6
    hi &= HM;
  } else {
    constexpr uint32_t LM = KW<K>::LM;
    uint32_t x = lo;
    x = (x * ((1u << 21) - 1) - 1u) & LM;
    x ^= x >> 24;
    x = (x * 265u) & LM;
    x ^= x >> 14;
    x = (x * 21u) & LM;
    x ^= x >> 28;
    x = (x * 0x80000001u) & LM;
    lo = x;
    hi = 0;
  }
}

// 32 bits of the MSB-first bit string w[] starting at bit S (compile-time after unrolling)
template <int NW>
__device__ __forceinline__ uint32_t ext32(const uint32_t (&w)[NW], const int S) {
  const int i = S >> 5, o = S & 31;
  return o ? __funnelshift_l(word_at(w, i + 1), word_at(w, i), o) : word_at(w, i);
}
// the 2K-bit k-mer at bit S of w[] as hi:lo
template <int K, int NW>
__device__ __forceinline__ void kmer_2w(const uint32_t (&w)[NW], const int S, uint32_t& hi, uint32_t& lo) {
  constexpr int HB = KW<K>::HB;
  if constexpr (HB > 0) {
    lo = ext32(w, S + HB);
    hi = ext32(w, S) >> (32 - HB);
  } else {
    lo = ext32(w, S) >> (32 - 2 * K);
    hi = 0;
  }
}

// ---------------------------------------------------------------------------------------------
// Persistent CTAs take tiles in order (one ahead, descriptor prefetched).  Per tile: A (all warps)
// sparsify into SMEM; B/C per thread-block of W positions; the exact slow path when the tile needs
// it; E: every thread writes its own selected records straight to the output at the tile's base,
// which comes from a decoupled look-back over tiles (ORDERED: position order, as god_minimizers
// and the phase path need) or from one atomicAdd (the index path, whose sort orders by (hash, pos)).
template <int K, int W, int PP, int PX, bool ORDERED>
__global__ void __launch_bounds__(X2_NT, x2_minb<W>()) k_extract3(X2Args a) {
  static_assert((K & 1) == 1, "odd k only: no palindromic k-mers (O4); even k runs the generic kernel");
  using C = X2Cfg<K, W, PP, PX>;
  constexpr int NB = C::NB, NWIN = C::NWIN, NLOAD = C::NLOAD, POS = C::POS;
  constexpr int NWARP = X2_NT / 32;
  extern __shared__ __align__(16) unsigned char x2_smem[];
  uint32_t* lut = reinterpret_cast<uint32_t*>(x2_smem + C::O_LUT);
  uint32_t* codes = reinterpret_cast<uint32_t*>(x2_smem + C::O_CODES);
  uint32_t* nmask = reinterpret_cast<uint32_t*>(x2_smem + C::O_NMASK);
  uint32_t* xpf = reinterpret_cast<uint32_t*>(x2_smem + C::O_XCHG);
  uint32_t* xsf = xpf + NWARP * C::WP;
  // a warp's boundary values go through SMEM as 16-B vectors (W scalar stores/loads per value set cost
  // ~6 slots per position, measured)
  auto put_row = [&](uint32_t* row, const uint32_t (&v)[W]) {
#pragma unroll
    for (int j = 0; j < C::WP / 4; j++)
      reinterpret_cast<uint4*>(row)[j] = make_uint4(v[4 * j], 4 * j + 1 < W ? v[4 * j + 1] : 0u,
                                                    4 * j + 2 < W ? v[4 * j + 2] : 0u, 4 * j + 3 < W ? v[4 * j + 3] : 0u);
  };
  auto get_row = [&](const uint32_t* row, uint32_t (&v)[W]) {
#pragma unroll
    for (int j = 0; j < C::WP / 4; j++) {
      const uint4 q = reinterpret_cast<const uint4*>(row)[j];
      v[4 * j] = q.x;
      if (4 * j + 1 < W) v[4 * j + 1] = q.y;
      if (4 * j + 2 < W) v[4 * j + 2] = q.z;
      if (4 * j + 3 < W) v[4 * j + 3] = q.w;
    }
  };
  uint64_t* const HZ0 = reinterpret_cast<uint64_t*>(x2_smem + C::O_HZ);  // [NHZ][POS] hash | strand << 63
  // Unordered: thread 0 stages the NEXT tile's ASCII bytes into raw[] by one bulk copy (cp.async.bulk,
  // completion on an mbarrier) while this tile computes, so the sparsify stage reads SMEM, not global
  // memory, on its critical path.
  const uint32_t* raw = reinterpret_cast<const uint32_t*>(x2_smem + C::O_RAW);
  __shared__ __align__(8) uint64_t s_mbar;
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
  uint32_t raw_phase = 0;
  auto raw_issue = [&](const X2Desc& d) {  // thread 0
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the previous tile's generic reads of raw[]
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(d.raw_len) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(raw)),
                 "l"(d.raw_lo), "r"(d.raw_len), "r"(mbar)
                 : "memory");
  };
  auto raw_wait = [&]() {  // every thread
    uint32_t done = 0;
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(mbar), "r"(raw_phase)
                   : "memory");
    } while (!done);
    raw_phase ^= 1u;
  };

  uint64_t* HZ = HZ0;
  // unordered output: the tile's selected positions (tile-local index) staged in position order
  uint16_t* SIDX = reinterpret_cast<uint16_t*>(x2_smem + C::O_STG);  // [X2_CAP]
  __shared__ uint32_t SBASE[X2_NT];  // per block: output position of its first k-mer start
  __shared__ uint8_t SR0[X2_NT];     // per block: its first k-mer index mod x
  __shared__ X2Tile T;
  __shared__ uint64_t skb[X2_NT + 2], scw[X2_NT + 2];
  __shared__ uint64_t sjb[X2_NT + 2];  // per job of the tile: byte address of its first patterned base
  __shared__ uint32_t sjn[X2_NT + 2];  // ... its k-mer count n_k
  __shared__ uint32_t sjp[X2_NT + 2];  // ... its output position base (pos_base + phase + one0)
  using swj_t = std::conditional_t<(X2_NT > 128), uint16_t, uint8_t>;
  __shared__ swj_t swj[(X2Cfg<K, W, PP, PX>::MAXWORDS + 3) / 4 * 4];  // code word -> job (relative)
  __shared__ uint32_t sjob[X2_NT];
  __shared__ uint32_t warp_cnt[NWARP];
  __shared__ uint32_t xlast[NWARP];    // per warp: lane 31's last selected (offset << 27 | key >> 5) ...
  __shared__ uint32_t xlastk[NWARP];   // ... and its key
  __shared__ uint64_t s_base;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t ntiles = a.ntiles;
  if (!ORDERED && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t ks = a.key_shift;  // <= 31
  {  // expected-letter table: for 4 MSB-first codes pk, bytes "ACGT"[c_i], base 0 in byte 0
    const uint32_t L4 = 0x54474341u;
    for (int pk = tid; pk < 256; pk += X2_NT) {
      uint32_t e = 0;
#pragma unroll
      for (int i = 0; i < 4; i++) e |= ((L4 >> (8 * ((pk >> (6 - 2 * i)) & 3u))) & 0xFFu) << (8 * i);
      lut[pk] = e;
    }
  }
  // tiles are claimed one ahead (descriptor prefetched) when the output is unordered; ORDERED claims
  // each tile when it starts, so tiles are computed in claim order and a tile's predecessors have
  // published their counts by the time its deferred look-back runs
  uint32_t next_t = 0;
  X2Desc nd{};
  if (!ORDERED && tid == 0) {
    next_t = atomicAdd(a.tile_ctr, 1u);
    if (next_t < ntiles) {
      nd = a.desc[next_t];
      if (nd.raw_len && !a.no_stage) raw_issue(nd);
    }
  }
  // ORDERED: the previous tile's records, written one iteration late so that its look-back finds the
  // predecessors' counts published instead of spinning on tiles that other CTAs are still computing
  int64_t p_tile = -1;
  uint32_t p_total = 0, p_sel = 0, p_rank = 0, p_pb = 0, p_r0 = 0, p_J = 0;
  bool p_start = false;
  const uint64_t* p_hz = HZ0;
  auto resolve_pending = [&]() {  // warp 0
    const uint64_t b = lb_resolve_warp(a.status, (uint64_t)p_tile, p_total);
    if (lane == 0) {
      s_base = b;
      if ((uint64_t)p_tile == ntiles - 1) *a.total_out = b + p_total;
    }
  };
  auto write_pending = [&]() {  // all threads, after a barrier that follows resolve_pending
    uint64_t gi = s_base + p_rank;
    if (a.job_off && p_start) a.job_off[p_J] = gi;
    uint32_t m = p_sel;
    while (m) {
      const int i = __ffs(m) - 1;
      m &= m - 1;
      if (gi < a.cap) {
        a.out_hz[gi] = p_hz[tid * W + i];
        a.out_pos[gi] = p_pb + pat_delta<PP, PX>(p_r0, (uint32_t)i);
        if (a.out_job) a.out_job[gi] = p_J;
      }
      ++gi;
    }
  };
  while (true) {
    if (tid == 0) {
      if (ORDERED) {
        next_t = atomicAdd(a.tile_ctr, 1u);
        if (next_t < ntiles) nd = a.desc[next_t];
      }
      T.tile = next_t < ntiles ? next_t : 0xFFFFFFFFu;
      if (next_t < ntiles) {
        T.j0 = nd.j0; T.j1 = nd.j1;
        T.cw_lo = nd.cw_lo; T.cw_hi = nd.cw_hi;
        T.simple = nd.simple;
        T.safe = nd.safe;
        T.slow = 0;
        T.b0 = nd.b0;
        T.nb = nd.nb;
        T.raw_len = (!ORDERED && !a.no_stage) ? nd.raw_len : 0u;
        T.raw_lo = nd.raw_lo;
        if (!ORDERED) {
          next_t = atomicAdd(a.tile_ctr, 1u);
          if (next_t < ntiles) nd = a.desc[next_t];
        }
      }
    }
    __syncthreads();
    const uint32_t tile = T.tile;
    if (tile == 0xFFFFFFFFu) break;

    const uint32_t j0 = T.j0, j1 = T.j1;
    const uint32_t nj = j1 - j0 + 1;
    const uint64_t cw_lo = T.cw_lo;
    const int nwords = (int)(T.cw_hi - cw_lo);
    // the tile's job bases in SMEM (a tile spans <= NT + 1 jobs: every job owns >= 1 block)
    GOD_DCHECK(j1 < a.n_jobs && nj <= X2_NT + 1 && nwords >= 0 && nwords <= C::MAXWORDS, "K1 tile descriptor");
    for (uint32_t q = tid; q <= nj; q += X2_NT) {
      skb[q] = a.kb[j0 + q];
      scw[q] = a.cw[j0 + q];
      if (q < nj) {
        const Job jq = a.jobs[j0 + q];
        sjb[q] = jq.seq_off + jq.phase + a.one0;
        sjn[q] = jq.nk;
        sjp[q] = (uint32_t)(jq.pos_base + jq.phase + a.one0);
      }
    }
    __syncthreads();
    const bool simple = T.simple;
    if (!simple) {  // code word -> job, filled job by job
      for (uint32_t q = tid; q < nj; q += X2_NT) {
        const int64_t w0 = (int64_t)scw[q] - (int64_t)cw_lo, w1 = (int64_t)scw[q + 1] - (int64_t)cw_lo;
        for (int64_t wi = w0 < 0 ? 0 : w0; wi < w1 && wi < nwords; wi++) swj[wi] = (swj_t)q;
      }
      __syncthreads();
    }
    // ------------------------------------------------------------------ A. sparsify into SMEM
    uint32_t my_n = 0;
    const bool staged = T.raw_len != 0;
    const uintptr_t raw_lo = (uintptr_t)T.raw_lo;
    if (staged) raw_wait();
    if (staged) {
      for (int wi = tid; wi < nwords; wi += X2_NT) {
        const uint32_t Jw = simple ? 0u : swj[wi];
        const uint64_t nkq = sjn[Jw];
        const uint64_t ncode = nkq ? nkq + K - 1 : 0;
        const uint64_t q0 = (cw_lo + wi - scw[Jw]) * 16;
        uint32_t nm = 0, word = 0;
        if (q0 < ncode)
          word = pack_word<PP, PX, false, true>(a.seq, a.seq_bytes, sjb[Jw], q0, (int)min((uint64_t)16, ncode - q0),
                                                lut, &nm, raw, raw_lo);
        codes[wi] = word;
        nmask[wi] = nm;
        my_n |= nm;
      }
    } else if (simple) {
      const uint64_t w0 = cw_lo - scw[0];
      const uint32_t ncode = sjn[0] ? sjn[0] + K - 1 : 0;
      const uint64_t A0 = sjb[0];
      for (int wi = tid; wi < nwords; wi += X2_NT) {
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
      for (int wi = tid; wi < nwords; wi += X2_NT) {
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
    const bool any_n = __syncthreads_or(my_n != 0);
    // raw[] is free again: stage the next tile (claimed one ahead) while this one computes
    if (!ORDERED && tid == 0 && next_t < ntiles && nd.raw_len && !a.no_stage) raw_issue(nd);

    // ---- my block: job J, first k-mer index l0
    // aligned tiles: blocks b0 .. b0 + nb - 1 (whole jobs, job boundaries are window barriers, no halo);
    // else blocks tile * 126 - 1 .. tile * 126 + 126, the first and last computed as halo only
    const bool aligned = a.aligned != 0;
    const int64_t myb = aligned ? (int64_t)(T.b0 + tid) : (int64_t)tile * X2_OUT_BLOCKS - 1 + tid;
    const bool blk_in = aligned ? (uint32_t)tid < T.nb : (myb >= 0 && (uint64_t)myb < a.total_blocks);
    const bool emit_blk = blk_in && (aligned || (tid > 0 && tid < X2_NT - 1));
    const int tile_nb = (int)T.nb;  // (T is rewritten for the next tile while this one writes out)
    uint32_t J = j0, l0 = 0, nk = 0;
    if (blk_in) {
      const uint64_t g = (uint64_t)myb * W;
      J = (j0 == j1) ? j0 : j0 + find_job_le(skb, 0, nj - 1, g);
      l0 = (uint32_t)(g - skb[J - j0]);
      nk = sjn[J - j0];
    }
    sjob[tid] = blk_in ? J : 0xFFFFFFFFu;  // block -> job (job boundaries are window barriers)

    // ------------------------------------------------------------------ B. k-mers and hashes
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
    const uint32_t nvalid = blk_has_kmers ? min((uint32_t)W, nk - l0) : 0u;
#pragma unroll
    for (int i = 0; i < W; i++) {
      uint32_t fh, fl, rh, rl;
      kmer_2w<K>(win, 2 * i, fh, fl);
      kmer_2w<K>(rcw, PADB + 2 * (NB - K - i), rh, rl);
      const bool z = (((uint64_t)fh << 32) | fl) > (((uint64_t)rh << 32) | rl);  // canonical (O4)
      uint32_t hi = z ? rh : fh, lo = z ? rl : fl;
      wang_hash_2w<K>(hi, lo);
      HZ[tid * W + i] = ((uint64_t)(hi | (z ? 0x80000000u : 0u)) << 32) | lo;
      const uint32_t kk = __funnelshift_r(lo, hi, ks) + 1u;  // top 31 hash bits + 1 (0 = barrier)
      key[i] = kk;
    }
    if (nvalid < (uint32_t)W) {  // the last block of a job (or past the data): barrier keys
#pragma unroll
      for (int i = 0; i < W; i++)
        if ((uint32_t)i >= nvalid) key[i] = 0u;
    }
    __syncthreads();  // sjob, and the code words are no longer needed by anyone but the slow path

    // ------------------------------------------------------------------ C. selection on keys
    uint32_t selmask = 0;
    uint32_t slow_flags = 0;  // 1: a run shorter than w, 2: a key tie (uniform: from the block-wide vote)
    if (!any_n) {
      bool need_slow = false;
      uint32_t PF[W], SF[W];
      PF[0] = key[0];
#pragma unroll
      for (int i = 1; i < W; i++) PF[i] = min(PF[i - 1], key[i]);
      SF[W - 1] = key[W - 1];
#pragma unroll
      for (int i = W - 2; i >= 0; i--) SF[i] = min(SF[i + 1], key[i]);
      if (lane == 0) {
        put_row(xpf + wid * C::WP, PF);
      }
      __syncthreads();
      uint32_t nPF[W];
#pragma unroll
      for (int i = 0; i < W; i++) nPF[i] = __shfl_down_sync(0xffffffffu, PF[i], 1);
      if (lane == 31) {
        if (wid < NWARP - 1) {
          get_row(xpf + (wid + 1) * C::WP, nPF);
        } else {
#pragma unroll
          for (int q = 0; q < W; q++) nPF[q] = 0u;
        }
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
      uint32_t PXM[W], SX[W];
      PXM[0] = WM[0];
#pragma unroll
      for (int i = 1; i < W; i++) PXM[i] = max(PXM[i - 1], WM[i]);
      SX[W - 1] = WM[W - 1];
#pragma unroll
      for (int i = W - 2; i >= 0; i--) SX[i] = max(SX[i + 1], WM[i]);
      if (lane == 31) {
        put_row(xsf + wid * C::WP, SX);
      }
      uint32_t pSX[W];
#pragma unroll
      for (int i = 0; i < W; i++) pSX[i] = __shfl_up_sync(0xffffffffu, SX[i], 1);
      // tie check, part 1: within the block, each selected position against the previous one
      bool tie = false;
      uint32_t prevk = 0;
      __syncthreads();
      if (lane == 0) {
        if (wid > 0) {
          get_row(xsf + (wid - 1) * C::WP, pSX);
        } else {
#pragma unroll
          for (int q = 0; q < W; q++) pSX[q] = 0u;
        }
      }
#pragma unroll
      for (int o = 0; o < W; o++) {
        const uint32_t mm = (o == W - 1) ? PXM[W - 1] : max(pSX[o + 1], PXM[o]);
        const uint32_t k = key[o];
        const bool s = (k == mm) && k != 0u;
        need_slow |= (k != 0u) & (mm == 0u);  // a run shorter than w: partial-window rule
        tie |= s & (k == prevk);
        selmask |= (uint32_t)s << o;
        prevk = s ? k : prevk;
      }
      // tie check, part 2: the first selected position against the previous block's last one when they
      // are closer than w (offset in this block < offset in the previous block)
      const uint32_t lasto = selmask ? 31u - __clz(selmask) : 0xFFu;
      uint32_t plo = __shfl_up_sync(0xffffffffu, lasto, 1), plk = __shfl_up_sync(0xffffffffu, prevk, 1);
      if (lane == 31) { xlast[wid] = lasto; xlastk[wid] = prevk; }
      __syncthreads();
      if (lane == 0) { plo = wid > 0 ? xlast[wid - 1] : 0xFFu; plk = wid > 0 ? xlastk[wid - 1] : 0u; }
      if (tid > 0 && plo != 0xFFu && selmask) {
        const uint32_t firsto = __ffs(selmask) - 1;
        const uint32_t firstk = (uint32_t)((HZ[tid * W + firsto] & ~(1ull << 63)) >> ks) + 1u;
        if (firsto < plo && firstk == plk) tie = true;
      }
      if (!aligned && (tid == 0 || tid == X2_NT - 1)) need_slow = false;  // halo blocks are not emitted
      if (a.dbg_flags & 2u) tie = false;
      slow_flags = (uint32_t)__syncthreads_or((need_slow ? 1 : 0) | (tie ? 2 : 0));
    }

    // ------------------------------------------------------------------ D. exact slow path (whole tile)
    if (any_n || slow_flags) {
      if (tid == 0 && a.dbg_counts) atomicAdd(&a.dbg_counts[(slow_flags & 2u) && !any_n ? 1 : 0], 1u);
      uint32_t zmask = 0;
#pragma unroll
      for (int i = 0; i < W; i++) zmask |= (uint32_t)(HZ[tid * W + i] >> 63) << i;
      uint64_t* H64 = HZ;  // hash+1, 0 barrier
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
          if (!anyn) hv = (HZ[tid * W + i] & ~(1ull << 63)) + 1;
        }
        H64[tid * W + i] = hv;
      }
      __syncthreads();
      uint32_t m = 0;
      if (emit_blk) {
        for (int i = 0; i < W; i++) {
          const int j = tid * W + i;
          const uint64_t hj = H64[j];
          if (hj == 0) continue;
          int lo = j, hi = j;
          while (lo > 0 && lo > j - (W - 1) && H64[lo - 1] != 0 && sjob[(lo - 1) / W] == J) --lo;
          while (hi + 1 < POS && hi < j + (W - 1) && H64[hi + 1] != 0 && sjob[(hi + 1) / W] == J) ++hi;
          bool s = false;
          if (hi - lo + 1 < W) {
            uint64_t mn = ~0ull;
            for (int q = lo; q <= hi; q++) mn = min(mn, H64[q]);
            s = (hj == mn);
          } else {
            const int a0 = max(lo, j - (W - 1)), a1 = min(j, hi - (W - 1));
            for (int st = a0; st <= a1 && !s; st++) {
              uint64_t mn = ~0ull;
              for (int q = st; q < st + W; q++) mn = min(mn, H64[q]);
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
    }
    if (!emit_blk) selmask = 0;

    // ------------------------------------------------------------------ E. output
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
    if constexpr (ORDERED) {
      // publish this tile's count, then write the PREVIOUS tile's records: its predecessors had a whole
      // tile's time to publish theirs, so the look-back rarely waits
      if (tid == 0) lb_publish(a.status, tile, total);
      if (p_tile >= 0) {
        if (wid == 0) resolve_pending();
        __syncthreads();
        write_pending();
      }
      p_tile = tile;
      p_total = total;
      p_sel = selmask;
      p_rank = before + incl - cnt;
      p_pb = sjp[J - j0] + pat_off_u<PP, PX>(l0);
      p_r0 = l0 % PX;
      p_J = J;
      p_start = emit_blk && l0 == 0;
      p_hz = HZ;
      HZ = (HZ == HZ0) ? HZ0 + POS : HZ0;
      continue;
    }
    if (a.tile_cnt) {
      if (tid == 0) {
        s_base = (uint64_t)tile * X2_CAP;
        a.tile_cnt[tile] = total <= (uint32_t)X2_CAP ? total : 0u;
        if (total > (uint32_t)X2_CAP) *a.overflow = 1u;
      }
      if (total > (uint32_t)X2_CAP) {  // (uniform) nothing is written: the caller falls back
        __syncthreads();
        continue;
      }
    } else if (tid == 0) {
      s_base = atomicAdd(reinterpret_cast<unsigned long long*>(a.total_out), (unsigned long long)total);
    }
    uint32_t rank = before + incl - cnt;
    if (total <= (uint32_t)X2_CAP && !a.out_job) {
      // stage the tile-local indices of the selected positions (u16, position order), then one
      // coalesced copy that reads each record's hash from HZ and computes its position from its
      // block's base (a predicated staging of full records cost ~13 slots per position, measured)
      SBASE[tid] = sjp[J - j0] + pat_off_u<PP, PX>(l0);
      if (PX > 1) SR0[tid] = (uint8_t)(l0 % PX);
      uint32_t m = selmask;
      while (m) {
        const int i = __ffs(m) - 1;
        m &= m - 1;
        GOD_DCHECK(rank < (uint32_t)X2_CAP, "K1 staging index");
        SIDX[rank++] = (uint16_t)(tid * W + i);
      }
      __syncthreads();
      const uint64_t base = s_base;
      GOD_DCHECK(!emit_blk || J < a.n_jobs, "K1 job index");
      if (a.job_off && emit_blk && l0 == 0) a.job_off[J] = base + before + incl - cnt;
      // aligned tiles: the last block of each job records the job's end (jobs lie in one tile)
      if (a.job_end && emit_blk && (tid + 1 >= tile_nb || sjob[tid + 1] != J)) a.job_end[J] = base + before + incl;
      for (uint32_t r = tid; r < total; r += X2_NT) {
        const uint64_t gi = base + r;
        if (gi < a.cap) {
          const uint32_t e = SIDX[r], blk = e / W, o = e - blk * W;
          a.out_hz[gi] = HZ[e];
          a.out_pos[gi] = SBASE[blk] + pat_delta<PP, PX>(PX > 1 ? SR0[blk] : 0u, o);
        }
      }
      continue;
    }
    __syncthreads();
    uint64_t gi = s_base + rank;
    if (a.job_off && emit_blk && l0 == 0) a.job_off[J] = gi;
    if (a.job_end && emit_blk && (tid + 1 >= tile_nb || sjob[tid + 1] != J)) a.job_end[J] = gi + cnt;
    if (selmask) {
      const uint32_t pb = sjp[J - j0] + pat_off_u<PP, PX>(l0);
      const uint32_t r0 = l0 % PX;
      uint32_t m = selmask;
      while (m) {
        const int i = __ffs(m) - 1;
        m &= m - 1;
        if (gi < a.cap) {
          a.out_hz[gi] = HZ[tid * W + i];
          a.out_pos[gi] = pb + pat_delta<PP, PX>(r0, (uint32_t)i);
          if (a.out_job) a.out_job[gi] = J;
        }
        ++gi;
      }
    }
  }
  if constexpr (ORDERED) {
    if (p_tile >= 0) {
      if (wid == 0) resolve_pending();
      __syncthreads();
      write_pending();
    }
  }
}

// per-tile descriptors: first and last job (binary searches over the padded bases), the tile's
// code-word range, and whether it is a single job whose bytes can be read unchecked
__global__ void k_x2_tile_desc(const uint64_t* __restrict__ kb, const uint64_t* __restrict__ cw,
                               const Job* __restrict__ jobs, uint32_t n_jobs, uint64_t total_blocks, int W, int NB,
                               int maxwords, int PP, int PX, uint32_t one0, uint64_t seq_bytes, uint64_t ntiles,
                               X2Desc* desc, const uint8_t* seq) {
  const int NL = pack_words_rt(PP, PX);
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
    // bytes touched: job j's words [max(cw_j, lo), min(cw_j+1, hi)) end at base 16 (wend - cw_j) at
    // offset <= (q / x + 1) p, plus the load width.  Every job of the tile is checked: jobs need not be
    // in sequence-buffer order (seeding's dedicated extraction takes an arbitrary read list; the checked
    // build caught the round-1 "last job ends last" shortcut reading past the buffer there)
    uint64_t last_byte = 0, sp_lo = ~0ull, sp_hi = 0;
    for (uint32_t j = j0; j <= j1; j++) {
      const uint64_t wend = cw[j + 1] < hi ? cw[j + 1] : hi;
      if (wend <= cw[j] || wend <= lo) continue;
      const Job jj = jobs[j];
      const uint64_t lb = jj.seq_off + jj.phase + one0 + (16 * (wend - cw[j]) / PX + 1) * PP + 48;
      last_byte = lb > last_byte ? lb : last_byte;
      const uint64_t wst = cw[j] > lo ? cw[j] : lo;
      uint64_t a, b;
      job_byte_span(jj.seq_off + jj.phase + one0, wst - cw[j], wend - cw[j], PP, PX, NL, a, b);
      sp_lo = a < sp_lo ? a : sp_lo;
      sp_hi = b > sp_hi ? b : sp_hi;
    }
    X2Desc d;
    d.j0 = j0;
    d.j1 = j1;
    d.simple = (j0 == j1) && last_byte <= seq_bytes;
    d.safe = last_byte <= seq_bytes;
    d.b0 = 0;
    d.nb = 0;
    d.need = tile_need(last_byte, sp_hi, seq_bytes);
    raw_span(seq, seq_bytes, sp_lo, sp_hi, d.raw_lo, d.raw_len);
    d.cw_lo = lo;
    d.cw_hi = hi;
    desc[t] = d;
  }
}

// job-aligned tiles (every job <= 129 - S blocks): tile t starts at the first job whose first block
// is >= t * S and ends where tile t + 1 starts, so it holds whole jobs and at most 128 blocks
__global__ void k_x2_tile_desc_aligned(const uint64_t* __restrict__ kb, const uint64_t* __restrict__ cw,
                                       const Job* __restrict__ jobs, uint32_t n_jobs, int W, uint32_t S, int PP,
                                       int PX, uint32_t one0, uint64_t seq_bytes, uint64_t ntiles, X2Desc* desc,
                                       const uint8_t* seq) {
  const int NL = pack_words_rt(PP, PX);
  auto first_job_at = [&](uint64_t g) -> uint32_t {  // smallest j with kb[j] >= g (n_jobs if none)
    uint32_t lo = 0, hi = n_jobs;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (kb[mid] < g) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntiles; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j0 = first_job_at(t * S * (uint64_t)W);
    const uint32_t je = first_job_at((t + 1) * S * (uint64_t)W);  // first job of the next tile
    X2Desc d;
    d.j0 = j0 < n_jobs ? j0 : n_jobs - 1;
    d.j1 = je > j0 ? je - 1 : d.j0;
    d.b0 = kb[j0 < n_jobs ? j0 : n_jobs] / W;
    d.nb = je > j0 ? (uint32_t)((kb[je] - kb[j0]) / W) : 0u;
    d.need = seq_bytes;  // (aligned tiles are never streamed)
    d.cw_lo = cw[d.j0];
    d.cw_hi = je > j0 ? cw[je] : cw[d.j0];
    uint64_t last_l = 0, sp_lo = ~0ull, sp_hi = 0;  // every job (jobs need not be in buffer order)
    for (uint32_t j = d.j0; je > j0 && j <= d.j1; j++) {
      if (cw[j + 1] <= cw[j]) continue;
      const Job jj = jobs[j];
      const uint64_t lb = jj.seq_off + jj.phase + one0 + (16 * (cw[j + 1] - cw[j]) / PX + 1) * PP + 48;
      last_l = lb > last_l ? lb : last_l;
      uint64_t a, b;
      job_byte_span(jj.seq_off + jj.phase + one0, 0, cw[j + 1] - cw[j], PP, PX, NL, a, b);
      sp_lo = a < sp_lo ? a : sp_lo;
      sp_hi = b > sp_hi ? b : sp_hi;
    }
    raw_span(seq, seq_bytes, sp_lo, sp_hi, d.raw_lo, d.raw_len);
    d.simple = (d.j0 == d.j1) && last_l <= seq_bytes;
    d.safe = last_l <= seq_bytes;
    desc[t] = d;
  }
}

// padded position bases (multiple of W) and code-word bases per job
__global__ void k_x2_sizes(const Job* __restrict__ jobs, uint32_t n, int K, int W, uint64_t* kb, uint64_t* cw,
                           unsigned long long* nk_sum) {
  uint64_t acc = 0, mxb = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint64_t nk = jobs[j].nk;
    kb[j] = (nk ? (nk + W - 1) / W : 1) * W;  // no separator: job boundaries are handled in-kernel
    const uint64_t ncode = nk ? nk + K - 1 : 0;
    cw[j] = (ncode + 15) / 16;
    acc += nk;
    mxb = max(mxb, kb[j] / W);
  }
  for (int d = 16; d; d >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, d);
    mxb = max(mxb, __shfl_xor_sync(0xffffffffu, mxb, d));
  }
  __shared__ unsigned long long s_mx, s_acc;  // one global atomic per CTA on each word
  if (threadIdx.x == 0) { s_mx = 0; s_acc = 0; }
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && mxb) atomicMax(&s_mx, (unsigned long long)mxb);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&s_acc, (unsigned long long)acc);
  __syncthreads();
  if (threadIdx.x == 0 && s_mx) atomicMax(nk_sum + 1, s_mx);
  if (threadIdx.x == 0 && s_acc) atomicAdd(nk_sum, s_acc);
}

// slotted output -> contiguous: one warp per tile copies its records to the tile's scanned offset
__global__ void k_x2_compact(const uint64_t* __restrict__ shz, const uint32_t* __restrict__ spos,
                             const uint32_t* __restrict__ tile_cnt, const uint64_t* __restrict__ toff, uint64_t ntiles,
                             uint64_t* __restrict__ hz, uint32_t* __restrict__ pos) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32; t < ntiles;
       t += (uint64_t)gridDim.x * blockDim.x / 32) {
    const uint32_t c = tile_cnt[t];
    const uint64_t src = t * X2_CAP, dst = toff[t];
    for (uint32_t i = lane; i < c; i += 32) {
      hz[dst + i] = __ldcs(shz + src + i);
      pos[dst + i] = __ldcs(spos + src + i);
    }
  }
}
// a job's first record: slot coordinate (tile * X2_CAP + rank) -> index in the compacted records
__global__ void k_x2_job_off_fix(uint64_t* job_off, uint32_t n_jobs, const uint64_t* __restrict__ toff) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n_jobs; j += gridDim.x * blockDim.x) {
    const uint64_t v = job_off[j];
    job_off[j] = toff[v / X2_CAP] + v % X2_CAP;
  }
}

// Streamed input (SeqStream): first[i] = the first tile that reads past chunk i, i.e. tiles
// [first[i - 1], first[i]) can run once chunks 0..i are in.  first[] starts at ntiles; a tile whose last
// chunk is above its predecessor's lowers every boundary in between (need is nondecreasing in t for a
// reference's jobs, and the minimum stays right if it is not).  ctr[i] = the tile counter each range starts at.
__global__ void k_x2_stream_plan(const X2Desc* __restrict__ desc, uint64_t ntiles, uint64_t chunk_bytes, uint32_t S,
                                 uint32_t* first) {
  auto chunk_of = [&](uint64_t t) -> uint32_t {
    const uint64_t need = desc[t].need;
    const uint64_t c = need ? (need - 1) / chunk_bytes : 0;
    return (uint32_t)(c < S - 1 ? c : S - 1);
  };
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntiles; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = chunk_of(t), cp = t ? chunk_of(t - 1) : 0u;
    for (uint32_t i = cp; i < c; i++) atomicMin(&first[i], (uint32_t)t);
  }
}
__global__ void k_x2_stream_ctrs(uint32_t* first, uint32_t S, uint32_t ntiles, uint32_t* ctr) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // a dip in `need` must not start a later range before an earlier one: running minimum from the right
    uint32_t m = ntiles;
    first[S - 1] = ntiles;
    for (int i = (int)S - 1; i >= 0; i--) {
      m = first[i] < m ? first[i] : m;
      first[i] = m;
    }
    for (uint32_t i = 0; i < S; i++) ctr[i] = i ? first[i - 1] : 0u;
  }
}

template <int K, int W, int PP, int PX, bool ORDERED>
size_t x2_smem_bytes() {
  return X2Cfg<K, W, PP, PX>::smem(ORDERED);
}

// ntiles: the tiles this launch will claim (sizes the grid; a.ntiles is the end of its tile range)
template <int K, int W, int PP, int PX, bool ORDERED>
void launch_x3(const X2Args& a, uint64_t ntiles, cudaStream_t st, const char* tag) {
  static int grid[64] = {0};  // per device
  static DeviceOnce once;
  int dev = 0;
  GOD_CUDA(cudaGetDevice(&dev));
  const size_t smem = x2_smem_bytes<K, W, PP, PX, ORDERED>();
  once.run([&] {
    GOD_CUDA(cudaFuncSetAttribute(k_extract3<K, W, PP, PX, ORDERED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    int per_sm = 0;
    GOD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_extract3<K, W, PP, PX, ORDERED>, X2_NT, smem));
    grid[dev & 63] = (per_sm > 0 ? per_sm : 1) * num_sms();
  });
  const int g0 = grid[dev & 63];
  const unsigned g = (unsigned)(ntiles < (uint64_t)g0 ? ntiles : (uint64_t)g0);
  GOD_LAUNCH(tag, (k_extract3<K, W, PP, PX, ORDERED>), g, X2_NT, smem, st, a);
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
                  uint64_t cap_hint, const char* tag, const X2Layout* x2, RecOrder order, const SeqStream* ss) {
  if (!x2_supported(P)) return false;
  const int PP = (int)P.pat.p, PX = (int)P.pat.x;
  const int K = P.k, W = P.w;
  rec.n = 0;
  if (n_jobs == 0) return false;
  // padded layouts (built by make_jobs in the same pass as the jobs, else here)
  const uint64_t* kb;
  const uint64_t* cw;
  uint64_t total_pos, nk_sum, max_jb;
  if (x2) {
    kb = x2->kb;
    cw = x2->cw;
    total_pos = x2->total_pos;
    nk_sum = x2->nk_sum;
    max_jb = x2->max_job_blocks;
  } else {
    uint64_t* kbw = scr.alloc<uint64_t>(n_jobs + 1);
    uint64_t* cww = scr.alloc<uint64_t>(n_jobs + 1);
    uint64_t* tot = scr.alloc<uint64_t>(4);
    GOD_CUDA(cudaMemsetAsync(tot + 2, 0, 2 * sizeof(uint64_t), st));
    GOD_LAUNCH("k_x2_sizes", k_x2_sizes, grid_for(n_jobs, 256), 256, 0, st, jobs, n_jobs, K, W, kbw, cww,
               reinterpret_cast<unsigned long long*>(tot + 2));
    scan_exclusive_u64(kbw, kbw, n_jobs, tot, st, scr, "scan_x2_jobs");
    scan_exclusive_u64(cww, cww, n_jobs, tot + 1, st, scr, "scan_x2_jobs");
    GOD_CUDA(cudaMemcpyAsync(kbw + n_jobs, tot, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    GOD_CUDA(cudaMemcpyAsync(cww + n_jobs, tot + 1, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    uint64_t htot[4];
    d2h_small(htot, tot, sizeof(htot), st);
    kb = kbw;
    cw = cww;
    total_pos = htot[0];
    nk_sum = htot[2];
    max_jb = htot[3];
  }
  prof_add_units(tag, nk_sum);
  const uint64_t total_blocks = total_pos / W;
  // Output order (RecOrder): ORDER_NONE -> tiles at atomically claimed offsets; ORDER_JOB with short jobs
  // -> job-aligned tiles at atomically claimed offsets (each job contiguous, in position order); else
  // position order through the decoupled look-back.  Unordered instances exist for 2k >= 36.
  const bool can_unordered = 2 * K >= 36 && !want_job && !getenv("GOD_X2_ORDERED");
  const bool aligned = can_unordered && order == ORDER_JOB && max_jb <= X2_NT / 4 && !getenv("GOD_X2_NO_ALIGN");
  // GOD_X2_FORCE_UNORDERED: developer timing aid (records of a multi-tile job are then NOT contiguous)
  const bool ordered = !(can_unordered && (order == ORDER_NONE || aligned || getenv("GOD_X2_FORCE_UNORDERED")));
  // a streamed input (SeqStream) is consumed chunk by chunk only by the unordered kernel over strided tiles
  const bool streamed = ss && !ss->arrived.empty() && ss->chunk_bytes && !ordered && !aligned;
  if (ss && !streamed) ss->wait_all(st);
  const uint32_t S_al = (uint32_t)(X2_NT + 1 - max_jb);  // tile stride (blocks) of the aligned layout
  const uint64_t ntiles = aligned ? (total_blocks + S_al - 1) / S_al : (total_blocks + X2_OUT_BLOCKS - 1) / X2_OUT_BLOCKS;
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
    if (aligned)
      GOD_LAUNCH("k_x2_tile_desc", k_x2_tile_desc_aligned, grid_for(ntiles, 256), 256, 0, st, kb, cw, jobs, n_jobs, W,
                 S_al, PP, PX, P.pat.one[0], seq_bytes, ntiles, desc, seq);
    else
      GOD_LAUNCH("k_x2_tile_desc", k_x2_tile_desc, grid_for(ntiles, 256), 256, 0, st, kb, cw, jobs, n_jobs, total_blocks,
                 W, NB, maxwords, PP, PX, P.pat.one[0], seq_bytes, ntiles, desc, seq);
  }
  uint64_t* dtotal = scr.alloc<uint64_t>(1);
  if (want_job_off) {
    rec.job_off = scr.alloc<uint64_t>(n_jobs + 1);
    // a job's end is the next job's start unless jobs are placed tile by tile (aligned)
    rec.job_end = aligned ? scr.alloc<uint64_t>(n_jobs) : rec.job_off + 1;
  }
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
    if (kbits > 0 && kbits < 2 * K) key_shift = std::min(2 * K - kbits, 31);  // keys of >= 2k - 31 bits
  }
  // launch the specialised kernel for (K, W, pattern); ordered_kernel: the look-back instance
  auto launch = [&](const X2Args& a, bool ordered_kernel, uint64_t count) {
    auto by_pattern = [&](auto kc, auto wc) {
      constexpr int KK = decltype(kc)::value, WW = decltype(wc)::value;
      auto go = [&](auto oc) {
        constexpr bool O = decltype(oc)::value;
        if (PX == 1 && PP == 1) launch_x3<KK, WW, 1, 1, O>(a, count, st, tag);
        else if (PX == 1 && PP == 2) launch_x3<KK, WW, 2, 1, O>(a, count, st, tag);
        else if (PX == 1) launch_x3<KK, WW, 3, 1, O>(a, count, st, tag);
        else if (PX == 2) launch_x3<KK, WW, 3, 2, O>(a, count, st, tag);
        else launch_x3<KK, WW, 4, 3, O>(a, count, st, tag);
      };
      if (!ordered_kernel) go(std::false_type());
      else go(std::true_type());
    };
    if (K == 21 && W == 11) by_pattern(std::integral_constant<int, 21>(), std::integral_constant<int, 11>());
    else if (K == 19 && W == 19) by_pattern(std::integral_constant<int, 19>(), std::integral_constant<int, 19>());
    else if (K == 19 && W == 16) by_pattern(std::integral_constant<int, 19>(), std::integral_constant<int, 16>());
    else by_pattern(std::integral_constant<int, 15>(), std::integral_constant<int, 10>());
  };
  // Position order for jobs that span tiles (long reads), without inter-CTA waiting: the unordered
  // kernel writes tile t's records at slot t * X2_CAP and its count; a scan of the counts and one copy
  // close the gaps.  (The look-back instance spent 56% of its stall samples waiting for predecessor
  // tiles on the HiFi reads: extract_seed 19.2 ms; measured, round 2.)
  if (ordered && !want_job && ntiles && !getenv("GOD_X2_NO_SLOTS")) {  // ORDER_JOB across tiles, ORDER_GLOBAL
    const uint64_t scap = ntiles * (uint64_t)X2_CAP;
    uint64_t* shz = scr.alloc<uint64_t>(scap);
    uint32_t* spos = scr.alloc<uint32_t>(scap);
    uint32_t* tile_cnt = scr.alloc<uint32_t>(ntiles);
    uint32_t* overflow = scr.alloc<uint32_t>(1);
    GOD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
    GOD_CUDA(cudaMemsetAsync(overflow, 0, sizeof(uint32_t), st));
    X2Args a{seq, seq_bytes, jobs, kb, cw, n_jobs, total_blocks, P.pat.one[0], key_shift, status, ctr,
             shz, spos, nullptr, rec.job_off, nullptr, scap, dtotal, dbg_flags,
             dbg_counts, desc, 0u, ntiles, getenv("GOD_X2_NO_STAGE") ? 1u : 0u, tile_cnt, overflow};
    launch(a, false, ntiles);
    const uint32_t over = d2h_scalar(overflow, st);
    if (getenv("GOD_DEBUG_SLOTS")) fprintf(stderr, "[x2] %s slotted tiles=%llu overflow=%u\n", tag, (unsigned long long)ntiles, over);
    if (over == 0) {
      uint64_t* toff = scr.alloc<uint64_t>(ntiles + 1);  // [ntiles] = the total (a job starting past the last record)
      scan_exclusive_u32_to_u64(tile_cnt, toff, ntiles, dtotal, st, scr, "scan_x2_tiles");
      GOD_CUDA(cudaMemcpyAsync(toff + ntiles, dtotal, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
      const uint64_t n = d2h_scalar(dtotal, st);
      rec.cap = n ? n : 1;
      rec.hz = scr.alloc<uint64_t>(rec.cap);
      rec.pos = scr.alloc<uint32_t>(rec.cap);
      rec.job = nullptr;
      GOD_LAUNCH("k_x2_compact", k_x2_compact, grid_for(ntiles * 32, 256), 256, 0, st, shz, spos, tile_cnt, toff, ntiles,
                 rec.hz, rec.pos);
      if (want_job_off) {
        GOD_LAUNCH("k_x2_job_off_fix", k_x2_job_off_fix, grid_for(n_jobs, 256), 256, 0, st, rec.job_off, n_jobs, toff);
        GOD_CUDA(cudaMemcpyAsync(rec.job_off + n_jobs, dtotal, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
      }
      rec.n = n;
      return true;
    }
    // a tile with more than X2_CAP minimizers (all-ties runs): the look-back kernel below
  }
  for (int attempt = 0; attempt < 2; attempt++) {
    rec.cap = cap;
    rec.hz = scr.alloc<uint64_t>(cap);
    rec.pos = scr.alloc<uint32_t>(cap);
    rec.job = want_job ? scr.alloc<uint32_t>(cap) : nullptr;
    GOD_CUDA(cudaMemsetAsync(status, 0, (ntiles + 1) * sizeof(uint64_t), st));
    GOD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
    GOD_CUDA(cudaMemsetAsync(dtotal, 0, sizeof(uint64_t), st));  // the unordered kernel's output counter
    X2Args a{seq, seq_bytes, jobs, kb, cw, n_jobs, total_blocks, P.pat.one[0], key_shift, status, ctr,
             rec.hz, rec.pos, rec.job, rec.job_off, aligned ? rec.job_end : nullptr, cap, dtotal, dbg_flags,
             dbg_counts, desc, aligned ? 1u : 0u, ntiles, getenv("GOD_X2_NO_STAGE") ? 1u : 0u, nullptr, nullptr};
    if (ntiles && streamed && attempt == 0) {
      // tiles [first[i - 1], first[i]) as soon as chunk i is in: one launch per chunk, each with its own
      // tile counter starting at the range's first tile; all append to the same output
      const uint32_t S = (uint32_t)ss->arrived.size();
      uint32_t* first = scr.alloc<uint32_t>(S);
      uint32_t* ctrs = scr.alloc<uint32_t>(S);
      GOD_CUDA(cudaMemsetAsync(first, 0xFF, S * sizeof(uint32_t), st));
      GOD_LAUNCH("k_x2_stream_plan", k_x2_stream_plan, grid_for(ntiles, 256), 256, 0, st, desc, ntiles, ss->chunk_bytes, S,
                 first);
      GOD_LAUNCH("k_x2_stream_plan", k_x2_stream_ctrs, 1, 32, 0, st, first, S, (uint32_t)ntiles, ctrs);
      std::vector<uint32_t> hf(S);
      d2h_small(hf.data(), first, S * sizeof(uint32_t), st);
      uint32_t prev = 0;
      for (uint32_t i = 0; i < S; i++) {
        GOD_CUDA(cudaStreamWaitEvent(st, ss->arrived[i], 0));
        if (hf[i] <= prev) continue;
        X2Args ai = a;
        ai.tile_ctr = ctrs + i;
        ai.ntiles = hf[i];
        launch(ai, false, hf[i] - prev);
        prev = hf[i];
      }
    } else if (ntiles) {
      launch(a, ordered, ntiles);
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
