// K1 core variants (round 2): the per-position core of the specialised minimizer kernel (k = 21,
// w = 11; see k1_floor.cu for the base variant), register-resident, with the arithmetic spread
// differently over the two integer pipes.  On Blackwell the alu pipe (LOP3/SHF/SEL/ISETP/IMNMX) and
// the fma pipe (IMAD) each take one warp instruction every 2 cycles per SMSP; the base variant issues
// ~30 alu and ~10 fma instructions per position, so it is alu-bound.  The variants move shifts onto
// the fma pipe: x >> s = mul.hi(x, 2^(32-s)), x << s = mul.lo(x, 2^s), disjoint or = add.  The
// multipliers come from kernel parameters so that ptxas cannot strength-reduce them back to shifts.
//   V0: base (two-word masked hash: mask + funnel + xor per xor-shift)
//   V1: xor-shifts and the key on the fma pipe (hi kept left-aligned as h22 = hi << 22)
//   V2: V1 + the k-mer hi words by mul.hi
//   V3: V2 + selection without the prefix-max pass (MM by a second van Herk on the fma pipe? no:
//       plain) -- reserved
// Also: raw pipe rates of IMAD, IMAD.HI, IMAD.WIDE, LOP3, VIMNMX (independent chains).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/k1_floor2 tools/k1_floor2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <type_traits>

constexpr int K = 21, W = 11, NB = W + K - 1, NWIN = (2 * NB + 31) / 32;
constexpr uint32_t HM = (1u << (2 * K - 32)) - 1;

struct Mul {  // opaque powers of two (and the hash multipliers)
  uint32_t p2[33];  // p2[s] = 2^s (p2[32] unused)
  uint32_t c21, c265, c21b, c31, one;
};

__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t madhi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t mullo(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t madlo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

__device__ __forceinline__ uint32_t rev2(uint32_t x) {
  const uint32_t y = __brev(x);
  return ((y >> 1) & 0x55555555u) | ((y & 0x55555555u) << 1);
}
__device__ __forceinline__ uint32_t ext32(const uint32_t (&w)[NWIN], int S) {
  const int i = S >> 5, o = S & 31;
  const uint32_t a = i < NWIN ? w[i] : 0u, b = i + 1 < NWIN ? w[i + 1] : 0u;
  return o ? __funnelshift_l(b, a, o) : a;
}

// V0 hash
__device__ __forceinline__ void wang0(uint32_t& hi, uint32_t& lo) {
  auto mul = [&](uint32_t c) {
    const uint64_t p = (uint64_t)lo * c;
    hi = hi * c + (uint32_t)(p >> 32);
    lo = (uint32_t)p;
  };
  {
    const uint64_t p = (uint64_t)lo * ((1u << 21) - 1) + ~0ull;
    hi = hi * ((1u << 21) - 1) + (uint32_t)(p >> 32);
    lo = (uint32_t)p;
  }
  hi &= HM; lo ^= __funnelshift_r(lo, hi, 24);
  mul(265u);
  hi &= HM; lo ^= __funnelshift_r(lo, hi, 14);
  mul(21u);
  hi &= HM; lo ^= __funnelshift_r(lo, hi, 28);
  mul(0x80000001u);
  hi &= HM;
}

// V1 hash: returns lo and h22 = (hash >> 32) << 22 (the 10 hi bits left-aligned, zeros below)
__device__ __forceinline__ void wang1(uint32_t hi, uint32_t lo, const Mul& M, uint32_t& olo, uint32_t& oh22) {
  // x1 = (2^21 - 1) x - 1
  uint64_t p = (uint64_t)lo * M.c21 + ~0ull;
  hi = madlo(hi, M.c21, (uint32_t)(p >> 32));
  lo = (uint32_t)p;
  auto xs = [&](int s) {  // lo ^= (lo >> s) | (hi_clean << (32 - s)), s >= 10
    const uint32_t h22 = mullo(hi, M.p2[22]);
    const uint32_t t = madhi(lo, M.p2[32 - s], mulhi(h22, M.p2[42 - s]));
    lo ^= t;
  };
  auto mul = [&](uint32_t c) {
    const uint64_t q = (uint64_t)lo * c;
    hi = madlo(hi, c, (uint32_t)(q >> 32));
    lo = (uint32_t)q;
  };
  xs(24);
  mul(M.c265);
  xs(14);
  mul(M.c21b);
  xs(28);
  mul(M.c31);
  olo = lo;
  oh22 = mullo(hi, M.p2[22]);
}

template <int V, bool TIE = false, bool STORE = false>
__global__ void __launch_bounds__(128, 8) k_core(uint32_t iters, uint32_t seed, unsigned long long* out, Mul M) {
  __shared__ uint64_t HZ[128 * W];
  uint32_t st = (blockIdx.x * 128 + threadIdx.x) * 0x9E3779B9u ^ seed;
  uint64_t acc = 0;
  uint32_t hacc = 0;
  const int lane = threadIdx.x & 31;
  for (uint32_t it = 0; it < iters; it++) {
    uint32_t win[NWIN], rcw[NWIN];
#pragma unroll
    for (int i = 0; i < NWIN; i++) {
      st ^= st << 13; st ^= st >> 17; st ^= st << 5;
      win[i] = st;
    }
#pragma unroll
    for (int i = 0; i < NWIN; i++) rcw[i] = ~rev2(win[NWIN - 1 - i]);
    constexpr int PADB = 32 * NWIN - 2 * NB;
    uint32_t key[W];
#pragma unroll
    for (int i = 0; i < W; i++) {
      const int SR = PADB + 2 * (NB - K - i);
      if constexpr (V == 0) {
        const uint32_t fl = ext32(win, 2 * i + 10), fh = ext32(win, 2 * i) >> 22;
        const uint32_t rl = ext32(rcw, SR + 10), rh = ext32(rcw, SR) >> 22;
        const bool z = (((uint64_t)fh << 32) | fl) > (((uint64_t)rh << 32) | rl);
        uint32_t hi = z ? rh : fh, lo = z ? rl : fl;
        wang0(hi, lo);
        hacc ^= hi | (z ? 0x80000000u : 0u);
        key[i] = __funnelshift_r(lo, hi, 11) + 1u;
      } else {
        uint32_t fl = ext32(win, 2 * i + 10), rl = ext32(rcw, SR + 10);
        uint32_t fh, rh;
        if constexpr (V == 1) {
          fh = ext32(win, 2 * i) >> 22;
          rh = ext32(rcw, SR) >> 22;
        } else {
          fh = mulhi(ext32(win, 2 * i), M.p2[10]);
          rh = mulhi(ext32(rcw, SR), M.p2[10]);
        }
        const bool z = (((uint64_t)fh << 32) | fl) > (((uint64_t)rh << 32) | rl);
        const uint32_t hi = z ? rh : fh, lo = z ? rl : fl;
        uint32_t olo, h22;
        wang1(hi, lo, M, olo, h22);
        const uint32_t hz_hi = madlo((uint32_t)z, M.p2[31], mulhi(h22, M.p2[10]));
        if constexpr (STORE) HZ[threadIdx.x * W + i] = ((uint64_t)hz_hi << 32) | olo;
        else hacc ^= hz_hi;
        key[i] = madhi(olo, M.p2[21], madhi(h22, M.p2[31], M.one));
      }
    }
    uint32_t PF[W], SF[W];
    PF[0] = key[0];
#pragma unroll
    for (int i = 1; i < W; i++) PF[i] = min(PF[i - 1], key[i]);
    SF[W - 1] = key[W - 1];
#pragma unroll
    for (int i = W - 2; i >= 0; i--) SF[i] = min(SF[i + 1], key[i]);
    uint32_t WM[W];
    WM[0] = SF[0];
#pragma unroll
    for (int i = 1; i < W; i++) {
      const uint32_t nx = __shfl_down_sync(0xffffffffu, PF[i - 1], 1);
      WM[i] = min(SF[i], lane < 31 ? nx : 0u);
    }
    uint32_t PX[W], SX[W];
    PX[0] = WM[0];
#pragma unroll
    for (int i = 1; i < W; i++) PX[i] = max(PX[i - 1], WM[i]);
    SX[W - 1] = WM[W - 1];
#pragma unroll
    for (int i = W - 2; i >= 0; i--) SX[i] = max(SX[i + 1], WM[i]);
    uint32_t sel = 0;
    bool tie = false;
    uint32_t prevk = 0;
#pragma unroll
    for (int o = 0; o < W; o++) {
      const uint32_t p = __shfl_up_sync(0xffffffffu, SX[o < W - 1 ? o + 1 : o], 1);
      const uint32_t mm = o == W - 1 ? PX[W - 1] : max(lane ? p : 0u, PX[o]);
      const bool s = key[o] == mm;
      sel |= (uint32_t)s << o;
      if constexpr (TIE) {
        tie |= s & (key[o] == prevk);
        prevk = s ? key[o] : prevk;
      }
    }
    acc += __popc(sel) + (tie ? 1 : 0);
    if constexpr (STORE) {
      __syncwarp();
      if (sel) hacc ^= (uint32_t)HZ[threadIdx.x * W + __ffs(sel) - 1];
      __syncwarp();
    }
  }
  if (acc == 0x12345678ull || hacc == 0x9u) out[0] = acc;  // keeps the work live
  atomicAdd(out + 1, acc);
}

// raw pipe rates: 8 independent chains per thread of one op kind
template <int OP>
__global__ void __launch_bounds__(128, 8) k_pipe(uint32_t iters, uint32_t seed, unsigned long long* out, Mul M) {
  uint32_t x[8];
#pragma unroll
  for (int j = 0; j < 8; j++) x[j] = (threadIdx.x + 1) * (j + 3) ^ seed;
  const uint32_t c = M.c265, d = M.p2[7];
  for (uint32_t it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int j = 0; j < 8; j++) {
        if constexpr (OP == 0) x[j] = madlo(x[j], c, d);                  // IMAD
        else if constexpr (OP == 1) x[j] = madhi(x[j], c, d);             // IMAD.HI
        else if constexpr (OP == 2) {                                      // IMAD.WIDE
          const uint64_t p = (uint64_t)x[j] * c + d;
          x[j] = (uint32_t)p ^ (uint32_t)(p >> 32);
        } else if constexpr (OP == 3) x[j] = (x[j] ^ c) & (x[j] | d);     // LOP3
        else if constexpr (OP == 4) x[j] = min(x[j] + 0u, c) ^ d;         // IMNMX (+ lop)
        else x[j] = __funnelshift_r(x[j], d, 7);                           // SHF
      }
  }
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s ^= x[j];
  if (s == 0x12345u) out[0] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  Mul M;
  for (int s = 0; s < 32; s++) M.p2[s] = 1u << s;
  M.p2[32] = 0;
  M.c21 = (1u << 21) - 1;
  M.c265 = 265u;
  M.c21b = 21u;
  M.c31 = 0x80000001u;
  M.one = 1u;
  const int blocks = sms * 8;
  const uint32_t iters = 4096;
  const double pos = (double)blocks * 128 * iters * W;
  unsigned long long sel[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto core = [&](auto vc, auto tc, auto sc) {
    constexpr int V = decltype(vc)::value;
    constexpr bool TIE = decltype(tc)::value, STORE = decltype(sc)::value;
    cudaMemset(d, 0, 16);
    const float ms = time_it([&] { k_core<V, TIE, STORE><<<blocks, 128>>>(iters, 7, d, M); });
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    if (!TIE && !STORE) sel[V] = h[1];
    const double per_s = pos / (ms * 1e-3);
    const double slots = (double)sms * 4 * 1.965e9 * 32 / per_s;  // thread slots per position at 1965 MHz
    printf("{\"bench\":\"k1_core\",\"tie\":%d,\"store\":%d,\"variant\":%d,\"ms\":%.3f,\"g_positions_per_s\":%.2f,\"human10_ms\":%.3f,"
           "\"thread_slots_per_position_at_1965\":%.1f,\"selected\":%llu}\n",
           (int)TIE, (int)STORE, V, ms, per_s / 1e9, 1.55e9 / per_s * 1e3, slots, h[1]);
  };
  using F = std::false_type;
  using T = std::true_type;
  core(std::integral_constant<int, 0>(), F(), F());
  core(std::integral_constant<int, 1>(), F(), F());
  core(std::integral_constant<int, 2>(), F(), F());
  core(std::integral_constant<int, 2>(), T(), F());
  core(std::integral_constant<int, 2>(), F(), T());
  core(std::integral_constant<int, 2>(), T(), T());
  printf("{\"bench\":\"k1_core_agree\",\"same_selection\":%s}\n", (sel[0] == sel[1] && sel[1] == sel[2]) ? "true" : "false");
  const char* names[6] = {"IMAD", "IMAD.HI", "IMAD.WIDE+LOP3", "LOP3x2", "IMNMX+LOP3", "SHF"};
  auto pipe = [&](auto oc) {
    constexpr int OP = decltype(oc)::value;
    const uint32_t it2 = 2048;
    const float ms = time_it([&] { k_pipe<OP><<<blocks, 128>>>(it2, 3, d, M); });
    const double ops = (double)blocks * 128 * it2 * 16 * 8;  // thread-ops of the chain step
    const double per_smsp_clk = ops / 32 / (ms * 1e-3) / (sms * 4) / 1.965e9;
    printf("{\"bench\":\"pipe\",\"op\":\"%s\",\"ms\":%.3f,\"warp_steps_per_smsp_clk\":%.3f}\n", names[OP], ms, per_smsp_clk);
  };
  pipe(std::integral_constant<int, 0>());
  pipe(std::integral_constant<int, 1>());
  pipe(std::integral_constant<int, 2>());
  pipe(std::integral_constant<int, 3>());
  pipe(std::integral_constant<int, 4>());
  pipe(std::integral_constant<int, 5>());
  printf("{\"error\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
