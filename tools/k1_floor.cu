// K1 compute floor (round 2): the per-position core of the specialised minimizer kernel with
// nothing else around it — register-resident code words (synthetic, from a counter-based mix of the
// thread id: no loads), k-mer + reverse complement by funnel shifts, canonical by one 64-bit compare,
// the two-word masked Wang hash (k = 21: hi holds 10 bits), key = top 31 bits + 1, then the van
// Herk window selection on 32-bit keys with the cross-block values by warp shuffles (w = 11, block
// = w positions per thread) and a count of selected positions (kept live by a sum).  No sparsify,
// no SMEM staging, no output, no tie check, no job logic.  Measures positions/s on all SMs and reports
// the time this floor implies for the human '10' extraction (1.55 G positions).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/k1_floor tools/k1_floor.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int K = 21, W = 11, NB = W + K - 1, NWIN = (2 * NB + 31) / 32;
constexpr uint32_t HM = (1u << (2 * K - 32)) - 1;

__device__ __forceinline__ uint32_t rev2(uint32_t x) {
  const uint32_t y = __brev(x);
  return ((y >> 1) & 0x55555555u) | ((y & 0x55555555u) << 1);
}
__device__ __forceinline__ uint32_t ext32(const uint32_t (&w)[NWIN], int S) {
  const int i = S >> 5, o = S & 31;
  const uint32_t a = i < NWIN ? w[i] : 0u, b = i + 1 < NWIN ? w[i + 1] : 0u;
  return o ? __funnelshift_l(b, a, o) : a;
}
__device__ __forceinline__ void wang(uint32_t& hi, uint32_t& lo) {
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

__global__ void __launch_bounds__(128, 8) k_floor(uint32_t iters, uint32_t seed, unsigned long long* out) {
  uint32_t st = (blockIdx.x * 128 + threadIdx.x) * 0x9E3779B9u ^ seed;
  uint64_t acc = 0;
  const int lane = threadIdx.x & 31;
  for (uint32_t it = 0; it < iters; it++) {
    uint32_t win[NWIN], rcw[NWIN];
#pragma unroll
    for (int i = 0; i < NWIN; i++) {  // a fresh window per iteration (xorshift: a few ops per word)
      st ^= st << 13; st ^= st >> 17; st ^= st << 5;
      win[i] = st;
    }
#pragma unroll
    for (int i = 0; i < NWIN; i++) rcw[i] = ~rev2(win[NWIN - 1 - i]);
    constexpr int PADB = 32 * NWIN - 2 * NB;
    uint32_t key[W];
#pragma unroll
    for (int i = 0; i < W; i++) {
      const uint32_t fl = ext32(win, 2 * i + 10), fh = ext32(win, 2 * i) >> 22;
      const uint32_t rl = ext32(rcw, PADB + 2 * (NB - K - i) + 10), rh = ext32(rcw, PADB + 2 * (NB - K - i)) >> 22;
      const bool z = (((uint64_t)fh << 32) | fl) > (((uint64_t)rh << 32) | rl);
      uint32_t hi = z ? rh : fh, lo = z ? rl : fl;
      wang(hi, lo);
      key[i] = __funnelshift_r(lo, hi, 11) + 1u;
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
#pragma unroll
    for (int o = 0; o < W; o++) {
      const uint32_t p = __shfl_up_sync(0xffffffffu, SX[o < W - 1 ? o + 1 : o], 1);
      const uint32_t mm = o == W - 1 ? PX[W - 1] : max(lane ? p : 0u, PX[o]);
      sel |= (uint32_t)(key[o] == mm) << o;
    }
    acc += __popc(sel);
  }
  if (acc == 0x12345678ull) out[0] = acc;  // keeps the work live
  atomicAdd(out + 1, acc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  const int blocks = sms * 8;
  const uint32_t iters = 4096;
  k_floor<<<blocks, 128>>>(16, 1, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a);
    k_floor<<<blocks, 128>>>(iters, 7 + r, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double pos = (double)blocks * 128 * iters * W;
  const double per_s = pos / (best * 1e-3);
  printf("{\"bench\":\"k1_compute_floor\",\"k\":%d,\"w\":%d,\"positions\":%.0f,\"ms\":%.3f,\"g_positions_per_s\":%.2f,"
         "\"human10_floor_ms\":%.3f,\"selected_frac\":%.4f,\"error\":\"%s\"}\n",
         K, W, pos, best, per_s / 1e9, 1.55e9 / per_s * 1e3, (double)h[1] / (pos * 6), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
