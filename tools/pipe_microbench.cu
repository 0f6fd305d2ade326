// Pipe microbenchmarks for the K1 / index-sort design (round 2): per-SM throughput of the
// instructions the new kernels lean on.  Standalone; not part of libgod.
//   DMNMX / DSETP  (fp64 pipe: exact 52-bit-mantissa keys for the window minimum)
//   IMNMX, SHF, LOP3 (alu pipe), IMAD, IMAD.WIDE.U32 (fma pipe), SHFL
//   global atomicAdd to random counters (65 K / 4 M), scattered 8-B stores into 65 K bins
// Output: one JSON line per benchmark: warp instructions per SM per clock (at the clock measured with
// clock64 on the device) — 4.0 = one per SMSP per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
#define CHAINS 8

__global__ void k_dmnmx(double seed, double* out) {
  double x[CHAINS], y[CHAINS];
#pragma unroll
  for (int u = 0; u < CHAINS; u++) { x[u] = seed * (threadIdx.x + u); y[u] = seed * (blockIdx.x - u); }
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int u = 0; u < CHAINS; u++) { x[u] = fmin(x[u], y[u]); y[u] = fmax(y[u], x[u] + 0.0); }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < CHAINS; u++) s += x[u] + y[u];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dsetp(double seed, uint32_t* out) {
  double x[CHAINS];
  uint32_t m = 0;
#pragma unroll
  for (int u = 0; u < CHAINS; u++) x[u] = seed * (threadIdx.x + u);
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int u = 0; u < CHAINS; u++) m += (x[u] == x[(u + 1) % CHAINS]) ? 1u : 0u;
#pragma unroll
    for (int u = 0; u < CHAINS; u++) x[u] = fmin(x[u], x[(u + 3) % CHAINS]);
  }
  if (m == 77) out[0] = m;
}
__global__ void k_imnmx(uint32_t seed, uint32_t* out) {
  uint32_t x[CHAINS], y[CHAINS];
#pragma unroll
  for (int u = 0; u < CHAINS; u++) { x[u] = seed ^ (threadIdx.x * 77 + u); y[u] = seed + blockIdx.x * 13 + u; }
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int u = 0; u < CHAINS; u++) { x[u] = min(x[u], y[u]); y[u] = max(y[u], x[u]); }
  }
  uint32_t s = 0;
#pragma unroll
  for (int u = 0; u < CHAINS; u++) s ^= x[u] + y[u];
  if (s == 0x1234567u) out[0] = s;
}
__global__ void k_imad_wide(uint32_t seed, uint32_t* out) {
  uint64_t x[CHAINS];
#pragma unroll
  for (int u = 0; u < CHAINS; u++) x[u] = seed ^ (threadIdx.x * 77 + u);
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int u = 0; u < CHAINS; u++) x[u] = (uint64_t)(uint32_t)x[u] * 265u + (x[u] >> 32);
  }
  uint64_t s = 0;
#pragma unroll
  for (int u = 0; u < CHAINS; u++) s ^= x[u];
  if (s == 0x1234567u) out[0] = (uint32_t)s;
}
__global__ void k_imad(uint32_t seed, uint32_t* out) {
  uint32_t x[CHAINS];
#pragma unroll
  for (int u = 0; u < CHAINS; u++) x[u] = seed ^ (threadIdx.x * 77 + u);
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int u = 0; u < CHAINS; u++) x[u] = x[u] * 265u + seed;
  }
  uint32_t s = 0;
#pragma unroll
  for (int u = 0; u < CHAINS; u++) s ^= x[u];
  if (s == 0x1234567u) out[0] = s;
}
__global__ void k_shf(uint32_t seed, uint32_t* out) {
  uint32_t x[CHAINS], y[CHAINS];
#pragma unroll
  for (int u = 0; u < CHAINS; u++) { x[u] = seed ^ (threadIdx.x * 77 + u); y[u] = seed + u; }
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int u = 0; u < CHAINS; u++) { x[u] = __funnelshift_r(x[u], y[u], 7); y[u] = __funnelshift_l(y[u], x[u], 3); }
  }
  uint32_t s = 0;
#pragma unroll
  for (int u = 0; u < CHAINS; u++) s ^= x[u] + y[u];
  if (s == 0x1234567u) out[0] = s;
}
__global__ void k_shfl(uint32_t seed, uint32_t* out) {
  uint32_t x[CHAINS];
#pragma unroll
  for (int u = 0; u < CHAINS; u++) x[u] = seed ^ (threadIdx.x * 77 + u);
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int u = 0; u < CHAINS; u++) x[u] = __shfl_down_sync(0xffffffffu, x[u], 1);
  }
  uint32_t s = 0;
#pragma unroll
  for (int u = 0; u < CHAINS; u++) s ^= x[u];
  if (s == 0x1234567u) out[0] = s;
}
__global__ void k_clock(unsigned long long* out) {
  if (threadIdx.x == 0) {
    const unsigned long long a = clock64();
    unsigned long long t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned long long t1 = t0;
    while (t1 - t0 < 20000000ull) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[0] = clock64() - a;
    out[1] = t1 - t0;
  }
}
__global__ void k_atomics(uint32_t* ctr, uint32_t nctr_mask, uint64_t n, uint32_t* sink) {
  uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    acc += atomicAdd(&ctr[(uint32_t)(x >> 20) & nctr_mask], 1u);
  }
  if (acc == 0x7777777u) sink[0] = acc;
}
__global__ void k_scatter(uint32_t* ctr, uint32_t nbins_mask, uint32_t bin_cap, uint64_t n, uint64_t* dst) {
  uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const uint32_t b = (uint32_t)(x >> 20) & nbins_mask;
    const uint32_t slot = atomicAdd(&ctr[b], 1u);
    if (slot < bin_cap) dst[(uint64_t)b * bin_cap + slot] = x;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* dclk;
  cudaMalloc(&dclk, 16);
  k_clock<<<1, 32>>>(dclk);
  unsigned long long hclk[2];
  cudaMemcpy(hclk, dclk, 16, cudaMemcpyDeviceToHost);
  const double ghz = (double)hclk[0] / (double)hclk[1];
  printf("{\"bench\":\"clock\",\"sm_ghz\":%.3f,\"sms\":%d}\n", ghz, sms);
  uint32_t* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8;
  auto report = [&](const char* name, float ms, double warp_instr) {
    const double per_sm_clk = warp_instr / (ms * 1e-3) / sms / (ghz * 1e9);
    printf("{\"bench\":\"%s\",\"warp_instr_per_sm_per_clk\":%.3f,\"ms\":%.3f}\n", name, per_sm_clk, ms);
  };
  const double warps = (double)blocks * threads / 32;
#define RUN(name, call, per_iter)                                     \
  do {                                                                \
    call;                                                             \
    cudaEventRecord(e0);                                              \
    call;                                                             \
    cudaEventRecord(e1);                                              \
    cudaEventSynchronize(e1);                                         \
    float ms;                                                         \
    cudaEventElapsedTime(&ms, e0, e1);                                \
    report(name, ms, warps * ITERS * (per_iter));                     \
  } while (0)
  RUN("dmnmx", (k_dmnmx<<<blocks, threads>>>(1.5, (double*)out)), 2.0 * CHAINS);
  RUN("dsetp+dmnmx", (k_dsetp<<<blocks, threads>>>(1.5, out)), 2.0 * CHAINS);
  RUN("imnmx", (k_imnmx<<<blocks, threads>>>(7u, out)), 2.0 * CHAINS);
  RUN("imad_wide_u32", (k_imad_wide<<<blocks, threads>>>(7u, out)), 1.0 * CHAINS);
  RUN("imad", (k_imad<<<blocks, threads>>>(7u, out)), 1.0 * CHAINS);
  RUN("shf", (k_shf<<<blocks, threads>>>(7u, out)), 2.0 * CHAINS);
  RUN("shfl", (k_shfl<<<blocks, threads>>>(7u, out)), 1.0 * CHAINS);
  // atomics and scatter
  for (uint32_t nctr : {1u << 12, 1u << 16, 1u << 22}) {
    uint32_t* ctr;
    cudaMalloc(&ctr, (size_t)nctr * 4);
    cudaMemset(ctr, 0, (size_t)nctr * 4);
    const uint64_t n = 256ull << 20;
    k_atomics<<<sms * 16, 256>>>(ctr, nctr - 1, n, out);
    cudaEventRecord(e0);
    k_atomics<<<sms * 16, 256>>>(ctr, nctr - 1, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"bench\":\"atomicAdd_random\",\"counters\":%u,\"g_atomics_per_s\":%.1f}\n", nctr, n / ms / 1e6);
    cudaFree(ctr);
  }
  {
    const uint32_t nb = 1u << 16, cap = 5120;
    const uint64_t n = 256ull << 20;
    uint32_t* ctr;
    uint64_t* dst;
    cudaMalloc(&ctr, (size_t)nb * 4);
    cudaMalloc(&dst, (size_t)nb * cap * 8);
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
      cudaMemset(ctr, 0, (size_t)nb * 4);
      cudaEventRecord(e0);
      k_scatter<<<sms * 16, 256>>>(ctr, nb - 1, cap, n, dst);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("{\"bench\":\"scatter_8B_atomic_slot\",\"bins\":%u,\"g_records_per_s\":%.1f,\"gbs_written\":%.1f}\n", nb,
           n / best / 1e6, n * 8 / best / 1e6);
    cudaFree(ctr);
    cudaFree(dst);
  }
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) printf("{\"error\":\"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
