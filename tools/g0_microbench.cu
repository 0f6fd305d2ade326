// G0: microbenchmarks that give the probe kernels a roofline on this B200:
//  (1) random 4-byte loads, one per 32-B sector, over buffers of 64 MB (L2-resident) .. 4 GB (HBM);
//  (2) INT32 ALU throughput (LOP3/IADD3/SHF mix).  Standalone; not part of libgod.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_rand_gather(const uint32_t* __restrict__ buf, uint64_t nwords, uint64_t iters, uint32_t* out) {
  uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
  uint32_t acc = 0;
  for (uint64_t i = 0; i < iters; i += 8) {
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      v[u] = __ldg(buf + ((x >> 3) % (nwords / 8)) * 8);   // one word per 32-B sector
    }
#pragma unroll
    for (int u = 0; u < 8; u++) acc += v[u];
  }
  if (acc == 0x12345678u) out[0] = acc;
}
__global__ void k_alu(uint32_t iters, uint32_t* out) {
  uint32_t a = threadIdx.x, b = blockIdx.x, c = a ^ 0x5bd1e995u, d = b + 7;
  for (uint32_t i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      a = (a ^ (b >> 3)) + c; b = (b << 5) ^ d; c = __funnelshift_r(c, a, 7) ^ b; d = (d + a) ^ (c >> 11);
    }
  }
  if ((a ^ b ^ c ^ d) == 0x1u) out[0] = a;
}
int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint32_t* out; cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  uint64_t sizes[] = {64ull << 20, 512ull << 20, 4096ull << 20};
  for (uint64_t bytes : sizes) {
    uint32_t* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
    const int threads = 256, blocks = sms * 8; const uint64_t iters = 512;
    k_rand_gather<<<blocks, threads>>>(buf, bytes / 4, iters, out);
    cudaEventRecord(e0);
    k_rand_gather<<<blocks, threads>>>(buf, bytes / 4, iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double n = (double)blocks * threads * iters;
    printf("{\"bench\":\"random_sector_gather\",\"buffer_mb\":%llu,\"gsectors_per_s\":%.1f,\"equiv_gbs_32B\":%.1f}\n",
           (unsigned long long)(bytes >> 20), n / ms / 1e6, n * 32 / ms / 1e6);
    cudaFree(buf);
  }
  {
    const int threads = 256, blocks = sms * 8; const uint32_t iters = 4096;
    k_alu<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e0);
    k_alu<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 16 * 12;  // ~12 INT ops per inner step
    printf("{\"bench\":\"int32_alu\",\"tops\":%.2f,\"per_sm_per_clk_at_1965MHz\":%.1f}\n", ops / ms / 1e9,
           ops / ms / 1e-3 / sms / 1.965e9);
  }
  return 0;
}
