// G1: what one random access costs on this B200, by load flavour (round 2).  k_probe reads one random
// 32-B directory record per probe and ncu shows 4.7 L2 sectors / ~140 DRAM bytes per probe: this
// benchmark separates the load instruction's cache / prefetch-size qualifiers from the hardware's
// DRAM access granularity.  Each variant gathers random 32-B-aligned elements from a 4 GB buffer.
// Run under ncu (--metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum) to get
// sectors and DRAM bytes per gather; standalone it prints gathers/s.  Not part of libgod.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/g1_gather tools/g1_gather.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

enum { V_LDG4 = 0, V_CG4, V_CV4, V_NA64, V_P64, V_P128, V_P256, V_NCNA, V_LDG32, V_NA32, V_LINE128, V_LU4, V_CS4, NV };
static const char* names[NV] = {"ldg4_nc", "ld_cg4", "ld_cv4", "ld_L1na_L2_64B", "ld_L2_64B", "ld_L2_128B", "ld_L2_256B",
                                "ld_nc_L1na", "ldg32_nc(2x16B)", "ld_L1na_32B(2x16B)", "line128(4 lanes x 32B)", "ld_lu4", "ld_cs4"};

template <int V>
__device__ __forceinline__ uint32_t load_one(const uint32_t* p) {
  uint32_t r;
  if constexpr (V == V_LDG4) r = __ldg(p);
  else if constexpr (V == V_CG4) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
  else if constexpr (V == V_CV4) asm volatile("ld.global.cv.u32 %0, [%1];" : "=r"(r) : "l"(p));
  else if constexpr (V == V_NA64) asm volatile("ld.global.L1::no_allocate.L2::64B.u32 %0, [%1];" : "=r"(r) : "l"(p));
  else if constexpr (V == V_P64) asm volatile("ld.global.L2::64B.u32 %0, [%1];" : "=r"(r) : "l"(p));
  else if constexpr (V == V_P128) asm volatile("ld.global.L2::128B.u32 %0, [%1];" : "=r"(r) : "l"(p));
  else if constexpr (V == V_P256) asm volatile("ld.global.L2::256B.u32 %0, [%1];" : "=r"(r) : "l"(p));
  else if constexpr (V == V_NCNA) asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  else if constexpr (V == V_LU4) asm volatile("ld.global.lu.u32 %0, [%1];" : "=r"(r) : "l"(p));
  else if constexpr (V == V_CS4) asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(r) : "l"(p));
  else if constexpr (V == V_LDG32) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p)), b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
    r = a.x ^ a.w ^ b.y ^ b.w;
  } else if constexpr (V == V_NA32) {
    uint4 a, b;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(p));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p + 4));
    r = a.x ^ a.w ^ b.y ^ b.w;
  } else r = 0;
  return r;
}

template <int V>
__global__ void k_gather(const uint32_t* __restrict__ buf, uint64_t nsect, uint32_t iters, uint32_t* out) {
  uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
  uint32_t acc = 0;
  if constexpr (V == V_LINE128) {
    // groups of 4 lanes share one random 128-B line, each lane reads its own 32-B sector
    const uint32_t l4 = threadIdx.x & 3;
    x = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 2) * 0x9E3779B97F4A7C15ull + 1;
    for (uint32_t i = 0; i < iters; i += 4) {
      uint4 v[4][2];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        const uint32_t* p = buf + (((x >> 3) % (nsect / 4)) * 4 + l4) * 8;
        v[u][0] = __ldg(reinterpret_cast<const uint4*>(p));
        v[u][1] = __ldg(reinterpret_cast<const uint4*>(p) + 1);
      }
#pragma unroll
      for (int u = 0; u < 4; u++) acc += v[u][0].x ^ v[u][1].w;
    }
  } else {
    for (uint32_t i = 0; i < iters; i += 8) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        v[u] = load_one<V>(buf + ((x >> 3) % nsect) * 8);
      }
#pragma unroll
      for (int u = 0; u < 8; u++) acc += v[u];
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int V>
static void run(const uint32_t* buf, uint64_t bytes, int sms, uint32_t* out, cudaEvent_t e0, cudaEvent_t e1) {
  const int threads = 256, blocks = sms * 8;
  const uint32_t iters = 256;
  k_gather<V><<<blocks, threads>>>(buf, bytes / 32, iters, out);
  cudaEventRecord(e0);
  k_gather<V><<<blocks, threads>>>(buf, bytes / 32, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double n = (double)blocks * threads * iters;
  if (V == V_LINE128) n /= 4;  // gathers = lines
  printf("{\"bench\":\"g1_gather\",\"variant\":\"%s\",\"buffer_mb\":%llu,\"g_gathers_per_s\":%.2f,\"err\":\"%s\"}\n", names[V],
         (unsigned long long)(bytes >> 20), n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  int sms = 0;
  if (argc > 1) {  // L2 fetch granularity limit, set before the context allocates
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[1]));
    size_t g = 0;
    cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
    printf("{\"set_limit\":%d,\"err\":\"%s\",\"limit_now\":%zu}\n", atoi(argv[1]), cudaGetErrorString(e), g);
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint64_t bytes = 4096ull << 20;
  uint32_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  run<V_LDG4>(buf, bytes, sms, out, e0, e1);
  run<V_CG4>(buf, bytes, sms, out, e0, e1);
  run<V_CV4>(buf, bytes, sms, out, e0, e1);
  run<V_NA64>(buf, bytes, sms, out, e0, e1);
  run<V_P64>(buf, bytes, sms, out, e0, e1);
  run<V_P128>(buf, bytes, sms, out, e0, e1);
  run<V_P256>(buf, bytes, sms, out, e0, e1);
  run<V_NCNA>(buf, bytes, sms, out, e0, e1);
  run<V_LDG32>(buf, bytes, sms, out, e0, e1);
  run<V_NA32>(buf, bytes, sms, out, e0, e1);
  run<V_LINE128>(buf, bytes, sms, out, e0, e1);
  run<V_LU4>(buf, bytes, sms, out, e0, e1);
  run<V_CS4>(buf, bytes, sms, out, e0, e1);
  return 0;
}
