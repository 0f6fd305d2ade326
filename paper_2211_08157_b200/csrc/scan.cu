// scan.cu — device-wide exclusive prefix sums (single pass, decoupled look-back) and small utilities.
#include <cstring>

#include "common.cuh"

namespace god {

namespace {
constexpr int SCAN_NT = 256;
constexpr int SCAN_IPT = 16;
constexpr int SCAN_TILE = SCAN_NT * SCAN_IPT;

template <class TIn>
__global__ void __launch_bounds__(SCAN_NT) k_scan(const TIn* in, uint64_t* out, uint64_t n,
                                                  uint64_t* status, uint32_t* tile_ctr, uint64_t* total) {
  __shared__ uint64_t warp_sum[SCAN_NT / 32];
  __shared__ uint64_t s_excl;
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_IPT;
  uint64_t v[SCAN_IPT];
  uint64_t sum = 0;
  // a full tile of 16-B aligned arrays: 128-bit loads and stores (a thread's 16 items are contiguous)
  const bool vec = base + SCAN_IPT <= n && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0;
  if (vec) {
    if constexpr (sizeof(TIn) == 4) {
      const uint4* p4 = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
      for (int i = 0; i < SCAN_IPT / 4; i++) {
        const uint4 q = p4[i];
        v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
      }
    } else {
      const ulonglong2* p2 = reinterpret_cast<const ulonglong2*>(in + base);
#pragma unroll
      for (int i = 0; i < SCAN_IPT / 2; i++) {
        const ulonglong2 q = p2[i];
        v[2 * i] = q.x; v[2 * i + 1] = q.y;
      }
    }
#pragma unroll
    for (int i = 0; i < SCAN_IPT; i++) sum += v[i];
  } else {
#pragma unroll
    for (int i = 0; i < SCAN_IPT; i++) {
      uint64_t idx = base + i;
      v[i] = idx < n ? (uint64_t)in[idx] : 0;
      sum += v[i];
    }
  }
  // block exclusive scan of per-thread sums
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t x = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_sum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint64_t ws = lane < SCAN_NT / 32 ? warp_sum[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, ws, d);
      if (lane >= d) ws += y;
    }
    if (lane < SCAN_NT / 32) warp_sum[lane] = ws;  // inclusive
    const uint64_t tile_total = __shfl_sync(0xffffffffu, ws, SCAN_NT / 32 - 1);
    const uint64_t ex = lb_exclusive_warp(status, tile, tile_total);
    if (lane == 0) s_excl = ex;
  }
  __syncthreads();
  uint64_t run = s_excl + (wid ? warp_sum[wid - 1] : 0) + x - sum;
  if (vec) {
    ulonglong2* o2 = reinterpret_cast<ulonglong2*>(out + base);
#pragma unroll
    for (int i = 0; i < SCAN_IPT / 2; i++) {
      const uint64_t a = run, b = run + v[2 * i];
      run = b + v[2 * i + 1];
      o2[i] = make_ulonglong2(a, b);
    }
  } else {
#pragma unroll
    for (int i = 0; i < SCAN_IPT; i++) {
      uint64_t idx = base + i;
      if (idx < n) out[idx] = run;
      run += v[i];
    }
  }
  if (total && tile == (n + SCAN_TILE - 1) / SCAN_TILE - 1 && threadIdx.x == SCAN_NT - 1) *total = run;
}

template <class TIn>
void scan_impl(const TIn* in, uint64_t* out, uint64_t n, uint64_t* total, cudaStream_t st, Scratch& scr,
               const char* tag) {
  if (n == 0) {
    if (total) GOD_CUDA(cudaMemsetAsync(total, 0, sizeof(uint64_t), st));
    return;
  }
  uint64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  uint64_t* status = scr.alloc<uint64_t>(tiles);
  uint32_t* ctr = scr.alloc<uint32_t>(1);
  GOD_CUDA(cudaMemsetAsync(status, 0, tiles * sizeof(uint64_t), st));
  GOD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
  GOD_LAUNCH(tag, k_scan<TIn>, (unsigned)tiles, SCAN_NT, 0, st, in, out, n, status, ctr, total);
}
}  // namespace

void scan_exclusive_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* total, cudaStream_t st,
                        Scratch& scr, const char* tag) {
  scan_impl<uint64_t>(in, out, n, total, st, scr, tag);
}
void scan_exclusive_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n, uint64_t* total, cudaStream_t st,
                               Scratch& scr, const char* tag) {
  scan_impl<uint32_t>(in, out, n, total, st, scr, tag);
}

namespace {
__global__ void k_d2h_small(const uint8_t* __restrict__ src, uint8_t* dst, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
}  // namespace

thread_local bool t_copies_in_flight = false;
void set_copies_in_flight(bool on) { t_copies_in_flight = on; }

void d2h_small(void* host, const void* dev, size_t bytes, cudaStream_t st) {
  thread_local uint8_t* mapped = nullptr;  // host-mapped pinned page of this host thread
  if (!mapped) GOD_CUDA(cudaHostAlloc((void**)&mapped, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
  GOD_REQUIRE(bytes <= 4096, "d2h_small: at most 4096 bytes");
  if (bytes) {
    if (t_copies_in_flight)  // large copies of another stream occupy the copy engine: write through mapping
      GOD_LAUNCH("k_d2h_small", k_d2h_small, 1, 128, 0, st, static_cast<const uint8_t*>(dev), mapped, (uint32_t)bytes);
    else  // an idle copy engine: a pinned copy has the lower latency
      GOD_CUDA(cudaMemcpyAsync(mapped, dev, bytes, cudaMemcpyDeviceToHost, st));
  }
  GOD_CUDA(cudaStreamSynchronize(st));
  memcpy(host, mapped, bytes);
}

}  // namespace god
