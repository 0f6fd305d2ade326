// common.cuh — shared device/host helpers of libgod (the product path; never includes oracle/).
#pragma once
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda/atomic>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <string>
#include <mutex>
#include <vector>
#include "god.h"

namespace god {

// ------------------------------------------------------------------------------------ errors
void set_error(const std::string& msg);
struct Fail {
  god_status code;
};
#define GOD_CUDA(call)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess) {                                                                    \
      ::god::set_error(std::string(#call) + ": " + cudaGetErrorString(e_) + " @" + __FILE__ + \
                       ":" + std::to_string(__LINE__));                                         \
      throw ::god::Fail{e_ == cudaErrorMemoryAllocation ? GOD_ENOMEM : GOD_ECUDA};              \
    }                                                                                           \
  } while (0)
#define GOD_LAUNCH_CHECK() GOD_CUDA(cudaGetLastError())
#define GOD_REQUIRE(cond, msg)                         \
  do {                                                 \
    if (!(cond)) {                                     \
      ::god::set_error(std::string("EINVAL: ") + msg); \
      throw ::god::Fail{GOD_EINVAL};                   \
    }                                                  \
  } while (0)

// ------------------------------------------------------------------------------------ pattern
// The diet pattern P and the tables the kernels use to map a patterned (included) index
// q of a sequence with phase s to its original position: orig(q) = s + (q / x) * p + one[q % x]
// (P:286 (1)-(2): the pattern repeated to the sequence length, keep bases under '1').
struct Pattern {
  uint32_t p, x;
  uint64_t bits;          // bit i = P[i]
  uint8_t one[64];        // positions of the ones, ascending
  uint8_t gap[64];        // orig(q+1) - orig(q) for q % x == r
  uint8_t ones_before[65];
};

struct Params {           // kernel-side view of god_params
  Pattern pat;
  int32_t k, w;
  uint64_t kmask;         // 4^k - 1
};

Params make_params(const god_params* prm);   // validates (GOD_EINVAL) and builds tables

__host__ __device__ inline uint64_t included_count(const Pattern& P, uint64_t L, uint32_t s) {
  if (L <= s) return 0;
  uint64_t n = L - s;
  if (n <= 0xFFFFFFFFull) {  // 32-bit division (a 64-bit one is ~100 instructions on the device)
    const uint32_t n32 = (uint32_t)n;
    return (uint64_t)(n32 / P.p) * P.x + P.ones_before[n32 % P.p];
  }
  return (n / P.p) * P.x + P.ones_before[n % P.p];
}
__host__ __device__ inline uint64_t orig_of(const Pattern& P, uint64_t q, uint32_t s) {
  return s + (q / P.x) * P.p + P.one[q % P.x];
}

// ------------------------------------------------------------------------------------ hash
// Thomas Wang's 64-bit integer mix (ref. 120), every step reduced mod 4^k (the 2k-bit
// mask of minimap2's sketch): x1 = ~x + (x<<21); x2 = x1 ^ x1>>24; x3 = 265 x2; x4 = x3 ^ x3>>14;
// x5 = 21 x4; x6 = x5 ^ x5>>28; H = (2^31+1) x6.
__device__ __forceinline__ uint64_t wang_hash(uint64_t key, uint64_t mask) {
  key = (~key + (key << 21)) & mask;
  key = key ^ (key >> 24);
  key = (key * 265ull) & mask;
  key = key ^ (key >> 14);
  key = (key * 21ull) & mask;
  key = key ^ (key >> 28);
  key = (key + (key << 31)) & mask;
  return key;
}

// A/a->0 C/c->1 G/g->2 T/t->3, anything else -> 4 (N).  Branch-free table in a 64-bit constant:
// only bits 1..2 of the ASCII byte separate A(1) C(3) G(7) T(20) ... use a small LUT instead.
__device__ __forceinline__ uint32_t base_code(uint8_t b) {
  // ASCII: A=0x41 C=0x43 G=0x47 T=0x54, a=0x61 c=0x63 g=0x67 t=0x74
  uint32_t u = b & 0xDFu;  // upper-case
  uint32_t c = 4;
  c = (u == 'A') ? 0u : c;
  c = (u == 'C') ? 1u : c;
  c = (u == 'G') ? 2u : c;
  c = (u == 'T') ? 3u : c;
  return c;
}

// ------------------------------------------------------------------------------------ look-back
// Decoupled look-back for ordered, single-pass exclusive prefixes across tiles (tile order =
// position order).  status word: [63:62] flag (0 empty, 1 aggregate, 2 inclusive) | [61:0] value.
constexpr uint64_t LB_AGG = 1ull << 62;
constexpr uint64_t LB_INC = 2ull << 62;
constexpr uint64_t LB_VAL = (1ull << 62) - 1;

// The status word is the only datum exchanged (no payload is published through it), so relaxed
// accesses suffice; acquire/release here would add an L1 invalidate + fence to every spin.
__device__ __forceinline__ void lb_store(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t lb_load(uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Called by ONE thread of tile `tile` with the tile's local total; returns the exclusive prefix.
__device__ inline uint64_t lb_exclusive(uint64_t* status, uint64_t tile, uint64_t local) {
  if (tile == 0) {
    lb_store(&status[0], LB_INC | local);
    return 0;
  }
  lb_store(&status[tile], LB_AGG | local);
  uint64_t excl = 0;
  int64_t j = (int64_t)tile - 1;
  while (true) {
    uint64_t s = lb_load(&status[j]);
    uint64_t f = s & ~LB_VAL;
    if (f == 0) continue;  // predecessor not published yet (it is running: tiles are issued in order)
    excl += s & LB_VAL;
    if (f == LB_INC) break;
    --j;
  }
  lb_store(&status[tile], LB_INC | (excl + local));
  return excl;
}

// Warp-cooperative variant (call with a whole warp): each round inspects 32 predecessors at once.
__device__ inline uint64_t lb_exclusive_warp(uint64_t* status, uint64_t tile, uint64_t local) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) lb_store(&status[0], LB_INC | local);
    return 0;
  }
  if (lane == 0) lb_store(&status[tile], LB_AGG | local);
  uint64_t excl = 0;
  int64_t j = (int64_t)tile - 1 - lane;
  while (true) {
    uint64_t s = j >= 0 ? lb_load(&status[j]) : (LB_INC | 0ull);
    while (__any_sync(0xffffffffu, (s & ~LB_VAL) == 0)) {
      if ((s & ~LB_VAL) == 0) s = lb_load(&status[j]);
    }
    const uint32_t inc = __ballot_sync(0xffffffffu, (s & ~LB_VAL) == LB_INC);
    const int first = inc ? __ffs(inc) - 1 : 32;  // closest predecessor with an inclusive prefix
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

// One-time setup per device (kernel attributes, streams and pool settings belong to a device): f runs
// once for each device a call site is reached on, under a lock, before anyone passes.
struct DeviceOnce {
  std::mutex mu;
  uint64_t done = 0;  // bit per device ordinal (mod 64)
  template <class F>
  void run(F f) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    std::lock_guard<std::mutex> g(mu);
    if (done & bit) return;
    f();
    done |= bit;
  }
};

// ------------------------------------------------------------------------------------ memory
// Stream-ordered scratch allocation (cudaMallocAsync pool), freed in reverse at scope exit.
// Memory pools of the current device beside its default pool (api.cu): the index build's scratch and
// the index's own storage each get one, so that a build and a seeding call, whose multi-GB blocks have
// different sizes, never recycle each other's memory (alternating them in one pool made the allocator
// re-map physical memory every step: 40 ms of host-side gaps per human '1110' step, measured).
enum PoolKind { POOL_DEFAULT = 0, POOL_BUILD = 1, POOL_INDEX = 2 };
cudaMemPool_t god_pool(PoolKind kind);

struct Scratch {
  cudaStream_t st;
  cudaMemPool_t pool = nullptr;  // null: the device's default pool
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s, PoolKind kind = POOL_DEFAULT) : st(s) {
    keep_pool();
    if (kind != POOL_DEFAULT) pool = god_pool(kind);
  }
  // Keep freed pool memory mapped (release threshold = max): without this every synchronize
  // trims the pool and the next multi-GB cudaMallocAsync re-maps physical memory.
  static void keep_pool() {
    static DeviceOnce once;
    once.run([] {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    });
  }
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    size_t bytes = count * sizeof(T);
    if (bytes == 0) bytes = 16;
    if (pool) GOD_CUDA(cudaMallocFromPoolAsync(&p, bytes, pool, st));
    else GOD_CUDA(cudaMallocAsync(&p, bytes, st));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Scratch() {
    for (size_t i = ptrs.size(); i-- > 0;) cudaFreeAsync(ptrs[i], st);
  }
};

// Host-or-device pointer handling for the ABI (see god.h CONVENTIONS).
bool is_device_ptr(const void* p);

inline unsigned grid_for(uint64_t n, unsigned block) {
  uint64_t g = (n + block - 1) / block;
  if (g == 0) g = 1;
  if (g > 0x7FFFFFFFull) g = 0x7FFFFFFFull;
  return (unsigned)g;
}

int num_sms();

// ------------------------------------------------------------------------------------ checked build
// GOD_DCHECK(cond, what): with -DGOD_CHECKED (libgod_checked.so, loaded when GOD_CHECKED=1) a computed
// global index or address that leaves its buffer prints the site and traps (the launch then fails with
// an illegal-instruction error that the C ABI reports as GOD_ECUDA); compiled out otherwise.  This is
// the memory-safety layer that stands in for compute-sanitizer, which the GPU pool refuses.
#ifdef GOD_CHECKED
#define GOD_DCHECK(cond, what)                                                                             \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("GOD_CHECKED: %s violated at %s:%d (block %u, thread %u)\n", what, __FILE__, __LINE__,         \
             blockIdx.x, threadIdx.x);                                                                     \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define GOD_DCHECK(cond, what) \
  do {                         \
  } while (0)
#endif

// ------------------------------------------------------------------------------------ tracing
// Every kernel launch goes through GOD_LAUNCH: it counts launches (god_launch_count) and, when
// god_profile_enable(1) is on, brackets the launch with CUDA events on the launching stream so
// the per-kernel device time is accumulated by name (god_profile_query).
struct ProfScope {
  const char* name;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(const char* n, cudaStream_t s);
  ~ProfScope();
};
// Work units (e.g. k-mer start positions) processed by the launches named `name`, reported by
// god_profile_units for the roofline of bench.py (recorded only while profiling is on).
void prof_add_units(const char* name, uint64_t units);
// NVTX range over a host scope (API entry points and the stages inside them; SURVEY §5 tracing): shows
// up on the Nsight timeline, costs one predicted branch when no tool is attached
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define GOD_LAUNCH(NAME, KERNEL, GRID, BLOCK, SMEM, ST, ...)      \
  do {                                                           \
    ::god::ProfScope ps_(NAME, ST);                              \
    KERNEL<<<(GRID), (BLOCK), (SMEM), (ST)>>>(__VA_ARGS__);      \
    GOD_LAUNCH_CHECK();                                          \
  } while (0)

// ------------------------------------------------------------------------------------ scans
// Device-wide exclusive scan of n u64 values (in may alias out).  *total (device, may be null)
// receives the sum.  Single pass, decoupled look-back.
void scan_exclusive_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* total, cudaStream_t st,
                        Scratch& scr, const char* tag = "k_scan");
void scan_exclusive_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n, uint64_t* total, cudaStream_t st,
                               Scratch& scr, const char* tag = "k_scan");

// Small device->host reads (counts, totals; <= 4096 bytes) into a pinned page, then a synchronize of
// `st`.  While large device->host copies of other streams are in flight (the pipelined seeding's
// result copies) the page is written through its host mapping by a one-thread kernel instead, so the
// read does not queue behind them on the copy engine.
void d2h_small(void* host, const void* dev, size_t bytes, cudaStream_t st);
// set while this host thread streams large device->host copies on other streams (pipelined seeding)
void set_copies_in_flight(bool on);
template <class T>
inline T d2h_scalar(const T* dptr, cudaStream_t st) {
  T v;
  d2h_small(&v, dptr, sizeof(T), st);
  return v;
}

}  // namespace god
