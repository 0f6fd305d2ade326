#include <algorithm>
// api.cu — the C ABI (include/god.h): validation, host/device staging, dispatch to the kernels.
#include <atomic>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include "internal.cuh"

namespace god {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

int num_sms() {  // of the current device
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& n = sms[dev & 63];
  if (!n) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n = v > 0 ? v : 148;
  }
  return n;
}

cudaMemPool_t god_pool(PoolKind kind) {
  static cudaMemPool_t pools[64][3] = {};
  static std::mutex mu;
  int dev = 0;
  GOD_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  cudaMemPool_t& p = pools[dev & 63][kind];
  if (!p) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    GOD_CUDA(cudaMemPoolCreate(&p, &props));
    uint64_t thr = ~0ull;  // keep freed memory mapped
    GOD_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  return p;
}

// ---------------------------------------------------------------------------------- tracing
namespace {
struct ProfPending { const char* name; cudaEvent_t a, b; };
struct ProfAcc { double ms = 0; uint64_t n = 0; uint64_t units = 0; };
std::mutex g_prof_mu;
bool g_prof_on = false;
std::atomic<uint64_t> g_launches{0};
std::vector<ProfPending> g_pending;
std::map<std::string, ProfAcc> g_acc;
std::vector<std::string> g_order;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_flush_locked() {
  for (auto& p : g_pending) {
    cudaEventSynchronize(p.b);
    float ms = 0;
    cudaEventElapsedTime(&ms, p.a, p.b);
    auto it = g_acc.find(p.name);
    if (it == g_acc.end()) {
      g_order.push_back(p.name);
      it = g_acc.emplace(p.name, ProfAcc{}).first;
    }
    it->second.ms += ms;
    it->second.n += 1;
    g_pool.push_back(p.a);
    g_pool.push_back(p.b);
  }
  g_pending.clear();
}
}  // namespace

void prof_add_units(const char* name, uint64_t units) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  prof_flush_locked();
  auto it = g_acc.find(name);
  if (it == g_acc.end()) {
    g_order.push_back(name);
    it = g_acc.emplace(name, ProfAcc{}).first;
  }
  it->second.units += units;
}

ProfScope::ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  a = get_event();
  cudaEventRecord(a, st);
}
ProfScope::~ProfScope() {
  if (!a) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t b = get_event();
  cudaEventRecord(b, st);
  g_pending.push_back({name, a, b});
}

bool is_device_ptr(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

Params make_params(const god_params* prm) {
  GOD_REQUIRE(prm != nullptr, "params is NULL");
  GOD_REQUIRE(prm->pattern != nullptr, "pattern is NULL");
  const size_t p = strlen(prm->pattern);
  GOD_REQUIRE(p >= 1 && p <= 64, "pattern length must be 1..64");
  GOD_REQUIRE(prm->k >= 1 && prm->k <= 28, "k must be 1..28 (P:368)");
  GOD_REQUIRE(prm->w >= 1 && prm->w <= 255, "w must be 1..255");
  Params P;
  memset(&P, 0, sizeof(P));
  P.pat.p = (uint32_t)p;
  uint32_t x = 0;
  for (size_t i = 0; i < p; i++) {
    const char c = prm->pattern[i];
    GOD_REQUIRE(c == '0' || c == '1', "pattern must be over {0,1}");
    if (c == '1') {
      P.pat.bits |= 1ull << i;
      P.pat.one[x++] = (uint8_t)i;
    }
  }
  GOD_REQUIRE(x >= 1, "pattern must contain at least one '1' (weight >= 1)");
  P.pat.x = x;
  for (uint32_t r = 0; r < x; r++)
    P.pat.gap[r] = (uint8_t)(r + 1 < x ? P.pat.one[r + 1] - P.pat.one[r] : p - P.pat.one[x - 1] + P.pat.one[0]);
  uint32_t acc = 0;
  for (size_t i = 0; i <= p; i++) {
    P.pat.ones_before[i] = (uint8_t)acc;
    if (i < p && prm->pattern[i] == '1') ++acc;
  }
  P.k = prm->k;
  P.w = prm->w;
  P.kmask = (prm->k >= 32) ? ~0ull : ((1ull << (2 * prm->k)) - 1);
  return P;
}

// ---------------------------------------------------------------------------------- staging
struct Stage {
  cudaStream_t st;
  Scratch& scr;
  struct Back { void* user; void* dev; size_t bytes; };
  std::vector<Back> backs;
  bool synced_any = false;
  Stage(cudaStream_t s, Scratch& sc) : st(s), scr(sc) {}
  template <class T>
  const T* in(const T* p, size_t count) {
    if (!p || is_device_ptr(p)) return p;
    T* d = scr.alloc<T>(count);
    if (count) GOD_CUDA(cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, st));
    synced_any = true;
    return d;
  }
  template <class T>
  T* out(T* p, size_t count) {
    if (!p || is_device_ptr(p)) return p;
    T* d = scr.alloc<T>(count);
    backs.push_back({p, d, count * sizeof(T)});
    return d;
  }
  template <class T>
  T* inout(T* p, size_t count) {
    if (!p || is_device_ptr(p)) return p;
    T* d = scr.alloc<T>(count);
    if (count) GOD_CUDA(cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, st));
    backs.push_back({p, d, count * sizeof(T)});
    return d;
  }
  void finish() {
    for (auto& b : backs)
      if (b.bytes) GOD_CUDA(cudaMemcpyAsync(b.user, b.dev, b.bytes, cudaMemcpyDeviceToHost, st));
    GOD_CUDA(cudaStreamSynchronize(st));
  }
};

// offsets[n] (total bytes) readable from host or device
static uint64_t total_len(const uint64_t* offsets, uint32_t n, cudaStream_t st) {
  if (!offsets) return 0;
  if (!is_device_ptr(offsets)) return offsets[n];
  return d2h_scalar(offsets + n, st);
}

template <class F>
static god_status guarded(F&& f) {
  try {
    f();
    return GOD_OK;
  } catch (const Fail& e) {
    return e.code;
  } catch (const std::exception& e) {
    set_error(std::string("exception: ") + e.what());
    return GOD_ECUDA;
  } catch (...) {
    set_error("unknown exception");
    return GOD_ECUDA;
  }
}

namespace {
__global__ void k_split_records(const uint64_t* __restrict__ hz, const uint32_t* __restrict__ pos, uint64_t n,
                                uint64_t* hash, uint32_t* opos, uint8_t* strand) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = hz[i];
    if (hash) hash[i] = v & ((1ull << 63) - 1);
    if (opos) opos[i] = pos[i];
    if (strand) strand[i] = (uint8_t)(v >> 63);
  }
}
__global__ void k_rebase_u64(uint64_t* a, uint64_t n, uint64_t base, uint64_t add) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = a[i] - base + add;
}
// god_anchor -> god_anchor_compact (the read id is implied by the anchor offsets); a read position
// >= 2^31 cannot carry the strand bit
__global__ void k_compact_anchors(const god_anchor* __restrict__ in, uint64_t n, god_anchor_compact* __restrict__ out,
                                  uint32_t* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const god_anchor a = in[i];
    if (a.read_pos >> 31) atomicAdd(bad, 1u);
    out[i] = god_anchor_compact{a.ref_pos, a.read_pos | (a.strand << 31)};
  }
}
__global__ void k_check_phases(const uint8_t* ph, uint32_t n, uint32_t p, uint32_t* bad) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (ph[i] >= p) atomicAdd(bad, 1u);
}
}  // namespace

}  // namespace god

using namespace god;

// Host-buffer seeding, pipelined over read batches (the runtime analogue of minimap2's -K batching):
// batch b+1's reads are copied host->device on one stream while batch b is seeded on the caller's
// stream and batch b-1's anchors, offsets and phases are copied device->host on a third, through a
// ring of two device buffer sets.  Requires page-locked host buffers to overlap (pageable memory
// still works, serialised by the driver).  Returns the total number of anchors.
namespace {
struct PipeSlot {
  uint8_t* reads = nullptr;
  uint64_t reads_cap = 0;
  uint64_t* off = nullptr;
  uint64_t off_cap = 0;
  uint8_t* ph = nullptr;
  uint64_t* aoff = nullptr;
  god_anchor* an = nullptr;
  uint64_t an_cap = 0;
  god_anchor_compact* anc = nullptr;
  uint64_t anc_cap = 0;
  cudaEvent_t h2d_done = nullptr, comp_done = nullptr, d2h_done = nullptr;
  bool d2h_pending = false;
};
template <class T>
void grow(T*& p, uint64_t& cap, uint64_t need, cudaStream_t st) {
  if (need <= cap) return;
  if (p) GOD_CUDA(cudaFreeAsync(p, st));
  cap = need + need / 8 + 1024;
  GOD_CUDA(cudaMallocAsync((void**)&p, cap * sizeof(T), st));
}
}  // namespace

// the copy streams of the current device (created once per device)
static void copy_streams(cudaStream_t& s_h2d, cudaStream_t& s_d2h) {
  static cudaStream_t h2d_of[64] = {nullptr}, d2h_of[64] = {nullptr};
  static DeviceOnce once;
  int dev_ord = 0;
  GOD_CUDA(cudaGetDevice(&dev_ord));
  once.run([&] {
    GOD_CUDA(cudaStreamCreateWithFlags(&h2d_of[dev_ord & 63], cudaStreamNonBlocking));
    GOD_CUDA(cudaStreamCreateWithFlags(&d2h_of[dev_ord & 63], cudaStreamNonBlocking));
  });
  s_h2d = h2d_of[dev_ord & 63];
  s_d2h = d2h_of[dev_ord & 63];
}

// Pipelined seeding of host (or device) reads with host outputs: read batches go up on the copy stream,
// each is seeded on `st` when it is in, and its results go down on the other copy stream, through a ring
// of PIPE_SLOTS device buffer sets (uploads run up to PIPE_SLOTS - 1 batches ahead of the seeding).
// prefetch() needs no index: god_build_index_and_seed queues the first uploads right behind the
// reference's chunks, so the link stays busy while the index is sorted.
constexpr uint32_t PIPE_SLOTS = 4;
struct SeedPipe {
  const uint8_t* reads;
  const uint64_t* offs;
  uint32_t n_reads;
  god_phase_mode mode;
  uint8_t* phases;
  uint32_t t;
  void* anchors;
  uint64_t* anchor_offsets;
  uint64_t cap;
  uint32_t n_batches;
  cudaStream_t st, s_h2d, s_d2h;
  bool reads_on_device, compact;
  uint32_t* bad_compact;
  PipeSlot slot[PIPE_SLOTS];
  uint32_t per = 0, uploaded = 0;
  std::vector<uint64_t> boff;
  std::vector<const uint8_t*> breads;
  // GOD_PIPE_TRACE: developer aid, device timeline of every batch's upload / seeding / download
  bool trace = false;
  std::vector<cudaEvent_t> tev;  // 6 per batch: h2d begin/end, seeding begin/end, d2h begin/end
  cudaEvent_t t_origin = nullptr;

  SeedPipe(const uint8_t* reads_, const uint64_t* offs_, uint32_t n_reads_, god_phase_mode mode_, uint8_t* phases_,
           uint32_t t_, void* anchors_, uint64_t* anchor_offsets_, uint64_t cap_, uint32_t n_batches_, cudaStream_t st_,
           bool reads_on_device_, bool compact_, uint32_t* bad_compact_)
      : reads(reads_), offs(offs_), n_reads(n_reads_), mode(mode_), phases(phases_), t(t_), anchors(anchors_),
        anchor_offsets(anchor_offsets_), cap(cap_), n_batches(n_batches_), st(st_), reads_on_device(reads_on_device_),
        compact(compact_), bad_compact(bad_compact_) {
    copy_streams(s_h2d, s_d2h);
    for (auto& sl : slot) {
      GOD_CUDA(cudaEventCreateWithFlags(&sl.h2d_done, cudaEventDisableTiming));
      GOD_CUDA(cudaEventCreateWithFlags(&sl.comp_done, cudaEventDisableTiming));
      GOD_CUDA(cudaEventCreateWithFlags(&sl.d2h_done, cudaEventDisableTiming));
    }
    trace = getenv("GOD_PIPE_TRACE") != nullptr;
    if (trace) {
      tev.resize((size_t)n_batches * 6);
      for (auto& e : tev) GOD_CUDA(cudaEventCreate(&e));
      GOD_CUDA(cudaEventCreate(&t_origin));
      GOD_CUDA(cudaEventRecord(t_origin, st));
    }
    per = (n_reads + n_batches - 1) / n_batches;
    for (auto& sl : slot) {
      GOD_CUDA(cudaMallocAsync((void**)&sl.ph, (uint64_t)per + 1, st));
      GOD_CUDA(cudaMallocAsync((void**)&sl.aoff, ((uint64_t)per + 1) * sizeof(uint64_t), st));
    }
    // byte offset of each batch's first read (device-resident offsets: one small copy per batch start)
    boff.resize(n_batches + 1);
    for (uint32_t b = 0; b <= n_batches; b++) {
      if (reads_on_device) d2h_small(&boff[b], offs + r_begin(b), 8, st);
      else boff[b] = offs[r_begin(b)];
    }
    GOD_CUDA(cudaStreamSynchronize(st));  // the slots' phase / offset buffers exist before another stream uses them
    breads.resize(n_batches);
  }
  SeedPipe(const SeedPipe&) = delete;
  SeedPipe& operator=(const SeedPipe&) = delete;
  ~SeedPipe() {
    cudaStreamSynchronize(s_d2h);
    cudaStreamSynchronize(s_h2d);
    for (auto& sl : slot) {
      if (sl.reads) cudaFreeAsync(sl.reads, st);
      if (sl.off) cudaFreeAsync(sl.off, st);
      if (sl.ph) cudaFreeAsync(sl.ph, st);
      if (sl.aoff) cudaFreeAsync(sl.aoff, st);
      if (sl.an) cudaFreeAsync(sl.an, st);
      if (sl.anc) cudaFreeAsync(sl.anc, st);
      cudaEventDestroy(sl.h2d_done);
      cudaEventDestroy(sl.comp_done);
      cudaEventDestroy(sl.d2h_done);
    }
    for (auto& e : tev) cudaEventDestroy(e);
    if (t_origin) cudaEventDestroy(t_origin);
    cudaStreamSynchronize(st);
  }
  uint64_t r_begin(uint32_t b) const { return std::min<uint64_t>((uint64_t)b * per, n_reads); }
  void mark(uint32_t b, int which, cudaStream_t s) {
    if (trace) GOD_CUDA(cudaEventRecord(tev[b * 6 + which], s));
  }
  // queue the upload of batch b into its slot (its previous user, batch b - PIPE_SLOTS, has been seeded:
  // the slot's INPUT buffers are free then; the results leave from other buffers, so an upload never
  // waits for a download)
  void upload(uint32_t b) {
    PipeSlot& sl = slot[b % PIPE_SLOTS];
    const uint64_t r0 = r_begin(b), r1 = r_begin(b + 1), nb = r1 - r0;
    const uint64_t bytes = boff[b + 1] - boff[b];
    if (b >= PIPE_SLOTS) GOD_CUDA(cudaStreamWaitEvent(s_h2d, sl.comp_done, 0));
    grow(sl.off, sl.off_cap, nb + 1, s_h2d);
    if (!reads_on_device) grow(sl.reads, sl.reads_cap, bytes + 16, s_h2d);
    mark(b, 0, s_h2d);
    if (reads_on_device) {  // the reads stay where they are; only the batch's offsets are copied
      breads[b] = reads + boff[b];
      GOD_CUDA(cudaMemcpyAsync(sl.off, offs + r0, (nb + 1) * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s_h2d));
    } else {
      breads[b] = sl.reads;
      if (bytes) GOD_CUDA(cudaMemcpyAsync(sl.reads, reads + boff[b], bytes, cudaMemcpyHostToDevice, s_h2d));
      GOD_CUDA(cudaMemcpyAsync(sl.off, offs + r0, (nb + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s_h2d));
    }
    if (mode == GOD_PHASE_GIVEN && nb) GOD_CUDA(cudaMemcpyAsync(sl.ph, phases + r0, nb, cudaMemcpyHostToDevice, s_h2d));
    GOD_CUDA(cudaEventRecord(sl.h2d_done, s_h2d));
    mark(b, 1, s_h2d);
  }
  // uploads that fit the ring before any batch is seeded
  void prefetch() {
    while (uploaded < n_batches && uploaded < PIPE_SLOTS) upload(uploaded++);
  }
  // seed every batch against idx; returns the anchors in total (written while they fit cap)
  uint64_t run(const god_index* idx) {
    prefetch();
    uint64_t written = 0;  // anchors before the current batch
    const size_t asz_out = compact ? sizeof(god_anchor_compact) : sizeof(god_anchor);
    set_copies_in_flight(true);
    struct Reset { ~Reset() { set_copies_in_flight(false); } } reset_flag;
    for (uint32_t b = 0; b < n_batches; b++) {
      NvtxRange nvtx("seed batch");
      PipeSlot& sl = slot[b % PIPE_SLOTS];
      const uint64_t r0 = r_begin(b), r1 = r_begin(b + 1), nb = r1 - r0;
      GOD_CUDA(cudaStreamWaitEvent(st, sl.h2d_done, 0));
      mark(b, 2, st);
      GOD_LAUNCH("k_rebase", k_rebase_u64, grid_for(nb + 1, 256), 256, 0, st, sl.off, nb + 1, boff[b], 0ull);
      // anchors of this batch: a share of the caller's capacity, grown and redone if too small
      uint64_t want = cap ? std::min<uint64_t>(cap, cap / n_batches + cap / (4 * n_batches) + 4096) : 4096;
      uint64_t tot = 0;
      for (int attempt = 0; attempt < 2; attempt++) {
        if (sl.d2h_pending) GOD_CUDA(cudaStreamWaitEvent(st, sl.d2h_done, 0));
        grow(sl.an, sl.an_cap, want, st);
        tot = god::seed_reads(idx, breads[b], sl.off, (uint32_t)nb, mode, sl.ph, t, sl.an, sl.aoff, sl.an_cap, st,
                              (uint32_t)r0);
        if (tot <= sl.an_cap) break;
        want = tot;
      }
      // offsets of this batch -> global anchor offsets
      GOD_LAUNCH("k_rebase", k_rebase_u64, grid_for(nb + 1, 256), 256, 0, st, sl.aoff, nb + 1, 0ull, written);
      const void* src = sl.an;
      if (compact && tot && tot <= sl.an_cap) {  // 8-B anchors leave the device: half the copy
        grow(sl.anc, sl.anc_cap, tot, st);
        GOD_LAUNCH("k_compact_anchors", k_compact_anchors, grid_for(tot, 256), 256, 0, st, sl.an, tot, sl.anc,
                   bad_compact);
        src = sl.anc;
      }
      GOD_CUDA(cudaEventRecord(sl.comp_done, st));
      mark(b, 3, st);
      if (uploaded < n_batches) upload(uploaded++);  // batch b + PIPE_SLOTS takes this slot's input buffers
      GOD_CUDA(cudaStreamWaitEvent(s_d2h, sl.comp_done, 0));
      mark(b, 4, s_d2h);
      if (written + tot <= cap && tot)
        GOD_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(anchors) + written * asz_out, src, tot * asz_out,
                                 cudaMemcpyDeviceToHost, s_d2h));
      GOD_CUDA(cudaMemcpyAsync(anchor_offsets + r0, sl.aoff, (nb + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s_d2h));
      if (mode == GOD_PHASE_SELECT && nb) GOD_CUDA(cudaMemcpyAsync(phases + r0, sl.ph, nb, cudaMemcpyDeviceToHost, s_d2h));
      GOD_CUDA(cudaEventRecord(sl.d2h_done, s_d2h));
      mark(b, 5, s_d2h);
      sl.d2h_pending = true;
      written += tot;
    }
    GOD_CUDA(cudaStreamSynchronize(s_d2h));
    GOD_CUDA(cudaStreamSynchronize(s_h2d));
    if (trace) {
      for (uint32_t b = 0; b < n_batches; b++) {
        float tm[6];
        for (int q = 0; q < 6; q++) GOD_CUDA(cudaEventElapsedTime(&tm[q], t_origin, tev[b * 6 + q]));
        fprintf(stderr, "[pipe] batch %u: h2d %.2f-%.2f  seed %.2f-%.2f  d2h %.2f-%.2f ms\n", b, tm[0], tm[1], tm[2],
                tm[3], tm[4], tm[5]);
      }
    }
    return written;
  }
};

// whether a seeding call takes the pipelined path, and in how many batches (0: the plain path)
static uint32_t pipe_batches(const void* reads, const void* read_offsets, uint32_t n_reads, const void* phases,
                             const void* anchor_offsets, const void* anchors) {
  const char* pm = getenv("GOD_PIPE_MIN_READS");  // test hook: smaller batches
  const uint32_t pipe_min = pm ? (uint32_t)atoi(pm) : (1u << 20);  // reads per batch
  const uint32_t n_batches = std::min<uint32_t>(8u, n_reads / (pipe_min ? pipe_min : 1u));
  // reads and their offsets both on the host, or both on the device (then only the results are
  // streamed back); phases, anchor offsets and anchors on the host
  const bool rdev = is_device_ptr(reads), odev = is_device_ptr(read_offsets);
  if (n_batches >= 2 && rdev == odev && !is_device_ptr(phases) && !is_device_ptr(anchor_offsets) &&
      (!anchors || !is_device_ptr(anchors)))
    return n_batches;
  return 0;
}

extern "C" {

GOD_API const char* god_last_error(void) { return g_err.c_str(); }
GOD_API const char* god_version(void) { return "god-b200 0.1 (sm_100a)"; }

GOD_API void god_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
}
GOD_API void god_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  prof_flush_locked();
  g_acc.clear();
  g_order.clear();
}
GOD_API int god_profile_query(char* names, size_t names_len, double* ms, uint64_t* launches, int max_entries) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  prof_flush_locked();
  int n = 0;
  size_t off = 0;
  for (const auto& nm : g_order) {
    if (n >= max_entries) break;
    const auto& a = g_acc[nm];
    if (names && off + nm.size() + 1 <= names_len) {
      memcpy(names + off, nm.c_str(), nm.size() + 1);
      off += nm.size() + 1;
    }
    if (ms) ms[n] = a.ms;
    if (launches) launches[n] = a.n;
    ++n;
  }
  return n;
}
GOD_API uint64_t god_launch_count(void) { return g_launches.load(); }
GOD_API uint64_t god_profile_units(const char* name) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  auto it = g_acc.find(name ? name : "");
  return it == g_acc.end() ? 0 : it->second.units;
}

GOD_API god_status god_sparsify(const god_params* prm, const uint8_t* seq, const uint64_t* offsets, uint32_t n_seqs,
                                const uint8_t* phases, uint64_t* packed, uint64_t* nmask, uint64_t* out_offsets,
                                uint64_t* counts, uint64_t packed_cap_words, uint64_t* packed_needed,
                                god_stream stream) {
  return guarded([&] {
    Params P = make_params(prm);
    GOD_REQUIRE(offsets && out_offsets && counts && packed_needed, "NULL argument");
    GOD_REQUIRE(packed_cap_words == 0 || (packed && nmask), "NULL packed/nmask with nonzero capacity");
    if (phases && !is_device_ptr(phases))
      for (uint32_t i = 0; i < n_seqs; i++) GOD_REQUIRE(phases[i] < P.pat.p, "phase >= p");
    cudaStream_t st = (cudaStream_t)stream;
    Scratch scr(st);
    Stage sg(st, scr);
    const uint64_t L = total_len(offsets, n_seqs, st);
    const uint8_t* dseq = sg.in(seq, L);
    const uint64_t* doff = sg.in(offsets, (size_t)n_seqs + 1);
    const uint8_t* dph = sg.in(phases, n_seqs);
    uint64_t* doo = sg.out(out_offsets, (size_t)n_seqs + 1);
    uint64_t* dcnt = sg.out(counts, n_seqs);
    uint64_t* dpk = sg.out(packed, packed_cap_words);
    uint64_t* dnm = sg.out(nmask, packed_cap_words);
    god::sparsify(P, dseq, doff, n_seqs, dph, dpk, dnm, doo, dcnt, packed_cap_words, packed_needed, st);
    sg.finish();
  });
}

GOD_API god_status god_minimizers(const god_params* prm, const uint8_t* seq, const uint64_t* offsets, uint32_t n_seqs,
                                  const uint8_t* phases, int32_t global_pos, uint64_t* hash, uint32_t* pos,
                                  uint8_t* strand, uint64_t* out_offsets, uint64_t cap, uint64_t* needed,
                                  god_stream stream) {
  return guarded([&] {
    Params P = make_params(prm);
    GOD_REQUIRE(offsets && out_offsets && needed, "NULL argument");
    if (phases && !is_device_ptr(phases))
      for (uint32_t i = 0; i < n_seqs; i++) GOD_REQUIRE(phases[i] < P.pat.p, "phase >= p");
    cudaStream_t st = (cudaStream_t)stream;
    Scratch scr(st);
    Stage sg(st, scr);
    const uint64_t L = total_len(offsets, n_seqs, st);
    GOD_REQUIRE(!global_pos || L < (1ull << 32), "global positions need total length < 2^32");
    const uint8_t* dseq = sg.in(seq, L);
    const uint64_t* doff = sg.in(offsets, (size_t)n_seqs + 1);
    const uint8_t* dph = sg.in(phases, n_seqs);
    if (dph && is_device_ptr(phases)) {
      uint32_t* bad = scr.alloc<uint32_t>(1);
      GOD_CUDA(cudaMemsetAsync(bad, 0, 4, st));
      if (n_seqs) GOD_LAUNCH("k_check_phases", k_check_phases, grid_for(n_seqs, 256), 256, 0, st, dph, n_seqs, P.pat.p, bad);
      GOD_REQUIRE(d2h_scalar(bad, st) == 0, "phase >= p");
    }
    JobSet js = make_jobs(P, doff, n_seqs, dph, 0, 0, global_pos != 0, st, scr);
    Records rec;
    run_extract(P, dseq, js.seq_bytes, js.jobs, js.kb, js.n, js.total_pos, false, true, rec, st, scr,
                js.total_pos / (uint64_t)(P.w + 1) * 2 + js.total_pos / 8 + 4096, "extract_mz", js.x2p());
    *needed = rec.n;
    uint64_t* doo = sg.out(out_offsets, (size_t)n_seqs + 1);
    GOD_CUDA(cudaMemcpyAsync(doo, rec.job_off, ((size_t)n_seqs + 1) * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    if (rec.n > cap) {
      sg.finish();
      throw Fail{GOD_ETRUNC};
    }
    uint64_t* dh = sg.out(hash, rec.n);
    uint32_t* dp = sg.out(pos, rec.n);
    uint8_t* dz = sg.out(strand, rec.n);
    if (rec.n) {
      GOD_LAUNCH("k_split_records", k_split_records, grid_for(rec.n, 256), 256, 0, st, rec.hz, rec.pos, rec.n, dh, dp, dz);
    }
    sg.finish();
  });
}

}  // extern "C"

// god_build_index's body.  after_ref_queued (optional) runs once the reference's copies have been queued
// on the copy stream (or started on `st` when it is not streamed): god_build_index_and_seed queues the
// first read batches behind them there.
static void build_index_entry(const god_params* prm, const uint8_t* ref, const uint64_t* ref_offsets, uint32_t n_refs,
                              const god_cutoff* cutoff, god_index** out, god_stream stream,
                              const std::function<void()>& after_ref_queued) {
  NvtxRange nvtx("god_build_index");
  Params P = make_params(prm);
  GOD_REQUIRE(ref_offsets && out && cutoff, "NULL argument");
  GOD_REQUIRE(cutoff->mode <= 1, "cutoff mode must be 0 (fraction) or 1 (max_occ)");
  GOD_REQUIRE(cutoff->mode == 1 || cutoff->frac_den > 0, "cutoff frac_den must be > 0");
  *out = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch scr(st);
  Stage sg(st, scr);
  const uint64_t L = total_len(ref_offsets, n_refs, st);
  GOD_REQUIRE(L < (1ull << 32), "total reference length must be < 2^32 (u32 positions)");
  // A large host reference is streamed: chunks go up on the copy stream while K1 (stage 1+2) runs on
  // the tiles whose bytes are in, so only the sort and the table build follow the transfer.
  // GOD_STREAM_CHUNK_BYTES: test hook (chunk size; 0 disables streaming).
  const char* sc = getenv("GOD_STREAM_CHUNK_BYTES");
  const uint64_t want_chunk = sc ? strtoull(sc, nullptr, 10) : (32ull << 20);
  const uint64_t max_chunks = 16;
  god::SeqStream ss;
  struct EvGuard {
    god::SeqStream& s;
    ~EvGuard() {
      if (!s.arrived.empty()) set_copies_in_flight(false);
      for (cudaEvent_t e : s.arrived) cudaEventDestroy(e);
    }
  } ev_guard{ss};
  const uint8_t* dref;
  bool queued = false;
  if (ref && !is_device_ptr(ref) && want_chunk && L >= 2 * want_chunk) {
    uint8_t* d = scr.alloc<uint8_t>(L);
    cudaStream_t s_h2d, s_d2h;
    copy_streams(s_h2d, s_d2h);
    uint64_t chunk = std::max<uint64_t>(want_chunk, (L + max_chunks - 1) / max_chunks);
    chunk = (chunk + 255) & ~255ull;
    cudaEvent_t ready;  // the allocation is stream-ordered on st
    GOD_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    GOD_CUDA(cudaEventRecord(ready, st));
    GOD_CUDA(cudaStreamWaitEvent(s_h2d, ready, 0));
    GOD_CUDA(cudaEventDestroy(ready));  // (released once the wait has completed)
    ss.chunk_bytes = chunk;
    for (uint64_t o = 0; o < L; o += chunk) {
      cudaEvent_t e;
      GOD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ss.arrived.push_back(e);
      GOD_CUDA(cudaMemcpyAsync(d + o, ref + o, std::min<uint64_t>(chunk, L - o), cudaMemcpyHostToDevice, s_h2d));
      GOD_CUDA(cudaEventRecord(e, s_h2d));
    }
    set_copies_in_flight(true);  // small device->host reads go through the mapped page meanwhile
    if (after_ref_queued) after_ref_queued();
    queued = true;
    dref = d;
  } else {
    dref = sg.in(ref, L);
  }
  if (!queued && after_ref_queued) after_ref_queued();
  const uint64_t* doff = sg.in(ref_offsets, (size_t)n_refs + 1);
  god_index* ix = new god_index();
  try {
    god::build_index(P, dref, doff, n_refs, *cutoff, ix, st, ss.arrived.empty() ? nullptr : &ss);
  } catch (...) {
    if (!ss.arrived.empty()) {
      cudaStream_t s_h2d, s_d2h;
      copy_streams(s_h2d, s_d2h);
      cudaStreamSynchronize(s_h2d);  // the copies target scratch memory that is about to be freed
    }
    god_index_free(ix);
    throw;
  }
  sg.finish();
  *out = ix;
}

extern "C" {

GOD_API god_status god_build_index(const god_params* prm, const uint8_t* ref, const uint64_t* ref_offsets,
                                   uint32_t n_refs, const god_cutoff* cutoff, god_index** out, god_stream stream) {
  return guarded([&] { build_index_entry(prm, ref, ref_offsets, n_refs, cutoff, out, stream, nullptr); });
}

GOD_API god_status god_index_get_stats(const god_index* idx, god_index_stats* out_host) {
  return guarded([&] {
    GOD_REQUIRE(idx && out_host, "NULL argument");
    *out_host = idx->st;
  });
}

GOD_API god_status god_index_dump(const god_index* idx, uint64_t* hash, uint32_t* pos, uint8_t* strand, uint64_t cap,
                                  uint64_t* needed, god_stream stream) {
  return guarded([&] {
    GOD_REQUIRE(idx && needed, "NULL argument");
    const uint64_t n = idx->st.kept_entries;
    *needed = n;
    if (n > cap) throw Fail{GOD_ETRUNC};
    cudaStream_t st = (cudaStream_t)stream;
    Scratch scr(st);
    Stage sg(st, scr);
    uint64_t* dh = sg.out(hash, n);
    uint32_t* dp = sg.out(pos, n);
    uint8_t* dz = sg.out(strand, n);
    god::index_dump(idx, dh, dp, dz, st);
    sg.finish();
  });
}

GOD_API god_status god_index_count(const god_index* idx, const uint64_t* hashes, uint64_t n, uint32_t* counts,
                                   god_stream stream) {
  return guarded([&] {
    GOD_REQUIRE(idx && (n == 0 || (hashes && counts)), "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    Scratch scr(st);
    Stage sg(st, scr);
    const uint64_t* dh = sg.in(hashes, n);
    uint32_t* dc = sg.out(counts, n);
    // hashes must be < 4^k (a 2k-bit hash); larger values cannot be present
    god::index_count(idx, dh, n, dc, st);
    sg.finish();
  });
}

GOD_API void god_index_free(god_index* idx) {
  if (!idx) return;
  // the arrays come from the stream-ordered pool: wait for all users, then return them in order
  cudaDeviceSynchronize();
  if (idx->dir) cudaFreeAsync(idx->dir, 0);
  if (idx->ent) cudaFreeAsync(idx->ent, 0);
  if (idx->seg) cudaFreeAsync(idx->seg, 0);
  cudaStreamSynchronize(0);
  delete idx;
}

static void seed_entry(const god_index* idx, const uint8_t* reads, const uint64_t* read_offsets, uint32_t n_reads,
                       god_phase_mode mode, uint8_t* phases, uint32_t t, void* anchors, bool compact,
                       uint64_t* anchor_offsets, uint64_t cap, uint64_t* needed, god_stream stream) {
  NvtxRange nvtx("god_seed_reads");
  GOD_REQUIRE(idx && read_offsets && phases && anchor_offsets && needed, "NULL argument");
  GOD_REQUIRE(mode == GOD_PHASE_SELECT || mode == GOD_PHASE_GIVEN, "mode must be SELECT or GIVEN");
  GOD_REQUIRE(t >= 1, "t must be >= 1");
  GOD_REQUIRE(cap == 0 || anchors, "NULL anchors with nonzero capacity");
  if (mode == GOD_PHASE_GIVEN && !is_device_ptr(phases))
    for (uint32_t i = 0; i < n_reads; i++) GOD_REQUIRE(phases[i] < idx->P.pat.p, "phase >= p");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t asz = compact ? sizeof(god_anchor_compact) : sizeof(god_anchor);
  // all-host buffers and a large batch: pipelined transfers (SeedPipe)
  if (const uint32_t n_batches = pipe_batches(reads, read_offsets, n_reads, phases, anchor_offsets, anchors)) {
    Scratch scr(st);
    uint32_t* bad = scr.alloc<uint32_t>(1);
    GOD_CUDA(cudaMemsetAsync(bad, 0, 4, st));
    uint64_t tot;
    {
      SeedPipe pipe(reads, read_offsets, n_reads, mode, phases, t, anchors, anchor_offsets, anchors ? cap : 0, n_batches,
                    st, is_device_ptr(reads), compact, bad);
      tot = pipe.run(idx);
    }
    *needed = tot;
    if (compact) GOD_REQUIRE(d2h_scalar(bad, st) == 0, "compact anchors need read positions < 2^31");
    if (tot > cap) throw Fail{GOD_ETRUNC};
    return;
  }
  Scratch scr(st);
  Stage sg(st, scr);
  const uint64_t L = total_len(read_offsets, n_reads, st);
  const uint8_t* dreads = sg.in(reads, L);
  const uint64_t* doff = sg.in(read_offsets, (size_t)n_reads + 1);
  uint8_t* dph = mode == GOD_PHASE_GIVEN ? sg.inout(phases, n_reads) : sg.out(phases, n_reads);
  if (mode == GOD_PHASE_GIVEN && is_device_ptr(phases) && n_reads) {
    uint32_t* bad = scr.alloc<uint32_t>(1);
    GOD_CUDA(cudaMemsetAsync(bad, 0, 4, st));
    GOD_LAUNCH("k_check_phases", k_check_phases, grid_for(n_reads, 256), 256, 0, st, dph, n_reads, idx->P.pat.p, bad);
    GOD_REQUIRE(d2h_scalar(bad, st) == 0, "phase >= p");
  }
  uint64_t* dao = sg.out(anchor_offsets, (size_t)n_reads + 1);
  // anchors: a device god_anchor buffer (the caller's, or staging for host / compact outputs)
  const bool host_anchors = anchors && !is_device_ptr(anchors);
  god_anchor* dan = (!compact && !host_anchors) ? static_cast<god_anchor*>(anchors)
                                                : (cap ? scr.alloc<god_anchor>(cap) : nullptr);
  const uint64_t tot = god::seed_reads(idx, dreads, doff, n_reads, mode, dph, t, dan, dao, cap, st);
  *needed = tot;
  if (tot <= cap && tot) {
    const void* src = dan;
    if (compact) {
      god_anchor_compact* dc = host_anchors ? scr.alloc<god_anchor_compact>(tot)
                                            : static_cast<god_anchor_compact*>(anchors);
      uint32_t* bad = scr.alloc<uint32_t>(1);
      GOD_CUDA(cudaMemsetAsync(bad, 0, 4, st));
      GOD_LAUNCH("k_compact_anchors", k_compact_anchors, grid_for(tot, 256), 256, 0, st, dan, tot, dc, bad);
      GOD_REQUIRE(d2h_scalar(bad, st) == 0, "compact anchors need read positions < 2^31");
      src = dc;
    }
    if (host_anchors) GOD_CUDA(cudaMemcpyAsync(anchors, src, tot * asz, cudaMemcpyDeviceToHost, st));
  }
  sg.finish();
  if (tot > cap) throw Fail{GOD_ETRUNC};
}

GOD_API god_status god_seed_reads(const god_index* idx, const uint8_t* reads, const uint64_t* read_offsets,
                                  uint32_t n_reads, god_phase_mode mode, uint8_t* phases, uint32_t t,
                                  god_anchor* anchors, uint64_t* anchor_offsets, uint64_t cap, uint64_t* needed,
                                  god_stream stream) {
  return guarded([&] {
    seed_entry(idx, reads, read_offsets, n_reads, mode, phases, t, anchors, false, anchor_offsets, cap, needed, stream);
  });
}

GOD_API god_status god_seed_reads_compact(const god_index* idx, const uint8_t* reads, const uint64_t* read_offsets,
                                          uint32_t n_reads, god_phase_mode mode, uint8_t* phases, uint32_t t,
                                          god_anchor_compact* anchors, uint64_t* anchor_offsets, uint64_t cap,
                                          uint64_t* needed, god_stream stream) {
  return guarded([&] {
    seed_entry(idx, reads, read_offsets, n_reads, mode, phases, t, anchors, true, anchor_offsets, cap, needed, stream);
  });
}

GOD_API god_status god_build_index_and_seed(const god_params* prm, const uint8_t* ref, const uint64_t* ref_offsets,
                                            uint32_t n_refs, const god_cutoff* cutoff, god_index** out_index,
                                            const uint8_t* reads, const uint64_t* read_offsets, uint32_t n_reads,
                                            god_phase_mode mode, uint8_t* phases, uint32_t t, int compact,
                                            void* anchors, uint64_t* anchor_offsets, uint64_t cap, uint64_t* needed,
                                            god_stream stream) {
  return guarded([&] {
    NvtxRange nvtx("god_build_index_and_seed");
    GOD_REQUIRE(out_index && read_offsets && phases && anchor_offsets && needed, "NULL argument");
    GOD_REQUIRE(mode == GOD_PHASE_SELECT || mode == GOD_PHASE_GIVEN, "mode must be SELECT or GIVEN");
    GOD_REQUIRE(t >= 1, "t must be >= 1");
    GOD_REQUIRE(cap == 0 || anchors, "NULL anchors with nonzero capacity");
    *out_index = nullptr;
    const Params P = make_params(prm);
    if (mode == GOD_PHASE_GIVEN && !is_device_ptr(phases))
      for (uint32_t i = 0; i < n_reads; i++) GOD_REQUIRE(phases[i] < P.pat.p, "phase >= p");
    cudaStream_t st = (cudaStream_t)stream;
    const uint32_t n_batches = pipe_batches(reads, read_offsets, n_reads, phases, anchor_offsets, anchors);
    if (!n_batches) {  // nothing to overlap: the two calls one after the other
      build_index_entry(prm, ref, ref_offsets, n_refs, cutoff, out_index, stream, nullptr);
      seed_entry(*out_index, reads, read_offsets, n_reads, mode, phases, t, anchors, compact != 0, anchor_offsets, cap,
                 needed, stream);
      return;
    }
    Scratch scr(st);
    uint32_t* bad = scr.alloc<uint32_t>(1);
    GOD_CUDA(cudaMemsetAsync(bad, 0, 4, st));
    uint64_t tot;
    {
      SeedPipe pipe(reads, read_offsets, n_reads, mode, phases, t, anchors, anchor_offsets, anchors ? cap : 0, n_batches,
                    st, is_device_ptr(reads), compact != 0, bad);
      // the first read batches are queued on the copy stream right behind the reference
      build_index_entry(prm, ref, ref_offsets, n_refs, cutoff, out_index, stream, [&] { pipe.prefetch(); });
      tot = pipe.run(*out_index);
    }
    *needed = tot;
    if (compact) GOD_REQUIRE(d2h_scalar(bad, st) == 0, "compact anchors need read positions < 2^31");
    if (tot > cap) throw Fail{GOD_ETRUNC};
  });
}

GOD_API god_status god_vote_reads(const god_index* idx, const uint8_t* reads, const uint64_t* read_offsets,
                                  uint32_t n_reads, const uint8_t* phases, const god_anchor* anchors,
                                  const uint64_t* anchor_offsets, const god_vote_params* vp, god_vote* out,
                                  uint64_t* out_offsets, uint64_t cap, uint64_t* needed, god_stream stream) {
  return guarded([&] {
    GOD_REQUIRE(idx && read_offsets && anchor_offsets && vp && out_offsets && needed, "NULL argument");
    GOD_REQUIRE(n_reads == 0 || phases, "NULL phases");
    GOD_REQUIRE(cap == 0 || out, "NULL output with nonzero capacity");
    if (!is_device_ptr(phases) && phases)
      for (uint32_t i = 0; i < n_reads; i++) GOD_REQUIRE(phases[i] < idx->P.pat.p, "phase >= p");
    cudaStream_t st = (cudaStream_t)stream;
    Scratch scr(st);
    Stage sg(st, scr);
    const uint64_t L = total_len(read_offsets, n_reads, st);
    const uint64_t NA = total_len(anchor_offsets, n_reads, st);
    const uint8_t* dreads = sg.in(reads, L);
    const uint64_t* droff = sg.in(read_offsets, (size_t)n_reads + 1);
    const uint8_t* dph = sg.in(phases, n_reads);
    const god_anchor* dan = sg.in(anchors, NA);
    const uint64_t* daoff = sg.in(anchor_offsets, (size_t)n_reads + 1);
    GOD_REQUIRE(NA == 0 || dan, "NULL anchors");
    uint64_t* doo = sg.out(out_offsets, (size_t)n_reads + 1);
    god_vote* dout = out;
    const bool host_out = out && !is_device_ptr(out);
    if (host_out) dout = scr.alloc<god_vote>(cap);
    const uint64_t tot = god::vote_reads(idx, dreads, droff, n_reads, dph, dan, daoff, *vp, dout, doo, cap, st);
    *needed = tot;
    if (host_out && tot <= cap && tot)
      GOD_CUDA(cudaMemcpyAsync(out, dout, tot * sizeof(god_vote), cudaMemcpyDeviceToHost, st));
    sg.finish();
    if (tot > cap) throw Fail{GOD_ETRUNC};
  });
}

GOD_API god_status god_contain(const god_params* prm, const uint8_t* refs, const uint64_t* ref_offsets,
                               uint32_t n_refs, const god_cutoff* cutoff, const uint8_t* reads,
                               const uint64_t* read_offsets, uint32_t n_reads, uint32_t t,
                               const god_vote_params* vp, const god_contain_params* cp, uint64_t* mapped_reads,
                               uint64_t* mapped_bases, uint8_t* accepted, god_stream stream) {
  return guarded([&] {
    const Params P = make_params(prm);
    GOD_REQUIRE(refs || n_refs == 0, "NULL refs");
    GOD_REQUIRE(ref_offsets && read_offsets && cutoff && vp && cp, "NULL argument");
    GOD_REQUIRE(n_refs == 0 || (mapped_reads && mapped_bases && accepted), "NULL output");
    GOD_REQUIRE(t >= 1, "t must be >= 1");
    GOD_REQUIRE(cp->cov_den >= 1, "cov_den must be >= 1");
    GOD_REQUIRE(cutoff->mode == 1 || cutoff->frac_den >= 1, "cutoff fraction needs frac_den >= 1");
    cudaStream_t st = (cudaStream_t)stream;
    Scratch scr(st);
    Stage sg(st, scr);
    std::vector<uint64_t> hoff((size_t)n_refs + 1);
    if (is_device_ptr(ref_offsets))
      GOD_CUDA(cudaMemcpyAsync(hoff.data(), ref_offsets, hoff.size() * 8, cudaMemcpyDeviceToHost, st));
    else
      memcpy(hoff.data(), ref_offsets, hoff.size() * 8);
    GOD_CUDA(cudaStreamSynchronize(st));
    for (uint32_t i = 0; i < n_refs; i++) GOD_REQUIRE(hoff[i] <= hoff[i + 1], "ref_offsets must be ascending");
    const uint64_t LR = hoff[n_refs];
    const uint64_t LQ = total_len(read_offsets, n_reads, st);
    const uint8_t* dref = sg.in(refs, LR);
    const uint64_t* droff = sg.in(ref_offsets, (size_t)n_refs + 1);
    const uint8_t* dreads = sg.in(reads, LQ);
    const uint64_t* dqoff = sg.in(read_offsets, (size_t)n_reads + 1);
    uint64_t* dmr = sg.out(mapped_reads, n_refs);
    uint64_t* dmb = sg.out(mapped_bases, n_refs);
    uint8_t* dacc = sg.out(accepted, n_refs);
    if (n_refs)
      god::contain(P, dref, droff, hoff.data(), n_refs, *cutoff, dreads, dqoff, n_reads, t, *vp, cp->batch_bases,
                   cp->min_reads, cp->cov_num, cp->cov_den, dmr, dmb, dacc, st);
    sg.finish();
  });
}

GOD_API god_status god_seed_harness(const god_params* prm, const uint8_t* orig, const uint8_t* mut,
                                    const uint64_t* offsets, uint32_t n_pairs, uint64_t* edit, uint64_t* matches,
                                    uint64_t* totals, uint32_t* god_phase, god_stream stream) {
  return guarded([&] {
    const Params P = make_params(prm);
    GOD_REQUIRE(offsets && (n_pairs == 0 || (orig && mut && edit && matches && totals && god_phase)), "NULL argument");
    uint32_t x = 0;
    for (int j = 0; j < P.k; j++) x += (uint32_t)((P.pat.bits >> (j % P.pat.p)) & 1ull);
    GOD_REQUIRE(x <= 28, "spaced mask weight must be <= 28");
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<uint64_t> hoff((size_t)n_pairs + 1);
    if (is_device_ptr(offsets))
      GOD_CUDA(cudaMemcpyAsync(hoff.data(), offsets, hoff.size() * 8, cudaMemcpyDeviceToHost, st));
    else
      memcpy(hoff.data(), offsets, hoff.size() * 8);
    GOD_CUDA(cudaStreamSynchronize(st));
    for (uint32_t i = 0; i < n_pairs; i++)
      GOD_REQUIRE(hoff[i] <= hoff[i + 1] && hoff[i + 1] - hoff[i] <= god::harness_max_len(),
                  "pairs must be <= 4096 bases (and offsets ascending)");
    Scratch scr(st);
    Stage sg(st, scr);
    const uint64_t L = hoff[n_pairs];
    const uint8_t* da = sg.in(orig, L);
    const uint8_t* db = sg.in(mut, L);
    const uint64_t* doff = sg.in(offsets, (size_t)n_pairs + 1);
    uint64_t* de = sg.out(edit, n_pairs);
    uint64_t* dm = sg.out(matches, 4ull * n_pairs);
    uint64_t* dt = sg.out(totals, 4ull * n_pairs);
    uint32_t* dp = sg.out(god_phase, n_pairs);
    god::seed_harness(P, da, db, doff, n_pairs, de, dm, dt, dp, st);
    sg.finish();
  });
}

GOD_API god_status god_harness_accepted(const uint64_t* edit, const uint64_t* matches, const uint64_t* totals,
                                        uint32_t n_pairs, const uint64_t* thresholds, uint32_t n_thresholds,
                                        uint64_t* accepted, god_stream stream) {
  return guarded([&] {
    GOD_REQUIRE(n_thresholds == 0 || (thresholds && accepted), "NULL argument");
    GOD_REQUIRE(n_pairs == 0 || (edit && matches && totals), "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    Scratch scr(st);
    Stage sg(st, scr);
    const uint64_t* de = sg.in(edit, n_pairs);
    const uint64_t* dm = sg.in(matches, 4ull * n_pairs);
    const uint64_t* dt = sg.in(totals, 4ull * n_pairs);
    const uint64_t* dE = sg.in(thresholds, n_thresholds);
    uint64_t* da = sg.out(accepted, 4ull * n_thresholds);
    god::harness_accepted(de, dm, dt, n_pairs, dE, n_thresholds, da, st);
    sg.finish();
  });
}

}  // extern "C"
