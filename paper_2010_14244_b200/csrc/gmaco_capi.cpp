// gmaco_capi.cpp — host C++ engine behind the C ABI of include/gmaco.h.
//
// Mirrors the reference's executor contract: gmaco_create ≈ init_world
// (engine.cpp:116-144) on the device, gmaco_step ≈ sequential_step
// (engine.cpp:352-400) / ParallelRunner::step (parallel.cpp:123-193),
// gmaco_collect ≈ collect_result (engine.cpp:402-433).  Setup (validation,
// CSR build, spawn, initial pheromone) runs on the host exactly as the
// reference does it; every per-step stage runs in sm_100a kernels
// (kernels.cu), replayed as CUDA graphs of `kGraphSteps` steps.  There is no
// CPU execution path: without a CUDA device gmaco_create fails with status 2.

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <tuple>
#include <unordered_map>
#include <mutex>
#include <cstdio>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <queue>
#include <stdexcept>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "device.cuh"
#include "gmaco.h"
#include "kernels.h"
#include "nccl.h"
#include "nvtx3/nvToolsExt.h"

namespace gmaco {
namespace {

struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string fmt(const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}

#define CK(call)                                                                                \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                               #call);                                                          \
  } while (0)

constexpr int kGraphSteps = 32;
constexpr int64_t kCostCap = (int64_t(1) << 53) - 1;

int64_t tau_from_double(double v) { return std::llround(v * 1e6); }  // pheromone.hpp:18

// ---- host graph (RoadNetwork ctor semantics, net.cpp:38-98) ---------------
struct HostGraph {
  int32_t n = 0, m = 0;
  std::vector<int32_t> from, to, lanes;
  std::vector<int64_t> len;
  std::vector<uint8_t> sig;
  std::vector<int32_t> out_ptr, out_nbr, out_edge;  // CSR sorted by neighbour
  std::vector<int32_t> in_ptr, in_edge;             // ascending edge id
  std::vector<int32_t> edge_slot;                   // edge id -> slot
};

void build_graph(const gmaco_graph_desc* d, HostGraph& g) {
  if (!d) throw ValidationError("graph descriptor is null");
  const int32_t n = d->node_count, m = d->edge_count;
  if (n <= 0) throw ValidationError("network has no nodes");
  if (m < 0) throw ValidationError("network edge count must be >= 0");
  for (int32_t e = 0; e < m; ++e) {  // net.cpp:58-79, input order
    if (d->edge_from[e] < 0 || d->edge_from[e] >= n)
      throw ValidationError(fmt("edge %d references missing node %d", e, d->edge_from[e]));
    if (d->edge_to[e] < 0 || d->edge_to[e] >= n)
      throw ValidationError(fmt("edge %d references missing node %d", e, d->edge_to[e]));
    if (d->edge_from[e] == d->edge_to[e])
      throw ValidationError(fmt("edge %d is a self-loop at node %d", e, d->edge_from[e]));
    if (d->edge_length_mm[e] <= 0) throw ValidationError(fmt("edge %d has nonpositive length", e));
    if (d->edge_lanes && d->edge_lanes[e] < 1) throw ValidationError(fmt("edge %d has lanes < 1", e));
  }
  g.n = n;
  g.m = m;
  g.from.assign(d->edge_from, d->edge_from + m);
  g.to.assign(d->edge_to, d->edge_to + m);
  g.len.assign(d->edge_length_mm, d->edge_length_mm + m);
  g.lanes.resize(m);
  for (int32_t e = 0; e < m; ++e) g.lanes[e] = d->edge_lanes ? d->edge_lanes[e] : 1;
  g.sig.resize(n);
  for (int32_t i = 0; i < n; ++i) g.sig[i] = d->signalized ? d->signalized[i] : 0;
  g.out_ptr.assign(n + 1, 0);
  g.in_ptr.assign(n + 1, 0);
  for (int32_t e = 0; e < m; ++e) {
    g.out_ptr[g.from[e] + 1]++;
    g.in_ptr[g.to[e] + 1]++;
  }
  for (int32_t u = 0; u < n; ++u) {
    g.out_ptr[u + 1] += g.out_ptr[u];
    g.in_ptr[u + 1] += g.in_ptr[u];
  }
  g.out_nbr.resize(m);
  g.out_edge.resize(m);
  g.in_edge.resize(m);
  std::vector<int32_t> oc(g.out_ptr.begin(), g.out_ptr.end() - 1), ic(g.in_ptr.begin(), g.in_ptr.end() - 1);
  for (int32_t e = 0; e < m; ++e) {
    g.out_nbr[oc[g.from[e]]] = g.to[e];
    g.out_edge[oc[g.from[e]]++] = e;
    g.in_edge[ic[g.to[e]]++] = e;
  }
  // rows sorted by neighbour id, stable (input order among equal ids, which
  // are then rejected): an in-place insertion sort -- rows are short, and
  // std::stable_sort allocates a buffer per call (~50 us per 1k-node create)
  std::vector<std::pair<int32_t, int32_t>> tmp;
  for (int32_t u = 0; u < n; ++u) {
    const int32_t b = g.out_ptr[u], end = g.out_ptr[u + 1];
    if (end - b > 64) {  // (a hub: the engine rejects it later, kMaxDegree) sort it in O(d log d)
      tmp.clear();
      for (int32_t k = b; k < end; ++k) tmp.emplace_back(g.out_nbr[k], g.out_edge[k]);
      std::stable_sort(tmp.begin(), tmp.end(), [](auto& x, auto& y) { return x.first < y.first; });
      for (int32_t k = b; k < end; ++k) {
        g.out_nbr[k] = tmp[k - b].first;
        g.out_edge[k] = tmp[k - b].second;
      }
    }
    for (int32_t k = b + 1; k < end; ++k) {
      const int32_t nb = g.out_nbr[k], ed = g.out_edge[k];
      int32_t j = k;
      for (; j > b && g.out_nbr[j - 1] > nb; --j) {
        g.out_nbr[j] = g.out_nbr[j - 1];
        g.out_edge[j] = g.out_edge[j - 1];
      }
      g.out_nbr[j] = nb;
      g.out_edge[j] = ed;
    }
    for (int32_t k = b + 1; k < end; ++k)
      if (g.out_nbr[k] == g.out_nbr[k - 1])  // net.cpp:89-93
        throw ValidationError(fmt("duplicate edge between nodes %d and %d", u, g.out_nbr[k]));
  }
  g.edge_slot.resize(m);
  for (int32_t s = 0; s < m; ++s) g.edge_slot[g.out_edge[s]] = s;
}

// ---- config validation (engine.cpp:12-32 + param validate()s) -------------
void validate_config(const gmaco_sim_config* c) {
  if (!c) throw ValidationError("config is null");
  if (c->vehicle_count < 1) throw ValidationError("config: vehicle_count must be >= 1");
  if (c->options.flags >> 12) throw ValidationError("options: unknown flag bits");
  if (!(c->options.sssp_delta >= 0)) throw ValidationError("options: sssp_delta must be >= 0");
  if (!(c->dt_s > 0)) throw ValidationError("config: dt must be positive");
  if (c->max_steps < 0) throw ValidationError("config: max_steps must be >= 0");
  if (c->decision_latency_s < 0) throw ValidationError("config: decision_latency_s must be >= 0");
  if (c->spawn == GMACO_UNIFORM_WINDOW && c->spawn_window_steps < 1)
    throw ValidationError("config: spawn_window_steps must be >= 1");
  if (c->speed_min_mps <= 0 || c->speed_max_mps < c->speed_min_mps)
    throw ValidationError("config: speed range must satisfy 0 < min <= max");
  if (c->od_pattern == GMACO_OD_BLOCKS) {
    if (c->od_bias < 0 || c->od_bias > 1) throw ValidationError("config: od bias must lie in [0, 1]");
    if (c->od_block_a_len <= 0 || c->od_block_b_len <= 0)
      throw ValidationError("config: od blocks must be non-empty");
  }
  const gmaco_pheromone_params& p = c->pheromone;  // pheromone.cpp:9-19
  if (!(p.tau_min <= p.tau_init_lo && p.tau_init_lo <= p.tau_init_hi && p.tau_init_hi <= p.tau_max))
    throw ValidationError("pheromone init range must satisfy tau_min <= lo <= hi <= tau_max");
  if (p.delta_inc <= 0 || p.delta_dec <= 0)
    throw ValidationError("pheromone delta_inc and delta_dec must be positive");
  if (p.rho < 0 || p.rho >= 1) throw ValidationError("pheromone rho must lie in [0, 1)");
  if (p.tau_min < 0) throw ValidationError("pheromone tau_min must be >= 0");
  const gmaco_signal_params& s = c->signal;  // signals.cpp:8-21
  if (s.th_max < 1) throw ValidationError("signal th_max must be >= 1");
  if (s.t_max <= 0) throw ValidationError("signal t_max must be positive");
  if (s.green_duration_s <= 0) throw ValidationError("signal green_duration must be positive");
  if (s.saturation_flow <= 0) throw ValidationError("signal saturation_flow must be positive");
  bool seen[kPhases] = {};
  for (int i = 0; i < kPhases; ++i) {
    const int ph = s.fixed_cycle_order[i];
    if (ph < 0 || ph >= kPhases || seen[ph])
      throw ValidationError("signal fixed_cycle_order must be a permutation of 0..7");
    seen[ph] = true;
  }
  if (c->routing.deviation_threshold < 0)  // routing.cpp:9-14
    throw ValidationError("routing deviation_threshold must be >= 0");
  if (c->routing.aco_alpha < 0 || c->routing.aco_beta < 0)
    throw ValidationError("routing aco exponents must be >= 0");
  if (c->algorithm < GMACO_DIJKSTRA || c->algorithm > GMACO_COLONY)
    throw ValidationError(fmt("config: unknown algorithm %d", c->algorithm));
  if (c->controller < GMACO_FIXED || c->controller > GMACO_PREEMPTIVE)
    throw ValidationError(fmt("config: unknown controller %d", c->controller));
  if (c->algorithm == GMACO_COLONY) {
    const gmaco_colony_params& k = c->colony;
    if (k.ants < 1) throw ValidationError("colony: ants must be >= 1");
    if (k.ants > 1024) throw ValidationError("colony: ants must be <= 1024");
    if (k.hop_limit < 0 || k.max_hops < 0) throw ValidationError("colony: hop limits must be >= 0");
    if (k.rng != GMACO_RNG_PHILOX && k.rng != GMACO_RNG_REFERENCE) throw ValidationError("colony: unknown rng");
    if (k.deposit < GMACO_DEPOSIT_COMPLETION || k.deposit > GMACO_DEPOSIT_NONE)
      throw ValidationError("colony: unknown deposit mode");
  }
}

// ---- Dijkstra to a destination over reversed edges (net.cpp:359-383) ------
void reverse_csr(const HostGraph& g, std::vector<int32_t>& rptr, std::vector<int32_t>& rsrc,
                 std::vector<int32_t>& redge) {
  rptr.assign(g.n + 1, 0);
  rsrc.resize(g.m);
  redge.resize(g.m);
  for (int32_t e = 0; e < g.m; ++e) rptr[g.to[e] + 1]++;
  for (int32_t u = 0; u < g.n; ++u) rptr[u + 1] += rptr[u];
  std::vector<int32_t> c(rptr.begin(), rptr.end() - 1);
  for (int32_t e = 0; e < g.m; ++e) {
    rsrc[c[g.to[e]]] = g.from[e];
    redge[c[g.to[e]]++] = e;
  }
}

// ---- create-phase profiler (options.flags & GMACO_OPT_PROFILE_CREATE prints to stderr)
struct PhaseTimer {
  bool on = false;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gmaco create] %-28s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// ---- device buffers --------------------------------------------------------
// Process-wide pinned host memory: cudaMallocHost costs milliseconds per
// call, so engines take blocks from 4 MiB slabs and return them on destroy.
class PinnedPool {
 public:
  static void* take(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    std::lock_guard<std::mutex> lk(mu());
    auto& fr = free_list();
    for (size_t i = 0; i < fr.size(); ++i)
      if (fr[i].second >= bytes) {
        void* p = fr[i].first;
        if (fr[i].second > bytes) {
          fr[i].first = static_cast<char*>(p) + bytes;
          fr[i].second -= bytes;
        } else {
          fr.erase(fr.begin() + i);
        }
        sizes()[p] = bytes;
        return p;
      }
    const size_t slab = std::max(bytes, size_t(4) << 20);
    void* s = nullptr;
    // mapped: kernels write readbacks straight into it (k_pack)
    CK(cudaHostAlloc(&s, slab, cudaHostAllocMapped | cudaHostAllocPortable));
    if (slab > bytes) fr.emplace_back(static_cast<char*>(s) + bytes, slab - bytes);
    sizes()[s] = bytes;
    return s;
  }
  static void give(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu());
    auto it = sizes().find(p);
    if (it == sizes().end()) return;
    free_list().emplace_back(p, it->second);
    sizes().erase(it);
  }

 private:
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::vector<std::pair<void*, size_t>>& free_list() {
    static auto* v = new std::vector<std::pair<void*, size_t>>();  // process lifetime
    return *v;
  }
  static std::unordered_map<void*, size_t>& sizes() {
    static auto* m = new std::unordered_map<void*, size_t>();
    return *m;
  }
};

// Process-wide pool of non-blocking streams per device: creating one costs
// tens of microseconds of gmaco_create; engines created one after another
// (the bench legs, the tests, a harness matrix) reuse them.
class StreamPool {
 public:
  static cudaStream_t take(int device) {
    {
      std::lock_guard<std::mutex> lk(mu());
      auto& v = free_list()[device];
      if (!v.empty()) {
        cudaStream_t s = v.back();
        v.pop_back();
        return s;
      }
    }
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return s;
  }
  static void give(int device, cudaStream_t s) {  // the caller has synchronized it
    if (!s) return;
    std::lock_guard<std::mutex> lk(mu());
    free_list()[device].push_back(s);
  }

 private:
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::map<int, std::vector<cudaStream_t>>& free_list() {
    static auto* m = new std::map<int, std::vector<cudaStream_t>>();  // process lifetime
    return *m;
  }
};

// Device allocations of one engine.  Direct mode (default): one cudaMalloc
// and one synchronous copy per array.  Arena mode (build_world): arrays under
// kArenaMax are sub-allocated (256-B aligned) from kChunk device chunks and
// their contents are written into a host shadow of each chunk; flush() sends
// every chunk in one copy.  gmaco_create then costs a handful of CUDA calls
// instead of ~100 mallocs and synchronous copies.  Until flush() no kernel
// may touch arena memory and no other writer may target it.
struct DevBuffers {
  static constexpr size_t kChunk = size_t(8) << 20, kArenaMax = size_t(1) << 20, kAlign = 256;
  struct Chunk {
    char* dev = nullptr;
    // pinned host shadow from the process-wide pool (reused across engines:
    // no page faults on first touch, and the flush is a true async DMA);
    // uninitialized: only written ranges are touched / sent
    char* shadow = nullptr;
    size_t used = 0, sent = 0;  // [sent, used) not yet on the device
  };
  std::vector<void*> ptrs;
  std::vector<Chunk> chunks;
  bool arena = false;
  cudaStream_t stream = nullptr;  // flushes are ordered on the engine stream
  // Always a dedicated allocation: for arrays a kernel writes before seal()
  // (a later flush of the arena must never overwrite them).
  template <class T>
  T* alloc_direct(size_t n) {
    return static_cast<T*>(raw_alloc(std::max<size_t>(n, 1) * sizeof(T)));
  }
  // Stream-ordered allocations from the device's default pool, which keeps
  // up to kPoolKeep of freed memory: engines created one after another (the
  // bench legs, the tests) reuse it instead of paying cudaMalloc per array.
  static constexpr uint64_t kPoolKeep = uint64_t(4) << 30;
  // Checked builds of a world (GMACO_OPT_REDZONES): every allocation gets
  // kRedzone guard bytes of kRedzoneByte before and after it (arena arrays:
  // after), verified by gmaco_debug_check_redzones -- this engine's own
  // memcheck for out-of-bounds writes (compute-sanitizer is not available on
  // the GPU pool).
  static constexpr size_t kRedzone = 1024;
  static constexpr unsigned char kRedzoneByte = 0xA5;
  bool redzones = false;
  std::vector<std::pair<const char*, size_t>> zones;  // device guard ranges
  void* raw_alloc(size_t bytes, bool guard = true) {
    const size_t rz = redzones && guard ? kRedzone : 0;
    char* base = static_cast<char*>(raw_alloc_base(bytes + 2 * rz));
    if (rz) {
      CK(cudaMemsetAsync(base, kRedzoneByte, rz, stream));
      CK(cudaMemsetAsync(base + rz + bytes, kRedzoneByte, rz, stream));
      CK(cudaStreamSynchronize(stream));
      zones.emplace_back(base, rz);
      zones.emplace_back(base + rz + bytes, rz);
    }
    return base + rz;
  }
  void* raw_alloc_base(size_t bytes) {
    static thread_local int configured_dev = -1;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (configured_dev != dev) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = kPoolKeep;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      configured_dev = dev;
    }
    void* p = nullptr;
    if (bytes >= kPoolMax) {  // huge (tour scratch, distance tables): plain allocation, not pooled
      CK(cudaMalloc(&p, bytes));
      big.push_back(p);
      return p;
    }
    // (the pointer freed later is the base, the one pushed here)
    CK(cudaMallocAsync(&p, bytes, stream));
    CK(cudaStreamSynchronize(stream));  // usable by any stream / host call right away
    ptrs.push_back(p);
    return p;
  }
  static constexpr size_t kPoolMax = size_t(256) << 20;
  std::vector<void*> big;
  template <class T>
  T* alloc(size_t n) {
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    if (arena && bytes <= kArenaMax) return static_cast<T*>(carve(bytes, nullptr));
    return static_cast<T*>(raw_alloc(bytes));
  }
  template <class T>
  T* upload(const std::vector<T>& h) {
    const size_t bytes = h.size() * sizeof(T);
    if (arena && bytes && bytes <= kArenaMax) {
      T* d = static_cast<T*>(carve(bytes, nullptr));
      std::memcpy(shadow_of(d), h.data(), bytes);
      return d;
    }
    T* d = alloc<T>(h.size());
    if (!h.empty()) {  // complete before returning: a pageable cudaMemcpy may return with its DMA in
                       // flight, unordered with later kernels on a non-blocking engine stream
      CK(cudaMemcpyAsync(d, h.data(), bytes, cudaMemcpyHostToDevice, stream));
      CK(cudaStreamSynchronize(stream));
    }
    return d;
  }
  template <class T>
  T* filled(size_t n, T value) {
    const size_t bytes = n * sizeof(T);
    if (arena && bytes && bytes <= kArenaMax) {  // straight into the shadow (no temporary)
      T* d = static_cast<T*>(carve(bytes, nullptr));
      T* sh = reinterpret_cast<T*>(shadow_of(d));
      std::fill(sh, sh + n, value);
      return d;
    }
    std::vector<T> h(n, value);
    return upload(h);
  }
  template <class T>
  T* upload_one(const T& v) {
    return upload(std::vector<T>{v});
  }
  // Starts the copies of every arena chunk's not-yet-sent range (stream-
  // ordered, no wait): the DMA overlaps the host work that fills the next
  // ranges.  A shadow range is written only when it is carved (upload /
  // filled), so a range once sent is never written on the host again.
  void flush_async() {
    for (auto& ch : chunks)
      if (ch.used > ch.sent) {
        CK(cudaMemcpyAsync(ch.dev + ch.sent, ch.shadow + ch.sent, ch.used - ch.sent, cudaMemcpyHostToDevice,
                           stream));
        ch.sent = ch.used;
        pending = true;
      }
  }
  bool pending = false;  // copies started by flush_async, not yet waited for
  // Sends every arena chunk's not-yet-sent range to the device (one copy per
  // chunk); ranges already sent are device-authoritative from then on.
  void flush() {
    bool any = pending;
    pending = false;
    for (auto& ch : chunks)
      if (ch.used > ch.sent) {
        CK(cudaMemcpyAsync(ch.dev + ch.sent, ch.shadow + ch.sent, ch.used - ch.sent, cudaMemcpyHostToDevice,
                           stream));
        ch.sent = ch.used;
        any = true;
      }
    if (any) CK(cudaStreamSynchronize(stream));
  }
  void seal() {
    flush();  // (synchronizes: the DMA from the shadows is complete)
    for (auto& ch : chunks) {
      PinnedPool::give(ch.shadow);
      ch.shadow = nullptr;
    }
    arena = false;
  }
  // Back to the pool, ordered after the owner's work on `stream` (call
  // before that stream is destroyed).
  void release() {
    for (void* p : ptrs) cudaFreeAsync(p, stream);
    for (auto& ch : chunks) cudaFreeAsync(ch.dev, stream);
    if (!ptrs.empty() || !chunks.empty() || !big.empty()) cudaStreamSynchronize(stream);
    for (auto& ch : chunks) PinnedPool::give(ch.shadow);  // (a build that failed before seal)
    for (void* p : big) cudaFree(p);
    ptrs.clear();
    chunks.clear();
    big.clear();
  }
  ~DevBuffers() { release(); }

 private:
  void* carve(size_t bytes, const void*) {
    const size_t rz = redzones ? kRedzone : 0;
    const size_t need = (bytes + rz + kAlign - 1) & ~(kAlign - 1);
    if (chunks.empty() || chunks.back().used + need > kChunk) {
      Chunk ch;
      ch.dev = static_cast<char*>(raw_alloc(kChunk, /*guard=*/false));
      ptrs.pop_back();  // owned by the chunk list
      ch.shadow = static_cast<char*>(PinnedPool::take(kChunk));
      chunks.push_back(std::move(ch));
    }
    Chunk& ch = chunks.back();
    void* p = ch.dev + ch.used;
    if (rz) {  // trailing guard, sent with the chunk's next flush
      std::memset(ch.shadow + ch.used + bytes, kRedzoneByte, rz);
      zones.emplace_back(ch.dev + ch.used + bytes, rz);
    }
    ch.used += need;
    return p;
  }
  char* shadow_of(const void* d) {
    for (auto& ch : chunks)
      if (d >= ch.dev && d < ch.dev + kChunk) return ch.shadow + (static_cast<const char*>(d) - ch.dev);
    throw std::runtime_error("arena: pointer outside every chunk");
  }
};

// Exact tau^alpha table (DevWorld::taupow): pow(t / 1e6, alpha) by the
// host's glibc pow -- the call routing.cpp:93 makes -- for every pheromone
// value t in [lo, hi], across all host threads.  Skipped (nullptr: device pow,
// <= 1 ulp from glibc) when the range exceeds kTauPowMax entries.
constexpr int64_t kTauPowMax = int64_t(1) << 30;  // 8 GiB of the 180 GB HBM
const double* build_taupow(DevBuffers& B, int64_t lo, int64_t hi, double alpha, cudaStream_t st) {
  const int64_t n = hi - lo + 1;
  if (n <= 0 || n > kTauPowMax) return nullptr;
  double* host = nullptr;
  CK(cudaMallocHost(&host, n * sizeof(double)));
  const int nt = (int)std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (int k = 0; k < nt; ++k)
    th.emplace_back([=] {
      for (int64_t i = n * k / nt; i < n * (k + 1) / nt; ++i)
        host[i] = std::pow(static_cast<double>(lo + i) / 1e6, alpha);
    });
  for (auto& t : th) t.join();
  double* d = B.alloc_direct<double>((size_t)n);
  CK(cudaMemcpyAsync(d, host, n * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaFreeHost(host));
  return d;
}

template <class T>
std::vector<T> download(const T* d, size_t n) {
  std::vector<T> h(n);
  if (n) CK(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
  return h;
}

}  // namespace
}  // namespace gmaco

namespace gmaco {
// RoadNetwork ctor checks (net.cpp:38-98) on a descriptor, for the
// reference-schema loader / writer (netio.cpp).
bool validate_graph_desc(const gmaco_graph_desc* d, std::string* err) {
  try {
    HostGraph g;
    build_graph(d, g);
    return true;
  } catch (const ValidationError& e) {
    if (err) *err = e.what();
    return false;
  }
}
}  // namespace gmaco

using namespace gmaco;

struct gmaco_engine {
  std::string err;
  int device = 0;
  HostGraph g;
  gmaco_sim_config cfg{};
  int32_t S = 0;
  int32_t ell = 0, M = 0;            // slot space (ELL width, size)
  std::vector<int32_t> slot_edge;    // slot -> edge id (-1 padding)
  std::vector<int32_t> sig_node;
  DevBuffers buf;
  DevWorld w{};
  DevCtl* ctl = nullptr;
  DevCtl* ctl_host = nullptr;  // pinned mirror
  int64_t* stop_host = nullptr;
  int64_t stop_written = -1;  // last stop_at value enqueued to the device
  bool ctl_valid = false;     // ctl_host mirrors the device control block
  bool pending = false;       // steps enqueued without a host sync
  void* stage = nullptr;      // pinned staging for batched device->host reads
  size_t stage_bytes = 0;
  // double-buffered readback slots (gmaco_vehicles_enqueue / _wait)
  struct ReadSlot {
    void* buf = nullptr;
    size_t bytes = 0;
    cudaEvent_t done = nullptr;
    cudaGraphExec_t snap_graph = nullptr;  // gmaco_step_snapshot: one step + this slot's gather
    PackDesc snap_pd;
    std::vector<std::pair<size_t, size_t>> fields;  // (staging offset, bytes) per requested field, view order
    size_t oe_off = 0;
    uint32_t mask = 0;  // which view members the snapshot holds (view_mask)
    bool on_edge = false, armed = false;
    bool pd_valid = false;  // pd_cache is this slot's gather for field set pd_mask
    uint32_t pd_mask = 0;
    PackDesc pd_cache;
    // small worlds: the gather runs in the step's finalizing tail block
    // (DevWorld::snap) from this device copy of the descriptor
    PackDesc* pd_dev = nullptr;
    PackDesc pd_dev_val;
    bool pd_dev_set = false;
    // pinned source of the descriptor's stream-ordered upload; pd_copied
    // marks that upload's completion (the staging is rewritten only after it)
    PackDesc* pd_host = nullptr;
    cudaEvent_t pd_copied = nullptr;
    cudaGraphExec_t tail_snap_graph = nullptr;  // one step with the in-tail gather of this slot
  } rslot[2];
  StepResources res;
  cudaStream_t stream = nullptr;
  cudaGraphExec_t graph_big = nullptr, graph_one = nullptr;
  cudaGraphExec_t tgraph_big = nullptr, tgraph_one = nullptr;
  cudaGraphExec_t graph_walk = nullptr, graph_tail = nullptr;  // bench split
  // bench graph: [L2 flush memset] -> ev0 -> step (walk, ev1, tail) -> ev2; the
  // three event-record nodes are retargeted per launch to that step's events
  cudaGraph_t bench_tmpl = nullptr;
  cudaGraphExec_t bench_exec = nullptr;
  cudaGraphNode_t bench_ev_node[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t bench_ev[3] = {nullptr, nullptr, nullptr};
  int64_t bench_flush = -1;
  int bench_mode = 0;
  void* flush = nullptr;
  int64_t flush_bytes = 0;
  std::vector<cudaEvent_t> ev_begin, ev_end;  // timing mode, kGraphSteps pairs
  bool timing = false;
  double last_walk_ms = 0.0, last_step_ms = 0.0;
  int64_t last_walk_launches = 0;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  int64_t wall_ms = 0;
  int64_t direct_steps = 0;  // steps launched without a graph (run_steps, kDirectSteps)
  // multi-GPU
  int32_t rank = 0, world = 1, shard_pad = 0;
  // by-target sharding: node -> target table (TARGETS distances), the
  // allgather send / receive buffers and the received record -> vehicle map
  std::vector<int32_t> target_of_node;
  int32_t* xsend = nullptr;
  int32_t* xrecv = nullptr;
  int32_t* xgath = nullptr;
  ncclComm_t comm = nullptr;

  ~gmaco_engine() {
    if (device >= 0) cudaSetDevice(device);
    // settle every enqueued step / snapshot gather first: k_pack may still be
    // writing into the mapped pinned slots handed back to the pool below
    if (stream) cudaStreamSynchronize(stream);
    if (bench_exec) cudaGraphExecDestroy(bench_exec);
    if (bench_tmpl) cudaGraphDestroy(bench_tmpl);
    for (auto e : bench_ev)
      if (e) cudaEventDestroy(e);
    for (auto ge : {graph_big, graph_one, tgraph_big, tgraph_one, graph_walk, graph_tail})
      if (ge) cudaGraphExecDestroy(ge);
    if (flush) cudaFree(flush);
    for (auto e : ev_begin) cudaEventDestroy(e);
    for (auto e : ev_end) cudaEventDestroy(e);
    if (ev_a) cudaEventDestroy(ev_a);
    if (ev_b) cudaEventDestroy(ev_b);
    PinnedPool::give(ctl_host);
    // stop_host lives inside the ctl_host pinned block
    PinnedPool::give(stage);
    for (auto& s : rslot) {
      PinnedPool::give(s.buf);
      if (s.done) cudaEventDestroy(s.done);
      if (s.pd_copied) cudaEventDestroy(s.pd_copied);
      PinnedPool::give(s.pd_host);
      if (s.snap_graph) cudaGraphExecDestroy(s.snap_graph);
      if (s.tail_snap_graph) cudaGraphExecDestroy(s.tail_snap_graph);
    }
    buf.release();  // stream-ordered frees need the stream alive
    if (stream) StreamPool::give(device, stream);  // (synchronized at the top of the destructor)
    destroy_comm();
  }
  void destroy_comm();
  void reset_graphs() {
    for (auto* ge : {&graph_big, &graph_one, &tgraph_big, &tgraph_one, &graph_walk, &graph_tail, &rslot[0].snap_graph,
                     &rslot[1].snap_graph, &rslot[0].tail_snap_graph, &rslot[1].tail_snap_graph})
      if (*ge) {
        cudaGraphExecDestroy(*ge);
        *ge = nullptr;
      }
  }
};

namespace {

thread_local std::string g_create_err;

// NVTX range per C-ABI entry point (SURVEY §5 tracing): a no-op unless a
// profiler (nsys / ncu with NVTX filtering) attaches.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <class F>
int guarded(gmaco_engine* h, F&& f, bool stream_ordered = false) {
  try {
    if (h) CK(cudaSetDevice(h->device));
    // steps enqueued by gmaco_step(executed = NULL) may still be running on
    // the (non-blocking) engine stream: settle them before any entry point
    // that reads or writes device state outside that stream's order
    if (h && h->pending && !stream_ordered) {
      CK(cudaStreamSynchronize(h->stream));
      h->pending = false;
    }
    f();
    return GMACO_OK;
  } catch (const ValidationError& e) {
    (h ? h->err : g_create_err) = e.what();
    return GMACO_EVALIDATION;
  } catch (const std::exception& e) {
    (h ? h->err : g_create_err) = e.what();
    return GMACO_ERUNTIME;
  }
}

// ---- spawn_vehicles (engine.cpp:71-114), pool indexed not materialized ----
struct Spawned {
  std::vector<int32_t> origin, dest;
  std::vector<double> speed;
  std::vector<int64_t> advance, depart;
};

uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// The reference's draw(seed, stream, b, c) = mix64(mix64(mix64(mix64(seed) ^
// stream) ^ b) ^ c) (include/macosim/rng.hpp:28-40), with the (seed, stream)
// prefix of the chain computed once: the per-entity loops at create draw
// thousands of times per stream.
struct DrawStream {
  uint64_t h;
  DrawStream(uint64_t seed, uint64_t a) : h(mix64(mix64(seed) ^ a)) {}
  uint64_t operator()(uint64_t b, uint64_t c = 0) const { return mix64(mix64(h ^ b) ^ c); }
};
double to_unit(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }
double uniform(uint64_t bits, double lo, double hi) { return lo + to_unit(bits) * (hi - lo); }
uint64_t below(uint64_t bits, uint64_t n) {
  return static_cast<uint64_t>((static_cast<unsigned __int128>(bits) * n) >> 64);
}

struct DistHost {  // host view of the distance service (spawn reachability)
  int kind = 0;
  int32_t n = 0, cols = 0;
  int64_t grid_len = 0;
  // table kinds: reach[x * reach_words + t/64] bit t%64 = dist(x, row t) != inf
  const std::vector<uint64_t>* reach = nullptr;
  int64_t reach_words = 0;
  const std::vector<int32_t>* slot_of = nullptr;
  bool reachable(int32_t u, int32_t v) const {
    if (kind == GMACO_DIST_GRID) return true;  // a validated lattice is strongly connected
    const int32_t s = slot_of ? (*slot_of)[v] : v;
    if (s < 0) return false;
    return ((*reach)[(size_t)u * reach_words + (s >> 6)] >> (s & 63)) & 1u;
  }
};

Spawned spawn(const gmaco_sim_config& c, const HostGraph& g, const DistHost& dh,
              const std::vector<int32_t>& targets) {
  const int32_t n = g.n;
  std::vector<int32_t> dests;
  if (dh.kind == GMACO_DIST_TARGETS) {
    dests = targets;
    std::sort(dests.begin(), dests.end());
  }
  const int32_t nd = dh.kind == GMACO_DIST_TARGETS ? (int32_t)dests.size() : n;
  std::vector<int64_t> prefix(n + 1, 0);
  for (int32_t u = 0; u < n; ++u) {
    int64_t cnt = 0;
    if (dh.kind == GMACO_DIST_GRID) {
      cnt = n - 1;
    } else {
      for (int32_t j = 0; j < nd; ++j) {
        const int32_t v = dests.empty() ? j : dests[j];
        if (u != v && dh.reachable(u, v)) ++cnt;
      }
    }
    prefix[u + 1] = prefix[u] + cnt;
  }
  const int64_t pool = prefix[n];
  if (pool == 0) throw ValidationError("spawn: network has no reachable origin/destination pair");
  std::vector<std::pair<int32_t, int32_t>> ab, ba;
  auto block_pairs = [&](const int32_t* a, int32_t na, const int32_t* b, int32_t nb, auto& out) {
    for (int32_t i = 0; i < na; ++i)  // engine.cpp:59-66
      for (int32_t j = 0; j < nb; ++j)
        if (a[i] != b[j] && dh.reachable(a[i], b[j])) out.emplace_back(a[i], b[j]);
  };
  if (c.od_pattern == GMACO_OD_BLOCKS) {
    for (int32_t i = 0; i < c.od_block_a_len; ++i)
      if (c.od_block_a[i] < 0 || c.od_block_a[i] >= n) throw ValidationError("config: od block node out of range");
    for (int32_t i = 0; i < c.od_block_b_len; ++i)
      if (c.od_block_b[i] < 0 || c.od_block_b[i] >= n) throw ValidationError("config: od block node out of range");
    block_pairs(c.od_block_a, c.od_block_a_len, c.od_block_b, c.od_block_b_len, ab);
    block_pairs(c.od_block_b, c.od_block_b_len, c.od_block_a, c.od_block_a_len, ba);
  }
  Spawned s;
  const int32_t V = c.vehicle_count;
  s.origin.resize(V);
  s.dest.resize(V);
  s.speed.resize(V);
  s.advance.resize(V);
  s.depart.assign(V, 0);
  const DrawStream od(c.seed, 2), sp(c.seed, 3), dep(c.seed, 4);
  for (int32_t vid = 0; vid < V; ++vid) {
    const std::vector<std::pair<int32_t, int32_t>>* biased = nullptr;
    if (c.od_pattern == GMACO_OD_BLOCKS) {  // engine.cpp:88-97
      const double r = to_unit(od(vid, 0));
      if (r < c.od_bias) {
        const bool forward = to_unit(od(vid, 1)) < 0.5;
        const auto& b = forward ? ab : ba;
        if (!b.empty()) biased = &b;
      }
    }
    const uint64_t bits = od(vid, 2);
    if (biased) {
      const auto& pr = (*biased)[below(bits, biased->size())];
      s.origin[vid] = pr.first;
      s.dest[vid] = pr.second;
    } else {
      const int64_t idx = (int64_t)below(bits, (uint64_t)pool);
      // (grid: every node has n - 1 destinations)
      const int32_t u = dh.kind == GMACO_DIST_GRID
                            ? (int32_t)(idx / (n - 1))
                            : (int32_t)(std::upper_bound(prefix.begin(), prefix.end(), idx) - prefix.begin()) - 1;
      int64_t r = idx - prefix[u];
      int32_t v = -1;
      if (dh.kind == GMACO_DIST_GRID) {
        v = (int32_t)(r + (r >= u));
      } else {
        for (int32_t j = 0; j < nd; ++j) {
          const int32_t cand = dests.empty() ? j : dests[j];
          if (u != cand && dh.reachable(u, cand)) {
            if (r == 0) {
              v = cand;
              break;
            }
            --r;
          }
        }
      }
      s.origin[vid] = u;
      s.dest[vid] = v;
    }
    s.speed[vid] = uniform(sp(vid), c.speed_min_mps, c.speed_max_mps);  // engine.cpp:103-105
    s.advance[vid] = std::llround(s.speed[vid] * c.dt_s * 1000.0);
    if (c.spawn == GMACO_UNIFORM_WINDOW)
      s.depart[vid] = (int64_t)below(dep(vid), (uint64_t)c.spawn_window_steps);
  }
  return s;
}

// The device is required from here on (there is no CPU path): checked once,
// then the engine's stream and kernel attributes are set up.
void ensure_device(gmaco_engine* h) {
  if (h->stream) return;
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    throw std::runtime_error("no CUDA device available (the engine has no CPU path)");
  CK(cudaSetDevice(h->device));
  h->stream = StreamPool::take(h->device);
  h->buf.stream = h->stream;
  static std::mutex mu;  // kernel attributes are per device and process: set them once
  static std::vector<char> configured;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)configured.size() <= h->device) configured.resize(h->device + 1, 0);
  if (!configured[h->device]) {
    CK(configure_kernels());
    configured[h->device] = 1;
  }
}

// Exact distances dist(x -> dests[t]) for every node x on the device
// (all_pairs_distances / dijkstra_to results, net.cpp:359-437): returns the
// device table [T][n] (owned by B) and copies it to `host` for setup (spawn).
int64_t* device_distance_table(gmaco_engine* h, const HostGraph& g, const std::vector<int32_t>& dests,
                               std::vector<uint64_t>& reach, int64_t& reach_words) {
  const int32_t n = g.n, T = (int32_t)dests.size();
  const size_t total = (size_t)T * n;
  if (total >= (size_t(1) << 32)) throw ValidationError("distance table exceeds 2^32 entries");
  PhaseTimer pt;
  pt.on = (h->cfg.options.flags & GMACO_OPT_PROFILE_CREATE) != 0;
  DevBuffers& B = h->buf;
  std::vector<int32_t> rp, rs, re;
  reverse_csr(g, rp, rs, re);
  std::vector<int64_t> rl(g.m);
  for (int32_t k = 0; k < g.m; ++k) rl[k] = g.len[re[k]];
  DevBuffers tmp;  // scratch of the computation (frontiers, flags, reversed graph)
  SsspArgs a;
  a.n = n;
  a.rptr = tmp.upload(rp);
  a.rsrc = tmp.upload(rs);
  a.rlen = tmp.upload(rl);
  a.D = B.alloc_direct<int64_t>(total);  // written by kernels before the arena seal
  a.inq = tmp.alloc<uint32_t>(total);
  CK(cudaMemsetAsync(a.inq, 0, total * 4, h->stream));
  // near in/out and far cur/next lists (a state is in at most one list: inq)
  uint32_t* q[4] = {tmp.alloc<uint32_t>(total), tmp.alloc<uint32_t>(total), tmp.alloc<uint32_t>(total),
                    tmp.alloc<uint32_t>(total)};
  uint32_t* cnt = tmp.alloc<uint32_t>(4);
  const int32_t* ddests = tmp.upload(dests);
  CK(sssp_fill_seed(a.D, total, ddests, T, n, q[0], h->stream));
  CK(cudaStreamSynchronize(h->stream));
  pt.mark("sssp setup (reverse CSR, alloc)");
  // every round inside one persistent cooperative kernel (k_sssp_coop)
  // near/far threshold step: a few mean edge lengths (GMACO_SSSP_DELTA overrides, in edge lengths)
  int64_t lsum = 0;
  for (int32_t e = 0; e < g.m; ++e) lsum += g.len[e];
  const double mult = h->cfg.options.sssp_delta > 0 ? h->cfg.options.sssp_delta : 32.0;
  const int64_t delta = std::max<int64_t>(1, (int64_t)(mult * (double)lsum / std::max(1, g.m)));
  CK(cudaMemsetAsync(cnt, 0, 16, h->stream));
  CK(sssp_run_coop(a, q, cnt, (uint32_t)T, delta, h->device, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  pt.mark("sssp rounds");
  // spawn needs reachability only: a per-node bitmap over the table rows
  // (n * ceil(T/64) words) instead of the whole int64 table
  reach_words = (T + 63) / 64;
  uint64_t* rb = tmp.alloc<uint64_t>((size_t)n * reach_words);
  CK(build_reach_bits(a.D, T, n, reach_words, rb, h->stream));
  reach.resize((size_t)n * reach_words);
  CK(cudaMemcpyAsync(reach.data(), rb, reach.size() * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  pt.mark("reachability bitmap");
  return a.D;
}

// Per-target candidate rows for the ant-queue walker (DevTT, device.cuh).
// Built on the device from the progress-filter bitmaps: count record pairs
// per (target, row), scan, then metas and records.  Skipped (bitmap walker
// kept) when the tables would exceed their memory budget or the meta fields.
static void build_target_rows(gmaco_engine* h, const std::vector<int32_t>& place, int32_t T) {
  DevWorld& w = h->w;
  DevBuffers& B = h->buf;
  const int64_t n = w.g.n, TN = (int64_t)T * n;
  if (TN * 16 > (int64_t(8) << 30)) return;  // build temporaries + metas
  DevBuffers tmp;
  tmp.stream = h->stream;
  const int32_t* dplace = tmp.upload(place);
  int32_t* units = tmp.alloc_direct<int32_t>(TN);
  int64_t* offs = tmp.alloc_direct<int64_t>(TN + 1);
  CK(tt_count(w, T, dplace, units, h->stream));
  CK(tt_scan(units, offs, TN, h->stream));
  std::vector<int64_t> bnd(T + 1);  // table boundaries in pairs
  for (int32_t t = 0; t < T; ++t)
    CK(cudaMemcpyAsync(&bnd[t], offs + (int64_t)t * n, 8, cudaMemcpyDeviceToHost, h->stream));
  int32_t last = 0;
  CK(cudaMemcpyAsync(&bnd[T], offs + TN - 1, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(&last, units + TN - 1, 4, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  bnd[T] += last;
  for (int32_t t = 0; t < T; ++t)
    if (bnd[t + 1] - bnd[t] >= (int64_t(1) << 24)) return;  // 24-bit row offsets
  const int64_t nrec = 2 * (bnd[T] + 1);
  if (nrec >= (int64_t(1) << 31) || nrec * 24 > (int64_t(24) << 30)) return;
  w.tt.meta = B.alloc_direct<uint32_t>(TN);
  int64_t* base = B.alloc_direct<int64_t>(T);
  w.tt.T = T;
  w.tt.nch = (int32_t)((n + kTTChunk - 1) / kTTChunk);
  int64_t* cstart = B.alloc_direct<int64_t>((int64_t)T * (w.tt.nch + 1));
  CK(cudaMemcpyAsync(cstart + (int64_t)T * (w.tt.nch + 1) - 1, &nrec, 8, cudaMemcpyHostToDevice, h->stream));
  w.tt.rec = B.alloc_direct<int4>(nrec);
  int2* sm = B.alloc_direct<int2>(nrec);
  int64_t max_len = 0;
  for (int64_t L : h->g.len) max_len = std::max(max_len, L);
  int2* sl = max_len < (int64_t(1) << 31) ? B.alloc_direct<int2>(nrec) : nullptr;
  CK(tt_build(w, T, dplace, offs, const_cast<uint32_t*>(w.tt.meta), base, cstart, w.tt.rec, sm, sl, h->stream));
  w.tt.sl = sl;
  w.tt.base = base;
  w.tt.cstart = cstart;
  w.tt.sm = sm;
  w.tt.nrec = nrec;
  CK(tt_refresh(w, h->stream));
  CK(cudaStreamSynchronize(h->stream));
}

void build_world(gmaco_engine* h, const gmaco_graph_desc* gd, const gmaco_distance_desc* dd,
                 const gmaco_sim_config* cfg) {
  PhaseTimer pt0;
  pt0.on = cfg && (cfg->options.flags & GMACO_OPT_PROFILE_CREATE) != 0;
  build_graph(gd, h->g);
  validate_config(cfg);
  pt0.mark("graph + config validation");
  if (!dd) throw ValidationError("distance descriptor is null");
  HostGraph& g = h->g;
  const int32_t n = g.n, m = g.m;
  h->cfg = *cfg;
  gmaco_sim_config& c = h->cfg;
  const int alg = c.algorithm;
  for (int32_t u = 0; u < n; ++u)
    if (g.out_ptr[u + 1] - g.out_ptr[u] > kMaxDegree)
      throw ValidationError(fmt("node %d out-degree exceeds the engine bound of %d", u, kMaxDegree));

  DevBuffers& B = h->buf;
  B.redzones = (c.options.flags & GMACO_OPT_REDZONES) != 0;
  B.arena = true;  // sub-allocate + shadow small arrays; sealed (one copy per chunk) below
  DevWorld& w = h->w;
  PhaseTimer pt;
  pt.on = pt0.on;

  // ---- distance service ---------------------------------------------------
  DistHost dh;
  dh.kind = dd->kind;
  dh.n = n;
  std::vector<int64_t> table;  // user-supplied dense table only
  std::vector<uint64_t> reach;
  std::vector<int32_t> slot_of, targets;
  w.d.kind = dd->kind == GMACO_DIST_GRID ? 1 : 0;
  w.d.n = n;
  if (dd->kind == GMACO_DIST_DENSE) {
    if (dd->dist_mm) {
      table.resize((size_t)n * n);
      dh.reach_words = (n + 63) / 64;
      reach.assign((size_t)n * dh.reach_words, 0);
      for (int32_t u = 0; u < n; ++u)
        for (int32_t v = 0; v < n; ++v) {
          const int64_t dv = dd->dist_mm[(size_t)u * n + v];
          table[(size_t)v * n + u] = dv;
          if (dv != kInf) reach[(size_t)u * dh.reach_words + (v >> 6)] |= uint64_t(1) << (v & 63);
        }
    } else {  // all_pairs_distances (net.cpp:419-437): every node a destination, on the device
      ensure_device(h);
      std::vector<int32_t> all(n);
      for (int32_t d = 0; d < n; ++d) all[d] = d;
      w.d.table = device_distance_table(h, g, all, reach, dh.reach_words);
    }
    dh.reach = &reach;
  } else if (dd->kind == GMACO_DIST_GRID) {
    const int32_t R = dd->grid_rows, Cc = dd->grid_cols;
    if (R < 2 || Cc < 2 || (int64_t)R * Cc != n)
      throw ValidationError("grid distance: shape does not match the network");
    if ((int64_t)m != 2LL * (R * (Cc - 1) + Cc * (R - 1)))
      throw ValidationError("grid distance: network is not a full 4-neighbour lattice");
    for (int32_t e = 0; e < m; ++e) {
      const int32_t a = g.from[e], b = g.to[e];
      const int32_t ra = a / Cc, ca = a % Cc, rb = b / Cc, cb = b % Cc;
      if (std::abs(ra - rb) + std::abs(ca - cb) != 1 || g.len[e] != g.len[0])
        throw ValidationError("grid distance: network is not a uniform 4-neighbour lattice");
    }
    w.d.rows = R;
    w.d.cols = Cc;
    w.cols_magic = (uint64_t)((((unsigned __int128)1 << 64) + (unsigned)Cc - 1) / (unsigned)Cc);
    w.d.grid_len = g.len[0];
    dh.cols = Cc;
    dh.grid_len = g.len[0];
  } else if (dd->kind == GMACO_DIST_TARGETS) {
    if (dd->target_count < 1 || !dd->targets) throw ValidationError("targets distance: empty target set");
    targets.assign(dd->targets, dd->targets + dd->target_count);
    slot_of.assign(n, -1);
    for (int32_t t = 0; t < (int32_t)targets.size(); ++t) {
      const int32_t x = targets[t];
      if (x < 0 || x >= n || slot_of[x] >= 0)
        throw ValidationError(fmt("targets distance: invalid or duplicate target %d", x));
      slot_of[x] = t;
    }
    ensure_device(h);
    w.d.table = device_distance_table(h, g, targets, reach, dh.reach_words);
    dh.reach = &reach;
    dh.slot_of = &slot_of;
  } else {
    throw ValidationError(fmt("unknown distance kind %d", dd->kind));
  }
  pt.mark("distance service (host)");
  // ---- spawn (host, engine.cpp:71-114) -------------------------------------
  Spawned sp = spawn(c, g, dh, targets);
  pt.mark("spawn (host)");
  const int32_t V = c.vehicle_count;
  // all host-side validation is done: from here on the device is required
  ensure_device(h);
  pt.mark("device init");
  if (!table.empty() && !w.d.table) w.d.table = B.upload(table);  // user-supplied dense table
  if (!slot_of.empty()) w.d.slot_of = B.upload(slot_of);


  // ---- graph in slot order: ELL rows of width 4/8 when the out-degree allows
  // (one aligned vector load per row), plain CSR otherwise ------------------
  int32_t maxdeg = 0;
  for (int32_t u = 0; u < n; ++u) maxdeg = std::max(maxdeg, g.out_ptr[u + 1] - g.out_ptr[u]);
  const bool lattice = dd->kind == GMACO_DIST_GRID;  // lattice shape validated above
  const int32_t ell = lattice || maxdeg <= 4 ? 4 : (maxdeg <= 8 ? 8 : 0);
  // general-graph colony walker: CSR rows padded to multiples of 4 slots so
  // a row's slot records are whole 16-B vectors from a 64-B aligned start
  const bool csr_like = alg == GMACO_COLONY && dd->kind != GMACO_DIST_GRID && c.routing.progress_filter &&
                        c.colony.ants <= 256 && maxdeg <= 16;
  const bool align4 = ell == 0 && csr_like;
  std::vector<int64_t> off4;
  // Row placement order: rows are reached only through row descriptors, so
  // their order in slot space is free.  Aligned-CSR rows are placed in BFS
  // order (Cuthill-McKee without the degree sort): a walk's successive rows
  // and the rows of nearby walks share cache lines and DRAM pages, whatever
  // the input's node numbering (GMACO_ROW_ORDER=none keeps id order).
  std::vector<int32_t> place(n);
  for (int32_t u = 0; u < n; ++u) place[u] = u;
  if (align4) {
    if (!(c.options.flags & GMACO_OPT_NATURAL_ROWS)) {
      std::vector<char> seen(n, 0);
      int32_t qh = 0, qt = 0;
      for (int32_t r = 0; r < n; ++r) {
        if (seen[r]) continue;
        seen[r] = 1;
        place[qt++] = r;
        while (qh < qt) {
          const int32_t u = place[qh++];
          for (int32_t k = g.out_ptr[u]; k < g.out_ptr[u + 1]; ++k) {
            const int32_t v = g.to[g.out_edge[k]];
            if (!seen[v]) { seen[v] = 1; place[qt++] = v; }
          }
        }
      }
    }
    off4.assign(n + 1, 0);  // off4[u]: row start of node u
    // (a row without out-edges still takes 4 padding slots: every row start
    // is unique, so a head-row descriptor identifies its node)
    int64_t at = 0;
    for (int32_t i = 0; i < n; ++i) {
      const int32_t u = place[i];
      off4[u] = at;
      at += std::max(4, (g.out_ptr[u + 1] - g.out_ptr[u] + 3) & ~3);
    }
    off4[n] = at;
    if (off4[n] >= (int64_t(1) << 29)) throw ValidationError("graph too large for the aligned slot layout");
  }
  const int32_t M = ell ? n * ell : (align4 ? (int32_t)off4[n] : m);
  h->ell = ell;
  h->M = M;
  h->slot_edge.assign(M, -1);
  std::vector<int2> row(n);
  std::vector<int32_t> deg(n);
  for (int32_t u = 0; u < n; ++u) {
    const int32_t first = ell ? u * ell : (align4 ? (int32_t)off4[u] : g.out_ptr[u]);
    deg[u] = g.out_ptr[u + 1] - g.out_ptr[u];
    row[u] = make_int2(first, ell ? ell : (align4 ? (deg[u] + 3) & ~3 : deg[u]));
    for (int32_t i = 0; i < deg[u]; ++i) {
      const int32_t e = g.out_edge[g.out_ptr[u] + i];
      int32_t slot = first + i;
      if (lattice) {  // direction-slotted rows {up, left, right, down} = ascending neighbour id
        const int32_t Cc = dd->grid_cols, v = g.to[e];
        slot = first + (v == u - Cc ? 0 : v == u - 1 ? 1 : v == u + 1 ? 2 : 3);
      }
      h->slot_edge[slot] = e;
    }
  }
  for (int32_t s = 0; s < M; ++s)
    if (h->slot_edge[s] >= 0) g.edge_slot[h->slot_edge[s]] = s;
  if (dd->kind == GMACO_DIST_GRID && (dd->grid_rows >= 32768 || dd->grid_cols >= 32768))
    throw ValidationError("grid distance: rows and cols must be < 32768");
  std::vector<int32_t> col(M, -1), slot_from(M, -1), bind(M, -1), key(M, -1);
  std::vector<int64_t> slen(M, 0);
  std::vector<double> eta(M, 0.0);
  int64_t last_len = -1;  // eta depends on the length only: lattices have one (one pow call)
  double last_eta = 0.0;
  for (int32_t s = 0; s < M; ++s) {
    const int32_t e = h->slot_edge[s];
    if (e < 0) continue;
    col[s] = g.to[e];
    slot_from[s] = g.from[e];
    slen[s] = g.len[e];
    key[s] = dd->kind == GMACO_DIST_GRID ? ((g.to[e] / dd->grid_cols) << 16) | (g.to[e] % dd->grid_cols) : g.to[e];
    if (g.len[e] != last_len) {
      const double vis = 1.0 / (static_cast<double>(g.len[e]) / 1000.0);  // routing.cpp:92
      last_eta = std::pow(vis, c.routing.aco_beta);
      last_len = g.len[e];
    }
    eta[s] = last_eta;
  }
  // signals (engine.cpp:124-136, make_signal_state signals.cpp:29-46)
  std::vector<int32_t> sig_of_node(n, -1), lanes_s;
  int32_t S = 0;
  for (int32_t i = 0; i < n; ++i)
    if (g.sig[i]) sig_of_node[i] = S++;
  h->S = S;
  h->sig_node.assign(S, 0);
  lanes_s.assign(S, 1);
  for (int32_t i = 0; i < n; ++i) {
    const int32_t s = sig_of_node[i];
    if (s < 0) continue;
    h->sig_node[s] = i;
    int slot = 0;
    for (int32_t k = g.in_ptr[i]; k < g.in_ptr[i + 1]; ++k, ++slot) {
      const int32_t e = g.in_edge[k];
      bind[g.edge_slot[e]] = s * kPhases + slot % kPhases;
      lanes_s[s] = std::max(lanes_s[s], g.lanes[e]);
    }
  }
  w.g.n = n;
  w.g.m = m;
  w.g.ell = ell;
  w.g.M = M;
  w.g.row = B.upload(row);
  w.g.deg = B.upload(deg);
  w.g.key = B.upload(key);
  w.g.col = B.upload(col);
  w.g.len = B.upload(slen);
  w.g.bind = B.upload(bind);
  w.g.slot_edge = B.upload(h->slot_edge);
  w.g.slot_from = B.upload(slot_from);
  w.g.eta_beta = B.upload(eta);
  B.flush_async();  // the graph's arrays travel while the host builds the rest

  pt.mark("graph slots + upload");
  // ---- params ----------------------------------------------------------------
  DevParams& p = w.p;
  p.algorithm = alg;
  p.controller = c.controller;
  p.deviation_mode = c.routing.deviation_mode;
  p.progress_filter = c.routing.progress_filter != 0;
  p.V = V;
  p.S = S;
  p.deviation_threshold = c.routing.deviation_threshold;
  p.alpha = c.routing.aco_alpha;
  p.dt_s = c.dt_s;
  p.dt_us = std::llround(c.dt_s * 1e6);  // engine.cpp:124-125
  p.latency_us = std::llround(c.decision_latency_s * 1e6);
  p.max_steps = c.max_steps;
  p.seed = c.seed;
  p.tau_lo = tau_from_double(c.pheromone.tau_min);
  p.tau_hi = tau_from_double(c.pheromone.tau_max);
  p.inc = tau_from_double(c.pheromone.delta_inc);
  p.dec = tau_from_double(c.pheromone.delta_dec);
  p.one_minus_rho = 1.0 - c.pheromone.rho;
  p.deposit_q = c.pheromone.aco_deposit_q;
  p.siblings_only = c.pheromone.decrement_siblings_only != 0;
  p.th_max = c.signal.th_max;
  p.t_max = c.signal.t_max;
  p.green_duration_s = c.signal.green_duration_s;
  p.saturation_flow = c.signal.saturation_flow;
  for (int i = 0; i < kPhases; ++i) p.order[i] = c.signal.fixed_cycle_order[i];
  const gmaco_colony_params& k = c.colony;
  p.ants = alg == GMACO_COLONY ? k.ants : 1;
  p.hop_limit = alg == GMACO_COLONY ? k.hop_limit : 1;
  p.max_hops = alg == GMACO_COLONY && k.max_hops > 0 ? k.max_hops : std::max(n - 1, 1);
  p.rng = alg == GMACO_COLONY ? k.rng : GMACO_RNG_REFERENCE;
  p.congestion = alg == GMACO_COLONY ? k.congestion : 0;
  p.deposit = alg == GMACO_COLONY ? k.deposit : (alg == GMACO_ACO ? GMACO_DEPOSIT_COMPLETION : GMACO_DEPOSIT_NONE);
  p.cong_evap = alg == GMACO_COLONY ? k.congestion_evaporation : 0;
  p.replan_all = alg == GMACO_COLONY ? k.replan_all : 0;
  p.need_positions = (alg == GMACO_MACO || alg == GMACO_MACO_P) && !p.siblings_only;
  // debugging / A-B switches (defaults are the production configuration)
  // Bulk L2 prefetch of stages C..G's state (prefetch_tail_state) only when
  // that state fits comfortably in L2: a larger world would evict it again,
  // and the prefetching CTA would hold the walk kernel's end for milliseconds.
  {
    const int64_t Q = (int64_t)S * kPhases;
    const int64_t tail_bytes = (int64_t)V * 77 + Q * 32 + (int64_t)S * 40 + (int64_t)M * 48;
    p.prefetch = !(c.options.flags & GMACO_OPT_NO_PREFETCH) && tail_bytes <= (int64_t(48) << 20) ? 1 : 0;
  }
  p.pdl = (c.options.flags & GMACO_OPT_NO_PDL) ? 0 : 1;
  p.no_smem = (c.options.flags & GMACO_OPT_NO_SMEM) ? 1 : 0;
  p.max_degree = maxdeg;
  // general-graph colony walker: progress-filter bitmaps + next-row
  // descriptors replace the per-hop neighbour distance gathers
  p.csr_walker = alg == GMACO_COLONY && dd->kind != GMACO_DIST_GRID && p.progress_filter && ell != 4 &&
                 c.colony.ants <= 256 && maxdeg <= 16;
  if (p.csr_walker) {
    std::vector<int2> nrow(M, make_int2(0, 0));
    for (int32_t s = 0; s < M; ++s)
      if (col[s] >= 0) nrow[s] = make_int2(row[col[s]].x, row[col[s]].y | (deg[col[s]] << 8));
    w.g.nrow = B.upload(nrow);
    const int32_t T = dd->kind == GMACO_DIST_TARGETS ? (int32_t)targets.size() : n;
    const int64_t fbw = (M + 31) / 32 + 1;
    uint32_t* fb = B.alloc_direct<uint32_t>((size_t)T * fbw);  // filled by k_fbits from the device table
    w.d.fbw = fbw;
    B.flush();  // the kernel reads arena arrays (col, slot_from)
    CK(build_fbits(w, T, fb, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    w.d.fbits = fb;

  }
  p.shard_lo = 0;
  p.shard_hi = V;
  p.sharded = 0;
  for (int r = 0; r < 10; ++r) {  // Philox4x32-10 key schedule of the seed
    p.rk[2 * r] = (uint32_t)c.seed + (uint32_t)r * 0x9E3779B9u;
    p.rk[2 * r + 1] = (uint32_t)(c.seed >> 32) + (uint32_t)r * 0xBB67AE85u;
  }
  // realized-path storage: needed for completion deposits; paths are bounded by
  // the decision count (<= max_steps) and, with the progress filter, by n-1.
  p.path_cap = (int32_t)std::max<int64_t>(
      1, std::min<int64_t>(c.max_steps, p.progress_filter ? (int64_t)n - 1 : c.max_steps));
  const bool need_paths = p.deposit == GMACO_DEPOSIT_COMPLETION && (alg == GMACO_ACO || alg == GMACO_COLONY);
  const size_t path_bytes = (size_t)V * p.path_cap * 4;
  p.record_paths = need_paths || path_bytes <= (size_t(1) << 30);
  if (need_paths && path_bytes > (size_t(16) << 30))
    throw ValidationError("config: realized-path storage exceeds 16 GiB (lower max_steps)");
  if (!p.record_paths) p.path_cap = 1;
  // Tour storage.  With the progress filter every hop strictly decreases the
  // exact distance, so on a uniform grid a walk has at most rows+cols-2 hops;
  // elsewhere the cap is max_hops.
  int32_t walk_bound = p.max_hops;
  if (dd->kind == GMACO_DIST_GRID && p.progress_filter)
    walk_bound = std::min<int32_t>(walk_bound, dd->grid_rows + dd->grid_cols - 2);
  p.plan_cap = alg == GMACO_COLONY ? std::max(walk_bound, 1) : 1;
  if (alg == GMACO_COLONY && (size_t)V * p.plan_cap * 4 > (size_t(32) << 30))
    throw ValidationError("colony: planned-tour storage exceeds 32 GiB (set colony.max_hops)");
  // Tours on the lattice fast path live as move bits (one bit per hop, SMEM);
  // otherwise scratch mode keeps every ant's tour (no winner
  // replay) when it fits 48 GiB of the B200's 180 GB; larger colonies replay
  // the winner instead.
  // (V < 2^24: the walker sums a 64-hop segment's congestion loads, each
  // <= 2V, in 32 bits; its diagonal-major record tables are int32-indexed)
  const bool lattice_walker =
      alg == GMACO_COLONY && dd->kind == GMACO_DIST_GRID && p.progress_filter && p.ants <= 256 && V < (1 << 24) &&
      (int64_t)4 * (dd->grid_rows + dd->grid_cols - 1) * dd->grid_rows < (int64_t)INT32_MAX;
  // move bits: 1 bit per hop in 64-hop SMEM words per ant, when a CTA's
  // words fit 48 KB (lattice CTAs hold <= 256 ants)
  p.bit_words = (p.plan_cap + 63) / 64;
  p.grid_bits = lattice_walker && (size_t)256 * p.bit_words * 8 <= (size_t(48) << 10) && !(c.options.flags & GMACO_OPT_NO_BITS);
  p.scratch_mode = alg == GMACO_COLONY && !p.grid_bits && !(c.options.flags & GMACO_OPT_NO_SCRATCH) &&
                   (size_t)V * p.ants * p.plan_cap * 4 <= (size_t(48) << 30);
  if (alg == GMACO_COLONY) {  // packed (cost, ant) argmin key bound
    int64_t maxlen = 0;
    for (int64_t L : g.len) maxlen = std::max(maxlen, L);
    const long double bound = (long double)p.max_hops * maxlen * (1.0L + V);
    if (bound >= (long double)kCostCap)
      throw ValidationError("colony: tour cost bound exceeds 2^53 (lower max_hops)");
  }

  // ---- pheromone init (init_random, pheromone.cpp:21-32) + first weights ----
  std::vector<int64_t> tau(M, 0);
  std::vector<double> wt(M, 0.0);
  std::vector<int64_t> ecost(M, 0);
  const int64_t lo = p.tau_lo, hi = p.tau_hi;
  const DrawStream init(c.seed, 1);
  for (int32_t s = 0; s < M; ++s) {
    const int32_t e = h->slot_edge[s];
    if (e < 0) continue;
    const double v = uniform(init((uint64_t)e), c.pheromone.tau_init_lo, c.pheromone.tau_init_hi);
    tau[s] = std::clamp(tau_from_double(v), lo, hi);
    const double tau_d = static_cast<double>(tau[s]) / 1e6;
    const double ta = p.alpha == 1.0 ? tau_d : (p.alpha == 0.0 ? 1.0 : std::pow(tau_d, p.alpha));
    wt[s] = ta * eta[s];  // load 0: the congestion factor is exactly 1.0
    ecost[s] = slen[s];
  }
  if (p.alpha != 0.0 && p.alpha != 1.0) w.taupow = build_taupow(B, p.tau_lo, p.tau_hi, p.alpha, h->stream);
  w.tau = B.upload(tau);
  w.weight = B.upload(wt);
  w.ecost = B.upload(ecost);
  {  // int32 tour costs for the lattice walker's SMEM staging: load <= V, so
     // every cost len * (1 + load) <= max len * (1 + V) must stay below 2^31
    int64_t maxlen = 0;
    for (int64_t L : g.len) maxlen = std::max(maxlen, L);
    if (lattice_walker && (long double)maxlen * (1.0L + V) < 2147483648.0L) {
      std::vector<int32_t> e32(M);
      for (int32_t s = 0; s < M; ++s) e32[s] = (int32_t)ecost[s];
      w.ecost32 = B.upload(e32);
    }
  }
  // lattice walker records (LatRec), written by k_lattice_rec after the seal
  // and by stage F+G every step
  if (lattice_walker) {
    // staged in SMEM (node-major) when it fits, else diagonal-major tables
    const bool staged = !p.no_smem && (size_t)16 * M <= (size_t(96) << 10);
    const int32_t R = dd->grid_rows, Cc = dd->grid_cols;
    w.lrec_stride = staged ? 0 : (R + Cc - 1) * R;
    w.lrec = B.alloc_direct<LatRec>(staged ? (size_t)M : (size_t)4 * w.lrec_stride);
  }
  w.occ_cur = B.filled<int32_t>(M, 0);
  w.occ_new = B.filled<int32_t>(M, 0);
  w.dep = B.filled<int64_t>(M, 0);
  w.dec_head = B.filled<int32_t>(std::max(M, n), -1);
  {  // lattice tours have length hops * edge length: tabulate deposit_amount (pheromone.cpp:73-78)
    std::vector<int64_t> amt((size_t)p.plan_cap + 1, 0);
    if (dd->kind == GMACO_DIST_GRID)
      for (int32_t hh = 1; hh <= p.plan_cap; ++hh) {
        const double km = static_cast<double>((int64_t)hh * g.len[0]) / 1e6;
        amt[hh] = tau_from_double(c.pheromone.aco_deposit_q / km);
      }
    w.dep_amount = B.upload(amt);
  }

  // ---- signals -----------------------------------------------------------
  DevSignals& ds = w.s;
  std::vector<int32_t> cur(S, c.signal.fixed_cycle_order[kPhases - 1]);
  ds.node = B.upload(h->sig_node);
  ds.green = B.upload(cur);
  ds.cursor = B.upload(cur);
  ds.lanes = B.upload(lanes_s);
  ds.el_steps = B.filled<int64_t>(S, 0);
  ds.el_s = B.filled<double>(S, c.signal.green_duration_s);
  ds.qlen = B.filled<int32_t>((size_t)S * kPhases, 0);
  ds.qhead = B.filled<int32_t>((size_t)S * kPhases, -1);
  ds.qtail = B.filled<int32_t>((size_t)S * kPhases, -1);
  ds.arr_head = B.filled<int32_t>((size_t)S * kPhases, -1);
  ds.head_wait = B.filled<double>((size_t)S * kPhases, 0.0);
  ds.rem = B.filled<double>((size_t)S * kPhases, 0.0);
  B.flush_async();

  pt.mark("params, tables, pheromone, signals");
  // ---- vehicles ------------------------------------------------------------
  DevVehicles& dv = w.v;
  dv.origin = B.upload(sp.origin);
  dv.dest = B.upload(sp.dest);
  dv.advance = B.upload(sp.advance);
  dv.depart = B.upload(sp.depart);
  dv.state = B.filled<uint8_t>(V, kPending);
  dv.at_node = B.filled<int32_t>(V, -1);
  dv.on_edge = B.filled<int32_t>(V, -1);
  dv.progress = B.filled<int64_t>(V, 0);
  dv.overshoot = B.filled<int64_t>(V, 0);
  dv.queued_phase = B.filled<int32_t>(V, -1);
  dv.joined = B.filled<int64_t>(V, 0);
  dv.arrive = B.filled<int64_t>(V, -1);
  dv.latency_debt = B.filled<int64_t>(V, 0);
  dv.driving = B.filled<int64_t>(V, 0);
  dv.queued = B.filled<int64_t>(V, 0);
  dv.lat_steps = B.filled<int64_t>(V, 0);
  dv.path_len_mm = B.filled<int64_t>(V, 0);
  dv.decisions = B.filled<int32_t>(V, 0);
  dv.deviations = B.filled<int32_t>(V, 0);
  dv.qnext = B.filled<int32_t>(V, -1);
  dv.arr_next = B.filled<int32_t>(V, -1);
  dv.dec_next = B.filled<int32_t>(V, -1);
  dv.dflag = B.filled<int32_t>(V, 0);
  dv.pos = B.filled<int32_t>(V, 0);
  dv.path = B.alloc<int32_t>((size_t)V * p.path_cap);
  dv.path_n = B.filled<int32_t>(V, 0);
  dv.plan = B.alloc<int32_t>(p.scratch_mode ? 1 : (size_t)V * p.plan_cap);
  dv.scratch = B.alloc<int32_t>(p.scratch_mode ? (size_t)V * p.ants * p.plan_cap : 1);
  dv.plan_ant = B.filled<int32_t>(V, 0);
  if (lattice_walker && !(c.options.flags & GMACO_OPT_NO_ORDER)) {
    // Walk-length balance: vehicles sorted by origin->destination Manhattan
    // distance, dealt round-robin over the CTAs so every CTA (and SM) holds a
    // mix of long and short colonies; results do not depend on the order.
    const int32_t Cc = dd->grid_cols;
    // stable counting sort by decreasing Manhattan distance (O(V + rows + cols))
    std::vector<int32_t> dist(V), ord(V);
    int32_t dmax = 0;
    for (int32_t i = 0; i < V; ++i) {
      const int32_t o = sp.origin[i], t = sp.dest[i];
      dist[i] = std::abs(o / Cc - t / Cc) + std::abs(o % Cc - t % Cc);
      dmax = std::max(dmax, dist[i]);
    }
    std::vector<int32_t> at(dmax + 2, 0);
    for (int32_t i = 0; i < V; ++i) at[dmax - dist[i] + 1]++;
    for (int32_t k = 0; k <= dmax; ++k) at[k + 1] += at[k];
    for (int32_t i = 0; i < V; ++i) ord[at[dmax - dist[i]]++] = i;
    // vehicles per CTA of the launch (launch_step): staged tables pack 256/K;
    // otherwise one vehicle per CTA when K fills whole warps (then the order
    // is longest-first: CTAs start in index order, LPT packing of the waves)
    const int32_t K = std::max(1, c.colony.ants);
    const int32_t vpb = grid_smem_bytes(w) ? std::max(1, 256 / K) : ((K % 32 == 0) ? 1 : std::max(1, 256 / K));
    const int32_t ctas = (V + vpb - 1) / vpb;
    // rank r (0 = longest) -> CTA r % ctas, lane r / ctas
    std::vector<int32_t> order(V, -1);
    for (int32_t r = 0; r < V; ++r) {
      const int32_t s = (r % ctas) * vpb + r / ctas;
      order[s < V ? s : r] = ord[r];
    }
    bool ok = true;  // a permutation of 0..V-1 (falls back to identity otherwise)
    std::vector<char> seen(V, 0);
    for (int32_t s = 0; s < V; ++s) {
      if (order[s] < 0 || seen[order[s]]) ok = false;
      else seen[order[s]] = 1;
    }
    if (ok) dv.walk_order = B.upload(order);
  }
  p.ant_queue = p.csr_walker && p.scratch_mode && !(c.options.flags & GMACO_OPT_NO_QUEUE) && (ell == 8 || align4);
  if (p.ant_queue) {
    // slot records {weight (double), int32 edge cost, head row (first/4) << 5 | degree};
    // weight and cost are (re)written by sync_rec_weights and stage F+G
    std::vector<int4> rec(M, make_int4(0, 0, -1, 0));
    for (int32_t s = 0; s < M; ++s) {
      if (col[s] < 0) continue;
      const int32_t hd = col[s];
      rec[s] = make_int4(0, 0, 0, (int32_t)((((uint32_t)row[hd].x >> 2) << 5) | (uint32_t)deg[hd]));
    }
    w.rec = B.upload(rec);
    B.flush();  // the kernel below reads arena arrays
    CK(sync_rec_weights(w, h->stream));
    CK(cudaStreamSynchronize(h->stream));  // before any later flush rewrites the chunk
    dv.walk_start = B.filled<int32_t>(V, -1);
    dv.walk_dec = B.filled<uint8_t>(V, 0);
    dv.best_key = B.filled<unsigned long long>(V, ~0ull);
    dv.walkers = B.filled<int32_t>(V, 0);
    dv.ant_hops = B.filled<int32_t>((size_t)V * p.ants, 0);
    if (dd->kind == GMACO_DIST_TARGETS && maxdeg <= 15 && !(c.options.flags & GMACO_OPT_NO_TT))
      build_target_rows(h, place, (int32_t)targets.size());
    if (!(c.options.flags & GMACO_OPT_NO_ORDER)) {
      // Walk order for the queue: destination-major (the vehicles walking at
      // any moment share a few targets' rows, and their paths converge on
      // them, so those rows stay in L2), then by the origin's row position.
      // Results do not depend on the order.
      std::vector<int32_t> posn(n), ord(V);
      for (int32_t i = 0; i < n; ++i) posn[place[i]] = i;
      for (int32_t i = 0; i < V; ++i) ord[i] = i;
      auto tkey = [&](int32_t x) { return slot_of.empty() ? x : slot_of[x]; };
      // Longest walks first, in kLptBands bands of origin->destination
      // distance (a walk's hop count follows it): the queue's last ants are
      // short walks instead of stragglers holding the kernel's end.  Within a
      // band, destination-major order keeps the rows of a few targets hot.
      constexpr int kLptBands = 8;
      std::vector<int32_t> band(V, 0);
      if (w.d.table) {
        std::vector<int32_t> rowv(V), orgv(V);
        for (int32_t i = 0; i < V; ++i) {
          rowv[i] = tkey(sp.dest[i]);
          orgv[i] = sp.origin[i];
        }
        DevBuffers tmpb;
        tmpb.stream = h->stream;
        int32_t* drow = tmpb.upload(rowv);
        int32_t* dorg = tmpb.upload(orgv);
        int64_t* dd_ = tmpb.alloc<int64_t>(V);
        CK(gather_dist(w.d.table, n, drow, dorg, V, dd_, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        std::vector<int64_t> dv_ = download(dd_, V), sorted_ = dv_;
        std::sort(sorted_.begin(), sorted_.end());
        int64_t cut[kLptBands - 1];
        for (int b = 1; b < kLptBands; ++b) cut[b - 1] = sorted_[(size_t)V * (kLptBands - b) / kLptBands];
        for (int32_t i = 0; i < V; ++i) {
          int b = 0;
          while (b < kLptBands - 1 && dv_[i] < cut[b]) ++b;
          band[i] = b;  // 0: the longest eighth
        }
      }
      std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
        if (band[a] != band[b]) return band[a] < band[b];
        const int32_t ta = tkey(sp.dest[a]), tb = tkey(sp.dest[b]);
        return ta != tb ? ta < tb : posn[sp.origin[a]] < posn[sp.origin[b]];
      });
      dv.walk_order = B.upload(ord);
    }
  }
  dv.dec_rec = B.filled<int32_t>(V, -1);
  if (w.tt.rec) h->target_of_node = slot_of;  // by-target sharding (shard_by_target)
  dv.plan_n = B.filled<int32_t>(V, 0);
  dv.plan_step = B.filled<int64_t>(V, -1);
  dv.plan_done = B.filled<uint8_t>(V, 0);

  pt.mark("vehicles");
  // ---- control block -----------------------------------------------------------
  DevCtl c0{};
  c0.step = 0;
  c0.stop_at = 0;
  int64_t n0 = 0;
  for (int32_t vid = 0; vid < V; ++vid) n0 += sp.depart[vid] == 0;  // count_active at step 0
  c0.n_t = n0;
  c0.done = c.max_steps <= 0 ? 1 : 0;
  h->ctl = B.upload_one(c0);
  w.ctl = h->ctl;
  {  // one pinned block: control-block mirror + stop marker
    void* pin = PinnedPool::take(sizeof(DevCtl) + 64);
    h->ctl_host = static_cast<DevCtl*>(pin);
    h->stop_host = reinterpret_cast<int64_t*>(static_cast<char*>(pin) + sizeof(DevCtl));
  }
  *h->ctl_host = c0;
  pt.mark("ctl upload + pinned mirror");
  if (p.need_positions) {
    h->res.scan_temp_bytes = scan_temp_bytes(V);
    h->res.scan_temp = B.alloc<char>(h->res.scan_temp_bytes);
  }
  h->res.coop_blocks = coop_tail_blocks(w, h->device);
  if (p.need_positions) dv.bsum = B.alloc<int32_t>(std::max(h->res.coop_blocks, 1));
  // stages C, D, E1 beside the lattice walk (DevParams::e1_in_walk): needs the
  // cooperative colony tail, which then runs E3 and the kReleased fix-up
  p.e1_in_walk = lattice_walker && S > 0 && h->res.coop_blocks > 0 && !p.need_positions &&
                 !(c.options.flags & GMACO_OPT_NO_E1_WALK);
  if (p.e1_in_walk) {
    dv.rel = B.alloc<int32_t>(V);
    ds.qlen_e1 = B.filled<int32_t>((size_t)S * kPhases, 0);
    ds.arr_cnt = B.filled<int32_t>((size_t)2 * S * kPhases, 0);
  }
  h->res.queue_blocks = queue_blocks(w, h->device);
  CK(configure_grid_carveout(w));
  if (w.p.ant_queue && h->res.queue_blocks <= 0) throw std::runtime_error("ant-queue walker: no occupancy");
  pt.mark("occupancy queries");
  B.seal();
  CK(launch_lattice_rec(w, h->stream));
  pt.mark("arena seal (copies)");
  CK(cudaEventCreate(&h->ev_a));
  CK(cudaEventCreate(&h->ev_b));
  CK(cudaDeviceSynchronize());
  pt.mark("control block, occupancy, sync");
}

// part 1 = stage-B walk kernel only, part 2 = the rest of the step (C..G)
cudaGraphExec_t capture_part(gmaco_engine* h, int part) {
  StepResources r = h->res;
  r.capturing = true;
  r.part = part;
  cudaGraph_t graph = nullptr;
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t err = launch_step(h->w, r, h->stream, nullptr, nullptr);
  cudaError_t e2 = cudaStreamEndCapture(h->stream, &graph);
  CK(err);
  CK(e2);
  cudaGraphExec_t exec = nullptr;
  CK(cudaGraphInstantiate(&exec, graph, 0));
  cudaGraphDestroy(graph);
  return exec;
}

cudaGraphExec_t capture(gmaco_engine* h, int steps, bool timing) {
  StepResources r = h->res;
  r.capturing = true;
  cudaGraph_t graph = nullptr;
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t err = cudaSuccess;
  for (int i = 0; i < steps && err == cudaSuccess; ++i)
    err = launch_step(h->w, r, h->stream, timing ? h->ev_begin[i] : nullptr, timing ? h->ev_end[i] : nullptr);
  cudaError_t e2 = cudaStreamEndCapture(h->stream, &graph);
  CK(err);
  CK(e2);
  cudaGraphExec_t exec = nullptr;
  CK(cudaGraphInstantiate(&exec, graph, 0));
  cudaGraphDestroy(graph);
  return exec;
}

void refresh_ctl(gmaco_engine* h) {
  CK(cudaMemcpyAsync(h->ctl_host, h->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->ctl_valid = true;
  if (h->ctl_host->error) throw std::runtime_error("device path buffer overflow");
}

// Step graphs never overshoot a target (32-step graphs launch only while at
// least 32 steps remain), so the device-side stop marker stays unbounded and
// is written once instead of once per call.
void unbound_stop(gmaco_engine* h) {
  if (h->stop_written == INT64_MAX) return;
  *h->stop_host = INT64_MAX;
  CK(cudaMemcpyAsync(&h->ctl->stop_at, h->stop_host, sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
  h->stop_written = INT64_MAX;
}

// need_count = false: the steps stay enqueued (no final host sync); the
// control-block mirror is refreshed by the next synchronizing call (e.g. the
// batched gmaco_get_vehicles), so a step/read loop costs one round trip.
// Short runs launch their first kDirectSteps steps straight onto the stream:
// capturing and instantiating a step graph costs ~70-150 us of host time,
// more than a few dozen direct launches (the GPU runs ~25 us steps while the
// host enqueues the next).  Longer runs then switch to the captured graphs.
constexpr int64_t kDirectSteps = 48;
// Snapshots up to this many bytes are gathered by the step's finalizing tail
// block instead of a separate k_pack launch (one block writes them to mapped
// pinned memory; larger snapshots keep the grid-wide gather kernel).
constexpr size_t kTailSnapMax = size_t(64) << 10;
bool launch_direct(gmaco_engine* h) {
  if (h->direct_steps >= kDirectSteps) return false;
  ++h->direct_steps;
  CK(launch_step(h->w, h->res, h->stream, nullptr, nullptr));
  return true;
}

int64_t run_steps(gmaco_engine* h, int64_t steps, bool need_count = true) {
  // reference algorithms: several steps as ONE persistent cooperative launch
  // (k_run_coop: grid barriers between the stages and steps instead of a
  // launch per step); it stops by itself at finished()
  if (steps >= 2 && !h->timing && run_coop_ok(h->w, h->res)) {
    int64_t start = 0;
    if (need_count) {
      if (!h->ctl_valid) refresh_ctl(h);
      start = h->ctl_host->step;
      if (h->ctl_host->done) return 0;
    }
    unbound_stop(h);
    CK(launch_run_coop(h->w, h->res, steps, h->stream));
    h->ctl_valid = false;
    if (!need_count) {
      h->pending = true;
      return -1;
    }
    refresh_ctl(h);
    return h->ctl_host->step - start;
  }
  if (!need_count && !h->timing) {  // enqueue only: no mirror needed (steps past finished() are no-ops)
    if (steps <= 0) return -1;
    unbound_stop(h);
    if (!h->graph_one && !h->graph_big)
      while (steps > 0 && launch_direct(h)) --steps;
    for (int64_t i = 0; i < steps / kGraphSteps; ++i) {
      if (!h->graph_big) h->graph_big = capture(h, kGraphSteps, false);
      CK(cudaGraphLaunch(h->graph_big, h->stream));
    }
    for (int64_t i = 0; i < steps % kGraphSteps; ++i) {
      if (!h->graph_one) h->graph_one = capture(h, 1, false);
      CK(cudaGraphLaunch(h->graph_one, h->stream));
    }
    h->ctl_valid = false;
    h->pending = true;
    return -1;
  }
  if (!h->ctl_valid) refresh_ctl(h);  // else the mirror from the last synchronizing call is current
  const int64_t start = h->ctl_host->step;
  if (steps <= 0 || h->ctl_host->done) return 0;
  const int64_t target = start + steps;
  if (h->timing && h->ev_begin.empty()) {
    h->ev_begin.resize(kGraphSteps);
    h->ev_end.resize(kGraphSteps);
    for (int i = 0; i < kGraphSteps; ++i) {
      CK(cudaEventCreate(&h->ev_begin[i]));
      CK(cudaEventCreate(&h->ev_end[i]));
    }
  }
  unbound_stop(h);
  h->ctl_valid = false;
  h->last_walk_ms = 0.0;
  h->last_walk_launches = 0;
  if (h->timing) CK(cudaEventRecord(h->ev_a, h->stream));  // event nodes serialize the GPU: opt-in
  int64_t cur = start;
  while (cur < target && !h->ctl_host->done) {
    const int64_t remaining = target - cur;
    const bool big = remaining >= kGraphSteps;
    cudaGraphExec_t& ge = h->timing ? (big ? h->tgraph_big : h->tgraph_one) : (big ? h->graph_big : h->graph_one);
    if (!ge && !h->timing && !big && launch_direct(h)) {  // (direct: past finished() a step is a no-op)
      cur += 1;
      continue;
    }
    if (!ge) ge = capture(h, big ? kGraphSteps : 1, h->timing);
    CK(cudaGraphLaunch(ge, h->stream));
    if (h->timing) {
      refresh_ctl(h);
      const int64_t ran = h->ctl_host->step - cur;
      for (int64_t i = 0; i < ran; ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev_begin[i], h->ev_end[i]));
        h->last_walk_ms += ms;
      }
      h->last_walk_launches += ran;
      cur = h->ctl_host->step;
    } else if (big) {
      cur += kGraphSteps;
      if (cur < target) {  // peek for early completion every few chunks
        refresh_ctl(h);
        cur = h->ctl_host->step;
      }
    } else {
      cur += 1;
    }
  }
  if (h->timing) CK(cudaEventRecord(h->ev_b, h->stream));
  refresh_ctl(h);
  float ms = 0.f;
  if (h->timing) CK(cudaEventElapsedTime(&ms, h->ev_a, h->ev_b));
  h->last_step_ms = ms;
  return h->ctl_host->step - start;
}

void read_vehicles(gmaco_engine* h, const gmaco_vehicle_view* v);

void collect(gmaco_engine* h, gmaco_run_result* r, double* travel, int32_t* rvid, int32_t* rnode, int32_t cap) {
  const DevWorld& w = h->w;
  const int32_t V = w.p.V;
  // one gather + one sync for the six fields and the control block
  std::vector<uint8_t> state(V);
  std::vector<int64_t> arrive(V), depart(V), queued(V);
  std::vector<int32_t> decisions(V), at_node(V);
  gmaco_vehicle_view view{};
  view.state = state.data();
  view.arrive_step = arrive.data();
  view.depart_step = depart.data();
  view.queued_steps = queued.data();
  view.decisions = decisions.data();
  view.at_node = at_node.data();
  read_vehicles(h, &view);
  const DevCtl& c = *h->ctl_host;
  gmaco_run_result out{};
  out.steps_executed = c.step;
  double ts = 0.0, ws = 0.0;
  int32_t k = 0;
  const double dt = h->cfg.dt_s, lat = h->cfg.decision_latency_s;
  for (int32_t i = 0; i < V; ++i) {  // engine.cpp:407-422, vid order
    if (travel) travel[i] = -1.0;
    if (state[i] == kArrived) {
      const double t = static_cast<double>(arrive[i] - depart[i]) * dt;
      if (travel) travel[i] = t;
      ts += t;
      ws += static_cast<double>(queued[i]) * dt + static_cast<double>(decisions[i]) * lat;
      ++out.completed_count;
    } else if (state[i] == kRetired) {
      ++out.retired_count;
      if (k < cap) {
        if (rvid) rvid[k] = i;
        if (rnode) rnode[k] = at_node[i];
      }
      ++k;
    }
  }
  if (out.completed_count > 0) {
    out.mean_travel_s = ts / out.completed_count;
    out.mean_wait_s = ws / out.completed_count;
  }
  if (c.qsamples > 0) out.mean_queue_len = static_cast<double>(c.qtotal) / static_cast<double>(c.qsamples);
  out.max_edge_occupancy = c.max_occ;
  out.wall_clock_ms = h->wall_ms;
  *r = out;
}

template <class T>
void scatter_slots(const gmaco_engine* h, const std::vector<T>& by_slot, T* by_edge) {
  for (int32_t s = 0; s < h->M; ++s)
    if (h->slot_edge[s] >= 0) by_edge[h->slot_edge[s]] = by_slot[s];
}

// ---- NCCL (dlopen'ed: the library has no hard NCCL dependency) -------------
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (!api.lib) {
    void* l = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!l) l = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!l) throw std::runtime_error("NCCL runtime (libnccl.so.2) not found");
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(l, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(l, "ncclCommInitRank"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(l, "ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(l, "ncclAllReduce"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(l, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(l, "ncclGroupEnd"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(l, "ncclCommDestroy"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(l, "ncclGetErrorString"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.AllReduce || !api.CommDestroy ||
        !api.GroupStart || !api.GroupEnd)
      throw std::runtime_error("NCCL runtime lacks required symbols");
    api.lib = l;
  }
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string("NCCL error in ") + what + ": " +
                             (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

// Exchange of one step (enqueued between stage B and the rest, captured in
// the step graph): every rank's decision records -> all ranks (allgather of
// the padded shards), best-tour deposits summed (exact int64 allreduce).
cudaError_t nccl_exchange(void* ctx, cudaStream_t st) {
  auto* h = static_cast<gmaco_engine*>(ctx);
  const DevWorld& w = h->w;
  const size_t P = h->shard_pad;
  // both collectives in one NCCL group: a single fused launch per step
  const NcclApi& N = nccl();
  if (w.v.owner) {  // by-target shards: this rank's records in its walk order
    const cudaError_t e = rec_pack(w, h->xsend, (int32_t)P, st);
    if (e != cudaSuccess) return e;
  }
  if (N.GroupStart() != ncclSuccess) return cudaErrorUnknown;
  ncclResult_t r = w.v.owner ? N.AllGather(h->xsend, h->xrecv, P, ncclInt32, h->comm, st)
                             : N.AllGather(w.v.dec_rec + (size_t)h->rank * P, w.v.dec_rec, P, ncclInt32, h->comm, st);
  if (r == ncclSuccess && w.p.deposit == GMACO_DEPOSIT_BEST_TOUR)
    r = N.AllReduce(w.dep, w.dep, (size_t)w.g.M, ncclInt64, ncclSum, h->comm, st);
  const ncclResult_t e = N.GroupEnd();
  if (r != ncclSuccess || e != ncclSuccess) return cudaErrorUnknown;
  return w.v.owner ? rec_unpack(w, h->xrecv, h->xgath, (int32_t)(P * h->world), st) : cudaSuccess;
}

// By-target sharding (worlds with per-target candidate rows): rank r plans
// the vehicles bound for the targets dealt to it -- largest vehicle count
// first, each to the least-loaded rank (ties: lowest index), identically on
// every rank -- so it refreshes and walks only its own targets' tables
// (k_tt_refresh over T/world tables instead of T) and its walk stays
// destination-major.  The planning list is the full walk order filtered to
// the rank's vehicles.  Returns every rank's list (the allgather layout).
std::vector<std::vector<int32_t>> shard_by_target(gmaco_engine* h, int32_t rank, int32_t world) {
  DevWorld& w = h->w;
  if (w.p.sharded) throw ValidationError("sharding: the engine is already sharded");
  if (!w.tt.rec || h->target_of_node.empty())
    throw ValidationError("sharding: by-target shards need per-target rows (TARGETS distances, ant-queue walker)");
  if (rank < 0 || rank >= world || world > 32767) throw ValidationError("sharding: invalid rank / world");
  const int32_t V = w.p.V, T = w.tt.T;
  const std::vector<int32_t> dest = download(w.v.dest, V);
  std::vector<int32_t> order(V);
  if (w.v.walk_order) order = download(w.v.walk_order, V);
  else for (int32_t i = 0; i < V; ++i) order[i] = i;
  std::vector<int64_t> cnt(T, 0);
  for (int32_t i = 0; i < V; ++i) cnt[h->target_of_node[dest[i]]]++;
  std::vector<int32_t> ts(T);
  for (int32_t t = 0; t < T; ++t) ts[t] = t;
  std::stable_sort(ts.begin(), ts.end(), [&](int32_t a, int32_t b) { return cnt[a] > cnt[b]; });
  std::vector<int64_t> load(world, 0);
  std::vector<int16_t> towner(T, 0);
  for (int32_t t : ts) {
    int32_t best = 0;
    for (int32_t r = 1; r < world; ++r)
      if (load[r] < load[best]) best = r;
    towner[t] = (int16_t)best;
    load[best] += cnt[t];
  }
  std::vector<int16_t> owner(V);
  std::vector<std::vector<int32_t>> lists(world);
  for (int32_t i = 0; i < V; ++i) owner[i] = towner[h->target_of_node[dest[i]]];
  for (int32_t i = 0; i < V; ++i) lists[owner[order[i]]].push_back(order[i]);
  std::vector<int32_t> own_t;
  for (int32_t t = 0; t < T; ++t)
    if (towner[t] == rank) own_t.push_back(t);
  auto up = [&](const auto& vec) {
    using E = typename std::decay_t<decltype(vec)>::value_type;
    E* d = h->buf.alloc_direct<E>(std::max<size_t>(vec.size(), 1));
    if (!vec.empty()) CK(cudaMemcpyAsync(d, vec.data(), vec.size() * sizeof(E), cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return d;
  };
  const std::vector<int32_t>& mine = lists[rank];
  w.v.walk_order = up(mine);  // slots [0, n_own): this rank's vehicles
  w.v.owner = up(owner);
  w.tt.own_t = up(own_t);
  w.tt.T_own = (int32_t)own_t.size();
  w.p.shard_lo = 0;
  w.p.shard_hi = (int32_t)mine.size();
  w.p.rank = rank;
  w.p.sharded = 1;
  h->reset_graphs();
  return lists;
}

// Vehicle sharding (partition_entities ranges, parallel.cpp:8-21): this
// engine decides / plans vehicles [lo, hi); every rank replays stages C..G for
// the whole fleet from the exchanged decision records.  Every algorithm
// shards: colonies, and the reference's dijkstra / aco / maco / maco-p, whose
// network-wide MACO fold takes every decision's global position from the
// records (commit_pheromone, parallel.cpp:195-258).
void set_shard(gmaco_engine* h, int32_t lo, int32_t hi, int32_t pad_total) {
  DevWorld& w = h->w;
  if (lo < 0 || hi > w.p.V || lo > hi) throw ValidationError("sharding: invalid vehicle range");
  if (w.v.owner) throw ValidationError("sharding: the engine is sharded by target");
  if (w.g.M >= GMACO_REC_DEVIATED || h->g.m >= GMACO_REC_DEVIATED)
    throw ValidationError("sharding: decision records need fewer than 2^30 edges");
  if (pad_total > w.p.V) {  // allgather layout: world * shard_pad records
    int32_t* d = h->buf.filled<int32_t>(pad_total, -1);
    w.v.dec_rec = d;
  }
  // the walk order (destination-major / walk-length balanced) restricted to
  // the shard, in the same relative order: slot lo + i holds the shard's i-th
  // vehicle of the full order, so a rank keeps the order's locality
  if (w.v.walk_order) {
    const int32_t V = w.p.V;
    std::vector<int32_t> full = download(w.v.walk_order, V), mine(V, -1);
    int32_t k = lo;
    for (int32_t i = 0; i < V; ++i)
      if (full[i] >= lo && full[i] < hi) mine[k++] = full[i];
    int32_t* d = h->buf.alloc_direct<int32_t>(V);
    CK(cudaMemcpyAsync(d, mine.data(), (size_t)V * 4, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    w.v.walk_order = d;
  }
  w.p.shard_lo = lo;
  w.p.shard_hi = hi;
  w.p.sharded = 1;
  h->reset_graphs();
}

}  // namespace

// Process-wide communicators, one per (device, rank, world, unique id): an
// engine attaching with an id already used in this process reuses that
// communicator instead of paying ncclCommInitRank again (a job creates its
// communicator once; later engines of the same job reuse it).  A communicator
// is held EXCLUSIVELY by one live engine: two live engines capturing
// collectives on one communicator into their own graphs could interleave them
// in different orders on different ranks and hang the job, so a second attach
// while the holder is alive fails (status 1).  The holder releases it on
// destroy; idle communicators stay cached for the next engine of the job.
struct CommEntry {
  ncclComm_t comm = nullptr;
  const gmaco_engine* holder = nullptr;
};
static std::mutex g_comm_mu;
static std::map<std::string, CommEntry>& comm_cache() {
  static auto* m = new std::map<std::string, CommEntry>();  // process lifetime
  return *m;
}

void gmaco_engine::destroy_comm() {
  if (!comm) return;
  std::lock_guard<std::mutex> lk(g_comm_mu);
  for (auto& kv : comm_cache())
    if (kv.second.holder == this) kv.second.holder = nullptr;
  comm = nullptr;
}

// Host -> device copy ordered on the engine stream and complete on return
// (the source may be a temporary; a plain pageable cudaMemcpy can return with
// its DMA in flight and is unordered with the non-blocking engine stream).
static void h2d(gmaco_engine* h, void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
}

namespace {
// The requested vehicle fields (and the control block) in one gather into
// pinned staging memory plus one sync (gmaco_get_vehicles, collect).
void read_vehicles(gmaco_engine* h, const gmaco_vehicle_view* v) {
    const DevVehicles& d = h->w.v;
    const size_t V = h->w.p.V;
    // requested fields: async copies into one pinned staging buffer, one
    // stream sync, then host copies out (one round trip instead of one per field)
    std::vector<std::pair<void*, size_t>> outs;  // (user dst, staging offset)
    std::vector<std::pair<const void*, size_t>> srcs;
    size_t total = 0;
    auto plan = [&](void* dst, const void* src, size_t elem) {
      if (!dst) return;
      outs.emplace_back(dst, total);
      srcs.emplace_back(src, V * elem);
      total += (V * elem + 15) & ~size_t(15);
    };
    plan(v->origin, d.origin, 4);
    plan(v->dest, d.dest, 4);
    plan(v->advance_mm, d.advance, 8);
    plan(v->state, d.state, 1);
    plan(v->at_node, d.at_node, 4);
    plan(v->progress_mm, d.progress, 8);
    plan(v->overshoot_mm, d.overshoot, 8);
    plan(v->queued_phase, d.queued_phase, 4);
    plan(v->queue_joined_step, d.joined, 8);
    plan(v->depart_step, d.depart, 8);
    plan(v->arrive_step, d.arrive, 8);
    plan(v->latency_debt_us, d.latency_debt, 8);
    plan(v->driving_steps, d.driving, 8);
    plan(v->queued_steps, d.queued, 8);
    plan(v->latency_steps, d.lat_steps, 8);
    plan(v->decisions, d.decisions, 4);
    plan(v->deviations, d.deviations, 4);
    plan(v->path_length_mm, d.path_len_mm, 8);
    const size_t oe_off = total;
    if (v->on_edge) total += V * 4;
    total += 16;  // never empty: the control block copy + sync always run
    {
      if (h->stage_bytes < total) {
        PinnedPool::give(h->stage);
        h->stage = nullptr;
        h->stage = PinnedPool::take(total);
        h->stage_bytes = total;
      }
      char* st = static_cast<char*>(h->stage);
      char* st_dev = nullptr;
      void* ctl_dev = nullptr;
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&st_dev), h->stage, 0));
      CK(cudaHostGetDevicePointer(&ctl_dev, h->ctl_host, 0));
      // one gather kernel into mapped pinned memory; the control block rides
      // along, so the host mirror is current after the single sync
      PackDesc pd;
      for (size_t i = 0; i < outs.size(); ++i) pd.f[pd.n++] = PackField{srcs[i].first, st_dev + outs[i].second, srcs[i].second};
      if (v->on_edge) pd.f[pd.n++] = PackField{d.on_edge, st_dev + oe_off, V * 4};
      pd.f[pd.n++] = PackField{h->ctl, ctl_dev, sizeof(DevCtl)};
      CK(launch_pack(pd, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      h->pending = false;
      h->ctl_valid = true;
      if (h->ctl_host->error) throw std::runtime_error("device path buffer overflow");
      for (size_t i = 0; i < outs.size(); ++i) std::memcpy(outs[i].first, st + outs[i].second, srcs[i].second);
      if (v->on_edge) {
        const int32_t* oe = reinterpret_cast<const int32_t*>(st + oe_off);
        for (size_t i = 0; i < V; ++i) v->on_edge[i] = oe[i] < 0 ? -1 : h->slot_edge[oe[i]];
      }
    }
    if (v->speed_mps) {  // speed is host-side setup state: recompute as spawn did
      const DrawStream sp(h->cfg.seed, 3);
      for (size_t i = 0; i < V; ++i)
        v->speed_mps[i] = uniform(sp(i), h->cfg.speed_min_mps, h->cfg.speed_max_mps);
    }
  }
}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int32_t gmaco_abi_version(void) { return GMACO_ABI_VERSION; }

int gmaco_nccl_unique_id(void* out128) {
  if (!out128) return GMACO_EVALIDATION;
  return guarded(nullptr, [&] {
    ncclUniqueId id;
    nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof id);
  });
}

int gmaco_attach_comm(gmaco_engine* h, int32_t rank, int32_t world, const void* nccl_id) {
  NvtxRange nvtx_(__func__);
  if (h) h->ctl_valid = false;
  if (!h || !nccl_id || world < 1 || rank < 0 || rank >= world) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof id);
    h->destroy_comm();
    std::string key(reinterpret_cast<const char*>(&id), sizeof id);
    key += fmt("/%d/%d/%d", h->device, rank, world);
    std::lock_guard<std::mutex> lk(g_comm_mu);
    CommEntry& ce = comm_cache()[key];
    if (ce.holder)
      throw ValidationError("attach_comm: this communicator is held by another live engine "
                            "(destroy it first; one engine per communicator at a time)");
    const int32_t V = h->w.p.V;
    if (h->w.tt.rec) {  // per-target rows: shard by destination target
      const auto lists = shard_by_target(h, rank, world);
      int32_t P = 1;
      for (const auto& l : lists) P = std::max<int32_t>(P, (int32_t)l.size());
      std::vector<int32_t> gath((size_t)world * P, -1);
      for (int32_t r = 0; r < world; ++r)
        std::copy(lists[r].begin(), lists[r].end(), gath.begin() + (size_t)r * P);
      h->xsend = h->buf.alloc_direct<int32_t>(P);
      h->xrecv = h->buf.alloc_direct<int32_t>((size_t)world * P);
      h->xgath = h->buf.alloc_direct<int32_t>((size_t)world * P);
      CK(cudaMemcpyAsync(h->xgath, gath.data(), gath.size() * 4, cudaMemcpyHostToDevice, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      h->shard_pad = P;
    } else {
      const int32_t P = (V + world - 1) / world;  // padded contiguous shards (allgather layout)
      const int32_t lo = std::min(V, rank * P), hi = std::min(V, (rank + 1) * P);
      set_shard(h, lo, hi, world * P);
      h->shard_pad = P;
    }
    h->rank = rank;
    h->world = world;
    if (!ce.comm) nck(nccl().CommInitRank(&ce.comm, world, id, rank), "ncclCommInitRank");
    ce.holder = h;
    h->comm = ce.comm;
    h->res.exchange = nccl_exchange;
    h->res.exchange_ctx = h;
  });
}

int gmaco_set_shard(gmaco_engine* h, int32_t lo, int32_t hi) {
  NvtxRange nvtx_(__func__);
  if (h) h->ctl_valid = false;
  if (!h) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    set_shard(h, lo, hi, 0);
    h->res.exchange = nullptr;
  });
}

int gmaco_shard_by_target(gmaco_engine* h, int32_t rank, int32_t world) {
  NvtxRange nvtx_(__func__);
  if (h) h->ctl_valid = false;
  if (!h) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    shard_by_target(h, rank, world);
    h->res.exchange = nullptr;
  });
}

int gmaco_shard_vehicles(gmaco_engine* h, int32_t* vids, int32_t cap, int32_t* n) {
  if (!h || !n) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    const DevWorld& w = h->w;
    *n = w.p.shard_hi - w.p.shard_lo;
    if (vids && cap >= *n) {
      if (w.v.owner) {
        const auto mine = download(w.v.walk_order, *n);
        std::copy(mine.begin(), mine.end(), vids);
      } else {
        for (int32_t i = 0; i < *n; ++i) vids[i] = w.p.shard_lo + i;
      }
    }
  });
}

int gmaco_step_split(gmaco_engine* h, int32_t part) {
  NvtxRange nvtx_(__func__);
  if (h) h->ctl_valid = false;
  if (!h || (part != 1 && part != 2)) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    if (part == 1) {
      refresh_ctl(h);
      unbound_stop(h);
      if (!h->graph_walk) h->graph_walk = capture_part(h, 1);
      CK(cudaGraphLaunch(h->graph_walk, h->stream));
    } else {
      if (!h->graph_tail) h->graph_tail = capture_part(h, 2);
      CK(cudaGraphLaunch(h->graph_tail, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    refresh_ctl(h);
  });
}

int gmaco_exchange_export(gmaco_engine* h, int32_t* decisions, int64_t* deposits) {
  NvtxRange nvtx_(__func__);
  if (!h) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    const DevWorld& w = h->w;
    const int32_t lo = w.p.shard_lo, hi = w.p.shard_hi;
    if (decisions && hi > lo && w.v.owner) {  // by-target shard: own records in planning order
      const auto rec = download(w.v.dec_rec, w.p.V);
      const auto mine = download(w.v.walk_order, hi);
      for (int32_t i = 0; i < hi; ++i) decisions[i] = rec[mine[i]];
    } else if (decisions && hi > lo) {  // records at the boundary: edge id, -1 none, -2 retired
      CK(cudaMemcpy(decisions, w.v.dec_rec + lo, (size_t)(hi - lo) * 4, cudaMemcpyDeviceToHost));
    }
    if (decisions && hi > lo) {
      for (int32_t i = 0; i < hi - lo; ++i)
        if (decisions[i] >= 0)
          decisions[i] = h->slot_edge[decisions[i] & ~GMACO_REC_DEVIATED] | (decisions[i] & GMACO_REC_DEVIATED);
    }
    if (deposits) scatter_slots(h, download(w.dep, h->M), deposits);
  });
}

int gmaco_exchange_import(gmaco_engine* h, const int32_t* decisions, const int64_t* deposits) {
  NvtxRange nvtx_(__func__);
  if (h) h->ctl_valid = false;
  if (!h) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    const DevWorld& w = h->w;
    if (decisions) {
      std::vector<int32_t> d(decisions, decisions + w.p.V);
      for (auto& x : d)
        if (x >= 0) {
          const int32_t e = x & ~GMACO_REC_DEVIATED;
          if (e >= h->g.m) throw ValidationError("exchange_import: invalid edge id");
          x = h->g.edge_slot[e] | (x & GMACO_REC_DEVIATED);
        }
      h2d(h, w.v.dec_rec, d.data(), d.size() * 4);
    }
    if (deposits) {
      std::vector<int64_t> d(h->M, 0);
      for (int32_t s = 0; s < h->M; ++s)
        if (h->slot_edge[s] >= 0) d[s] = deposits[h->slot_edge[s]];
      h2d(h, w.dep, d.data(), d.size() * 8);
    }
  });
}

int gmaco_create(const gmaco_graph_desc* graph, const gmaco_distance_desc* dist, const gmaco_sim_config* cfg,
                 int32_t device, gmaco_engine** out) {
  NvtxRange nvtx_(__func__);
  if (!out) {
    g_create_err = "gmaco_create: out is null";
    return GMACO_EVALIDATION;
  }
  *out = nullptr;
  auto h = std::make_unique<gmaco_engine>();
  h->device = device;
  int rc = guarded(nullptr, [&] { build_world(h.get(), graph, dist, cfg); });
  if (rc != GMACO_OK) return rc;
  *out = h.release();
  return GMACO_OK;
}

int gmaco_step(gmaco_engine* h, int64_t steps, int64_t* executed) {
  NvtxRange nvtx_(__func__);
  if (!h) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    const int64_t k = run_steps(h, steps, executed != nullptr);
    if (executed) *executed = k;
  }, /*stream_ordered=*/true);
}

int gmaco_finished(gmaco_engine* h, int32_t* out) {
  if (!h || !out) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    refresh_ctl(h);
    *out = h->ctl_host->done;
  });
}

int gmaco_current_step(gmaco_engine* h, int64_t* out) {
  if (!h || !out) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    refresh_ctl(h);
    *out = h->ctl_host->step;
  });
}

int gmaco_run(gmaco_engine* h, gmaco_run_result* result, double* travel_times_s) {
  NvtxRange nvtx_(__func__);
  if (!h || !result) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    const auto t0 = std::chrono::steady_clock::now();
    while (true) {
      refresh_ctl(h);
      if (h->ctl_host->done) break;
      run_steps(h, int64_t(1) << 40);
    }
    h->wall_ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    collect(h, result, travel_times_s, nullptr, nullptr, 0);
  });
}

int gmaco_collect(gmaco_engine* h, gmaco_run_result* result, double* travel_times_s, int32_t* retired_vid,
                  int32_t* retired_node, int32_t retired_cap) {
  NvtxRange nvtx_(__func__);
  if (!h || !result) return GMACO_EVALIDATION;
  return guarded(h, [&] { collect(h, result, travel_times_s, retired_vid, retired_node, retired_cap); });
}

int gmaco_get_pheromone(gmaco_engine* h, int64_t* tau) {
  NvtxRange nvtx_(__func__);
  if (!h || !tau) return GMACO_EVALIDATION;
  return guarded(h, [&] { scatter_slots(h, download(h->w.tau, h->M), tau); });
}

int gmaco_set_pheromone(gmaco_engine* h, const int64_t* tau) {
  NvtxRange nvtx_(__func__);
  if (h) h->ctl_valid = false;
  if (!h || !tau) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    const int32_t m = h->M;
    std::vector<int64_t> t(m, 0);
    std::vector<double> wt(m, 0.0);
    auto eta = download(h->w.g.eta_beta, m);
    // colony congestion: the next walk's weight and tour cost carry the edge
    // load (occupancy + the fed queue's length) exactly as stage F+G computed
    // them (slot_fg): weight x 1/(1+load), cost = len + len*load
    // every update clamps the field to [tau_min, tau_max] (pheromone.cpp:34-67);
    // the device relies on it (tau^alpha table index)
    for (int32_t e = 0; e < h->g.m; ++e)
      if (tau[e] < h->w.p.tau_lo || tau[e] > h->w.p.tau_hi)
        throw ValidationError(fmt("set_pheromone: edge %d value %lld outside [tau_min, tau_max]", e,
                                  (long long)tau[e]));
    const bool cong = h->w.p.algorithm == GMACO_COLONY && h->w.p.congestion;
    std::vector<int32_t> occ, bind, qlen;
    std::vector<int64_t> len, cost;
    if (cong) {
      occ = download(h->w.occ_cur, m);
      bind = download(h->w.g.bind, m);
      qlen = download(h->w.s.qlen, (size_t)h->S * kPhases);
      len = download(h->w.g.len, m);
      cost = download(h->w.ecost, m);
    }
    for (int32_t s = 0; s < m; ++s) {
      if (h->slot_edge[s] < 0) continue;
      t[s] = tau[h->slot_edge[s]];
      const double tau_d = static_cast<double>(t[s]) / 1e6;
      const double a = h->w.p.alpha;
      wt[s] = (a == 1.0 ? tau_d : (a == 0.0 ? 1.0 : std::pow(tau_d, a))) * eta[s];
      if (cong) {
        const int32_t load = occ[s] + (bind[s] >= 0 ? qlen[bind[s]] : 0);
        wt[s] = wt[s] * (1.0 / (1.0 + static_cast<double>(load)));
        cost[s] = len[s] + len[s] * static_cast<int64_t>(load);
      }
    }
    h2d(h, h->w.tau, t.data(), m * 8);
    h2d(h, h->w.weight, wt.data(), m * 8);
    if (cong) {
      h2d(h, h->w.ecost, cost.data(), m * 8);
      if (h->w.ecost32) {
        std::vector<int32_t> c32(m);
        for (int32_t s = 0; s < m; ++s) c32[s] = static_cast<int32_t>(cost[s]);
        h2d(h, h->w.ecost32, c32.data(), m * 4);
      }
    }
    if (h->w.rec) {
      CK(sync_rec_weights(h->w, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    }
    if (h->w.lrec) {
      CK(launch_lattice_rec(h->w, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    }
  });
}

int gmaco_get_occupancy(gmaco_engine* h, int32_t* occ) {
  if (!h || !occ) return GMACO_EVALIDATION;
  return guarded(h, [&] { scatter_slots(h, download(h->w.occ_cur, h->M), occ); });
}

int gmaco_get_vehicles(gmaco_engine* h, const gmaco_vehicle_view* v) {
  NvtxRange nvtx_(__func__);
  if (!h || !v) return GMACO_EVALIDATION;
  return guarded(h, [&] { read_vehicles(h, v); }, /*stream_ordered=*/true);
}
// The requested vehicle fields of a view, in declaration order:
// (user destination, device source, element bytes).
static std::vector<std::tuple<void*, const void*, size_t>> vehicle_fields(const gmaco_engine* h,
                                                                          const gmaco_vehicle_view* v) {
  const DevVehicles& d = h->w.v;
  std::vector<std::tuple<void*, const void*, size_t>> f;
  auto add = [&](void* dst, const void* src, size_t e) {
    if (dst) f.emplace_back(dst, src, e);
  };
  add(v->origin, d.origin, 4);
  add(v->dest, d.dest, 4);
  add(v->advance_mm, d.advance, 8);
  add(v->state, d.state, 1);
  add(v->at_node, d.at_node, 4);
  add(v->progress_mm, d.progress, 8);
  add(v->overshoot_mm, d.overshoot, 8);
  add(v->queued_phase, d.queued_phase, 4);
  add(v->queue_joined_step, d.joined, 8);
  add(v->depart_step, d.depart, 8);
  add(v->arrive_step, d.arrive, 8);
  add(v->latency_debt_us, d.latency_debt, 8);
  add(v->driving_steps, d.driving, 8);
  add(v->queued_steps, d.queued, 8);
  add(v->latency_steps, d.lat_steps, 8);
  add(v->decisions, d.decisions, 4);
  add(v->deviations, d.deviations, 4);
  add(v->path_length_mm, d.path_len_mm, 8);
  return f;
}

}  // extern "C"

namespace gmaco {
namespace {
// Bit i set <=> the i-th device-gathered member of the view is non-NULL
// (speed_mps is recomputed on the host and is not part of a snapshot).
uint32_t view_mask(const gmaco_vehicle_view* v) {
  const void* m[] = {v->origin, v->dest, v->advance_mm, v->state, v->at_node, v->on_edge, v->progress_mm,
                     v->overshoot_mm, v->queued_phase, v->queue_joined_step, v->depart_step, v->arrive_step,
                     v->latency_debt_us, v->driving_steps, v->queued_steps, v->latency_steps, v->decisions,
                     v->deviations, v->path_length_mm};
  uint32_t bits = 0;
  for (size_t i = 0; i < sizeof m / sizeof m[0]; ++i)
    if (m[i]) bits |= 1u << i;
  return bits;
}

// Arms readback slot `slot` for `fields` (layout, pinned buffer, done event)
// and returns the gather descriptor of the snapshot.
PackDesc arm_slot(gmaco_engine* h, const gmaco_vehicle_view* fields, int32_t slot) {
  auto& rs = h->rslot[slot];
  rs.mask = view_mask(fields);
  // the layout depends only on the field set: a step / read loop re-arms a
  // slot with the same fields every step (no host work but this compare)
  if (rs.pd_valid && rs.pd_mask == rs.mask) return rs.pd_cache;
  const size_t V = h->w.p.V;
  const auto f = vehicle_fields(h, fields);
  size_t total = 0;
  rs.fields.clear();
  for (const auto& t : f) {
    rs.fields.emplace_back(total, V * std::get<2>(t));
    total += (V * std::get<2>(t) + 15) & ~size_t(15);
  }
  rs.on_edge = fields->on_edge != nullptr;
  rs.oe_off = total;
  if (rs.on_edge) total += V * 4;
  total = std::max<size_t>(total, 16);
  if (rs.bytes < total) {
    PinnedPool::give(rs.buf);
    rs.buf = PinnedPool::take(total);
    rs.bytes = total;
  }
  if (!rs.done) CK(cudaEventCreateWithFlags(&rs.done, cudaEventDisableTiming));
  char* dev = nullptr;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), rs.buf, 0));
  PackDesc pd{};
  for (size_t i = 0; i < f.size(); ++i) pd.f[pd.n++] = PackField{std::get<1>(f[i]), dev + rs.fields[i].first,
                                                                 rs.fields[i].second};
  if (rs.on_edge) pd.f[pd.n++] = PackField{h->w.v.on_edge, dev + rs.oe_off, V * 4};
  rs.pd_cache = pd;
  rs.pd_mask = rs.mask;
  rs.pd_valid = true;
  return pd;
}
}  // namespace
}  // namespace gmaco

extern "C" {

int gmaco_step_snapshot(gmaco_engine* h, const gmaco_vehicle_view* fields, int32_t slot) {
  NvtxRange nvtx_(__func__);
  if (h) h->ctl_valid = false;
  if (!h || !fields || slot < 0 || slot > 1) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    const PackDesc pd = arm_slot(h, fields, slot);
    auto& rs = h->rslot[slot];
    size_t snap_bytes = 0;
    for (int i = 0; i < pd.n; ++i) snap_bytes += pd.f[i].bytes;
    if (h->res.coop_blocks > 0 && snap_bytes <= kTailSnapMax) {
      // small worlds: the step's finalizing tail block gathers the fields
      // (no k_pack launch); its descriptor lives in device memory, rewritten
      // only when the field set changes, so one graph per slot serves any set
      if (!rs.pd_dev) rs.pd_dev = h->buf.alloc_direct<PackDesc>(1);
      if (!rs.pd_dev_set || std::memcmp(&rs.pd_dev_val, &pd, sizeof pd) != 0) {
        // a stream-ordered upload: gathers enqueued before it still read the
        // old descriptor, the steps after it the new one; no host sync, so a
        // step / snapshot loop keeps the GPU fed from its first iteration
        if (!rs.pd_host) {
          rs.pd_host = static_cast<PackDesc*>(PinnedPool::take(sizeof(PackDesc)));
          CK(cudaEventCreateWithFlags(&rs.pd_copied, cudaEventDisableTiming));
        } else {
          CK(cudaEventSynchronize(rs.pd_copied));  // the previous upload has read the staging
        }
        *rs.pd_host = pd;
        CK(cudaMemcpyAsync(rs.pd_dev, rs.pd_host, sizeof pd, cudaMemcpyHostToDevice, h->stream));
        CK(cudaEventRecord(rs.pd_copied, h->stream));
        rs.pd_dev_val = pd;
        rs.pd_dev_set = true;
      }
      DevWorld ws = h->w;
      ws.snap = rs.pd_dev;
      unbound_stop(h);
      if (!rs.tail_snap_graph && h->direct_steps < kDirectSteps) {
        ++h->direct_steps;
        CK(launch_step(ws, h->res, h->stream, nullptr, nullptr));
      } else {
        if (!rs.tail_snap_graph) {
          StepResources r = h->res;
          r.capturing = true;
          cudaGraph_t graph = nullptr;
          CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
          const cudaError_t err = launch_step(ws, r, h->stream, nullptr, nullptr);
          const cudaError_t e2 = cudaStreamEndCapture(h->stream, &graph);
          CK(err);
          CK(e2);
          CK(cudaGraphInstantiate(&rs.tail_snap_graph, graph, 0));
          cudaGraphDestroy(graph);
        }
        CK(cudaGraphLaunch(rs.tail_snap_graph, h->stream));
      }
      CK(cudaEventRecord(rs.done, h->stream));
      rs.armed = true;
      h->pending = true;
      return;
    }
    // the first kDirectSteps steps: a direct step launch + the gather kernel
    // (no capture cost for short runs)
    if (!rs.snap_graph && h->direct_steps < kDirectSteps) {
      unbound_stop(h);
      launch_direct(h);
      CK(launch_pack(pd, h->stream));
      CK(cudaEventRecord(rs.done, h->stream));
      rs.armed = true;
      h->pending = true;
      return;
    }
    // then one graph per slot: a step then the snapshot gather, re-captured
    // when the gather descriptor (field set, buffer) changes
    if (!rs.snap_graph || std::memcmp(&rs.snap_pd, &pd, sizeof pd) != 0) {
      if (rs.snap_graph) CK(cudaGraphExecDestroy(rs.snap_graph));
      StepResources r = h->res;
      r.capturing = true;
      cudaGraph_t graph = nullptr;
      CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
      cudaError_t err = launch_step(h->w, r, h->stream, nullptr, nullptr);
      if (err == cudaSuccess) err = launch_pack(pd, h->stream);
      const cudaError_t e2 = cudaStreamEndCapture(h->stream, &graph);
      CK(err);
      CK(e2);
      CK(cudaGraphInstantiate(&rs.snap_graph, graph, 0));
      cudaGraphDestroy(graph);
      rs.snap_pd = pd;
    }
    unbound_stop(h);
    CK(cudaGraphLaunch(rs.snap_graph, h->stream));
    CK(cudaEventRecord(rs.done, h->stream));
    rs.armed = true;
    h->pending = true;
  }, /*stream_ordered=*/true);
}

int gmaco_vehicles_enqueue(gmaco_engine* h, const gmaco_vehicle_view* fields, int32_t slot) {
  NvtxRange nvtx_(__func__);
  if (!h || !fields || slot < 0 || slot > 1) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    auto& rs = h->rslot[slot];
    CK(launch_pack(arm_slot(h, fields, slot), h->stream));
    CK(cudaEventRecord(rs.done, h->stream));
    rs.armed = true;
  }, /*stream_ordered=*/true);
}

int gmaco_vehicles_wait(gmaco_engine* h, int32_t slot, const gmaco_vehicle_view* view) {
  NvtxRange nvtx_(__func__);
  if (!h || !view || slot < 0 || slot > 1) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    auto& rs = h->rslot[slot];
    if (!rs.armed) throw ValidationError("vehicles_wait: no snapshot enqueued in this slot");
    // exactly the members the snapshot was taken for: the copies below are
    // sized by the snapshot's fields, so any other set could overrun `view`
    if (view_mask(view) != rs.mask)
      throw ValidationError("vehicles_wait: view fields differ from the enqueued snapshot");
    const auto f = vehicle_fields(h, view);
    CK(cudaEventSynchronize(rs.done));  // only this snapshot, not later steps
    const char* st = static_cast<const char*>(rs.buf);
    for (size_t i = 0; i < f.size(); ++i) std::memcpy(std::get<0>(f[i]), st + rs.fields[i].first, rs.fields[i].second);
    if (rs.on_edge) {
      const int32_t* oe = reinterpret_cast<const int32_t*>(st + rs.oe_off);
      for (size_t i = 0; i < (size_t)h->w.p.V; ++i) view->on_edge[i] = oe[i] < 0 ? -1 : h->slot_edge[oe[i]];
    }
    if (view->speed_mps) {
      const DrawStream sp(h->cfg.seed, 3);
      for (size_t i = 0; i < (size_t)h->w.p.V; ++i)
        view->speed_mps[i] = uniform(sp(i), h->cfg.speed_min_mps, h->cfg.speed_max_mps);
    }
    rs.armed = false;
  }, /*stream_ordered=*/true);
}

int gmaco_debug_check_redzones(gmaco_engine* h, int64_t* corrupted) {
  NvtxRange nvtx_(__func__);
  if (!h || !corrupted) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    CK(cudaStreamSynchronize(h->stream));
    if (!h->buf.redzones) throw ValidationError("check_redzones: the world was created without GMACO_OPT_REDZONES");
    int64_t bad = 0;
    std::string first;
    std::vector<unsigned char> tmp;
    for (size_t i = 0; i < h->buf.zones.size(); ++i) {
      const auto& z = h->buf.zones[i];
      tmp.resize(z.second);
      CK(cudaMemcpy(tmp.data(), z.first, z.second, cudaMemcpyDeviceToHost));
      for (size_t b = 0; b < z.second; ++b)
        if (tmp[b] != DevBuffers::kRedzoneByte) {
          if (!bad) first = fmt("guard %zu (%p) byte %zu overwritten", i, (const void*)z.first, b);
          ++bad;
          break;
        }
    }
    *corrupted = bad;
    h->err = bad ? first : fmt("%zu guards intact", h->buf.zones.size());
  });
}

int gmaco_signal_count(gmaco_engine* h, int32_t* out) {
  if (!h || !out) return GMACO_EVALIDATION;
  *out = h->S;
  return GMACO_OK;
}

int gmaco_get_signals(gmaco_engine* h, const gmaco_signal_view* v, int64_t cap) {
  NvtxRange nvtx_(__func__);
  if (!h || !v) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    const DevSignals& d = h->w.s;
    const size_t S = h->S, Q = S * kPhases;
    auto cp = [&](auto* dst, const auto* src, size_t n) {
      if (dst) CK(cudaMemcpy(dst, src, n * sizeof(*dst), cudaMemcpyDeviceToHost));
    };
    if (v->node) std::copy(h->sig_node.begin(), h->sig_node.end(), v->node);
    cp(v->green, d.green, S);
    cp(v->cycle_cursor, d.cursor, S);
    cp(v->discharge_lanes, d.lanes, S);
    cp(v->green_elapsed_steps, d.el_steps, S);
    cp(v->green_elapsed_s, d.el_s, S);
    cp(v->queue_len, d.qlen, Q);
    cp(v->head_wait_s, d.head_wait, Q);
    cp(v->service_remainder, d.rem, Q);
    if (v->queue_vid || v->queue_enqueue_step) {
      auto qlen = download(d.qlen, Q);
      auto qhead = download(d.qhead, Q);
      auto qnext = download(h->w.v.qnext, h->w.p.V);
      auto joined = download(h->w.v.joined, h->w.p.V);
      int64_t k = 0;
      for (size_t q = 0; q < Q; ++q) {
        int32_t vid = qhead[q];
        for (int32_t j = 0; j < qlen[q]; ++j, ++k) {
          if (k < cap) {
            if (v->queue_vid) v->queue_vid[k] = vid;
            if (v->queue_enqueue_step) v->queue_enqueue_step[k] = joined[vid];
          }
          vid = qnext[vid];
        }
      }
      if (k > cap) throw ValidationError("gmaco_get_signals: queue_cap too small");
    }
  });
}

int gmaco_get_counters(gmaco_engine* h, gmaco_counters* out) {
  if (!h || !out) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    refresh_ctl(h);
    const DevCtl& c = *h->ctl_host;
    out->ant_steps = c.ant_steps;
    out->vehicle_routes = c.vehicle_routes;
    out->decisions = c.decisions;
    out->candidates = c.candidates;
    out->degree_sum = c.degree_sum;
    out->kernels_per_step = kernels_per_step(h->w, h->res);
    // algorithmic bytes of the walks, SURVEY §8(d) / DESIGN.md §5: per
    // ant-step 8 (row pair) + 4 per scanned neighbour (column) + 4 per scanned
    // neighbour (int32 distance; 0 with the grid closed form) + 12 per
    // candidate (int32 tau + f64 eta) + 4 (tour write; 0 when tours are not
    // stored).  Independent of this engine's layouts (bitmaps, records).
    const DevWorld& w = h->w;
    const int64_t tour = w.p.scratch_mode ? 4 : 0;
    out->walk_bytes = (8 + tour) * c.ant_steps + 4 * c.degree_sum + (w.d.kind == 1 ? 0 : 4 * c.degree_sum) +
                      12 * c.candidates;
  });
}

int gmaco_route_query(gmaco_engine* h, int32_t vid, int32_t planned, int32_t* out_edges, int32_t cap,
                      int32_t* out_len) {
  NvtxRange nvtx_(__func__);
  if (!h || !out_len) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    const DevWorld& w = h->w;
    if (vid < 0 || vid >= w.p.V) throw ValidationError(fmt("route_query: invalid vehicle %d", vid));
    int32_t n = 0;
    const int32_t* base;
    int32_t pcap;
    if (planned) {
      if (w.p.algorithm != GMACO_COLONY) throw ValidationError("route_query: planned routes need the colony algorithm");
      CK(cudaMemcpy(&n, w.v.plan_n + vid, 4, cudaMemcpyDeviceToHost));
      pcap = w.p.plan_cap;
      if (w.p.scratch_mode) {  // the winner's row of the per-ant tour scratch
        int32_t ant = 0;
        CK(cudaMemcpy(&ant, w.v.plan_ant + vid, 4, cudaMemcpyDeviceToHost));
        base = w.v.scratch + ((size_t)vid * w.p.ants + ant) * pcap;
      } else {
        base = w.v.plan + (size_t)vid * pcap;
      }
    } else {
      if (!w.p.record_paths) throw ValidationError("route_query: realized paths are not recorded for this config");
      CK(cudaMemcpy(&n, w.v.path_n + vid, 4, cudaMemcpyDeviceToHost));
      pcap = w.p.path_cap;
      base = w.v.path + (size_t)vid * pcap;
    }
    *out_len = n;
    const int32_t k = std::min(n, cap);
    if (k > 0 && out_edges) {
      std::vector<int32_t> s(k);
      CK(cudaMemcpy(s.data(), base, k * 4, cudaMemcpyDeviceToHost));
      for (int32_t i = 0; i < k; ++i) out_edges[i] = h->slot_edge[s[i]];
    }
  });
}

int gmaco_next_node(gmaco_engine* h, int32_t algorithm, int32_t count, const int32_t* current, const int32_t* dest,
                    const uint64_t* rng_entity, const uint64_t* rng_step, int64_t n_t, int32_t* out_next,
                    int32_t* out_via, uint8_t* out_deviated) {
  NvtxRange nvtx_(__func__);
  if (!h) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    if (count < 0) throw ValidationError("next_node: negative count");
    if (count == 0) return;
    if (algorithm < GMACO_DIJKSTRA || algorithm > GMACO_MACO_P)
      throw ValidationError(fmt("next_node: unsupported algorithm %d", algorithm));
    for (int32_t i = 0; i < count; ++i)
      if (current[i] < 0 || current[i] >= h->g.n || dest[i] < 0 || dest[i] >= h->g.n)
        throw ValidationError("next_node: invalid node id");
    DevBuffers tmp;
    std::vector<int32_t> c(current, current + count), d(dest, dest + count);
    std::vector<uint64_t> e(count, 0), s(count, 0);
    if (rng_entity) e.assign(rng_entity, rng_entity + count);
    if (rng_step) s.assign(rng_step, rng_step + count);
    int32_t* dc = tmp.upload(c);
    int32_t* dd = tmp.upload(d);
    uint64_t* de = tmp.upload(e);
    uint64_t* ds = tmp.upload(s);
    int32_t* on = tmp.alloc<int32_t>(count);
    int32_t* ov = tmp.alloc<int32_t>(count);
    uint8_t* odv = tmp.alloc<uint8_t>(count);
    CK(launch_next_node(h->w, algorithm == GMACO_MACO_P ? GMACO_MACO : algorithm, count, dc, dd, de, ds, n_t, on,
                        ov, odv, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(out_next, on, count * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_via, ov, count * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_deviated, odv, count, cudaMemcpyDeviceToHost));
  });
}

int gmaco_debug_roulette_threshold(gmaco_engine* h, int32_t count, const double* wa, const double* wb,
                                   uint64_t* out) {
  NvtxRange nvtx_(__func__);
  if (!h || count < 0 || (count > 0 && (!wa || !wb || !out))) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    if (count == 0) return;
    DevBuffers tmp;
    std::vector<double> a(wa, wa + count), b(wb, wb + count);
    const double* da = tmp.upload(a);
    const double* db = tmp.upload(b);
    uint64_t* dout = tmp.alloc<uint64_t>(count);
    CK(launch_threshold_batch(count, da, db, dout, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(out, dout, (size_t)count * 8, cudaMemcpyDeviceToHost));
  });
}

// One graph per timed step: the L2 flush (outside the timed span), then the
// step bracketed by three event-record nodes (begin, walk end, step end).
// mode: 1 = step only (ev0, step, ev2), 2 = walk only (ev0, walk, ev1, tail),
// 3 = both.  Every event-record node serializes the GPU (~2-3 us on B200),
// so the headline leg brackets each step with exactly two.
void build_bench_graph(gmaco_engine* h, int64_t flush_bytes, int mode) {
  if (h->bench_exec) cudaGraphExecDestroy(h->bench_exec);
  if (h->bench_tmpl) cudaGraphDestroy(h->bench_tmpl);
  h->bench_exec = nullptr;
  h->bench_tmpl = nullptr;
  for (auto& e : h->bench_ev)
    if (!e) CK(cudaEventCreate(&e));
  StepResources r = h->res;
  r.capturing = true;
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t err = cudaSuccess;
  if (flush_bytes > 0) err = cudaMemsetAsync(h->flush, 0x5a, flush_bytes, h->stream);
  if (err == cudaSuccess) err = launch_step(h->w, r, h->stream, h->bench_ev[0], (mode & 2) ? h->bench_ev[1] : nullptr);
  if (err == cudaSuccess && (mode & 1))
    err = cudaEventRecordWithFlags(h->bench_ev[2], h->stream, cudaEventRecordExternal);
  cudaError_t e2 = cudaStreamEndCapture(h->stream, &h->bench_tmpl);
  CK(err);
  CK(e2);
  size_t nn = 0;
  CK(cudaGraphGetNodes(h->bench_tmpl, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  CK(cudaGraphGetNodes(h->bench_tmpl, nodes.data(), &nn));
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    CK(cudaGraphNodeGetType(nd, &t));
    if (t != cudaGraphNodeTypeEventRecord) continue;
    cudaEvent_t e = nullptr;
    CK(cudaGraphEventRecordNodeGetEvent(nd, &e));
    for (int k = 0; k < 3; ++k)
      if (e == h->bench_ev[k]) h->bench_ev_node[k] = nd;
  }
  if (!h->bench_ev_node[0] || ((mode & 2) && !h->bench_ev_node[1]) || ((mode & 1) && !h->bench_ev_node[2]))
    throw std::runtime_error("bench graph: event node not found");
  CK(cudaGraphInstantiate(&h->bench_exec, h->bench_tmpl, 0));
  CK(cudaGraphUpload(h->bench_exec, h->stream));
  h->bench_flush = flush_bytes;
  h->bench_mode = mode;
}

int gmaco_bench_steps(gmaco_engine* h, int32_t steps, int64_t flush_bytes, double* walk_ms, double* step_ms) {
  NvtxRange nvtx_(__func__);
  if (!h || steps < 0) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    refresh_ctl(h);
    unbound_stop(h);
    h->ctl_valid = false;
    if (flush_bytes > 0 && h->flush_bytes < flush_bytes) {
      if (h->flush) cudaFree(h->flush);
      CK(cudaMalloc(&h->flush, flush_bytes));
      h->flush_bytes = flush_bytes;
      h->bench_flush = -1;
    }
    const int mode = (step_ms ? 1 : 0) | (walk_ms ? 2 : 0);
    if (!mode) throw ValidationError("bench_steps: walk_ms or step_ms required");
    if (!h->bench_exec || h->bench_flush != flush_bytes || h->bench_mode != mode) {
      for (auto& nd : h->bench_ev_node) nd = nullptr;
      build_bench_graph(h, flush_bytes, mode);
    }
    std::vector<cudaEvent_t> ev(3 * (size_t)steps);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    for (int32_t i = 0; i < steps; ++i) {
      for (int k = 0; k < 3; ++k)
        if (h->bench_ev_node[k])
          CK(cudaGraphExecEventRecordNodeSetEvent(h->bench_exec, h->bench_ev_node[k], ev[3 * i + k]));
      CK(cudaGraphLaunch(h->bench_exec, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    for (int32_t i = 0; i < steps; ++i) {
      float a = 0.f, b = 0.f;
      if (walk_ms) {
        CK(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 1]));
        walk_ms[i] = a;
      }
      if (step_ms) {
        CK(cudaEventElapsedTime(&b, ev[3 * i], ev[3 * i + 2]));
        step_ms[i] = b;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    refresh_ctl(h);
  });
}

// Profiling hook: stage timestamps (%globaltimer ns) of the next `steps`
// steps' LAST step; see DevCtl::trace.  Not part of the reference surface.
int gmaco_debug_trace(gmaco_engine* h, int32_t steps, uint64_t* out16) {
  if (h) h->ctl_valid = false;
  if (!h || !out16) return GMACO_EVALIDATION;
  return guarded(h, [&] {
    for (int32_t i = 0; i < steps; ++i) {
      DevCtl t;
      CK(cudaMemcpy(&t, h->ctl, sizeof t, cudaMemcpyDeviceToHost));
      t.trace_on = 1;
      for (int k = 0; k < 16; ++k) t.trace[k] = (k == 0 || k == 3) ? ~0ull : 0ull;
      h2d(h, h->ctl, &t, sizeof t);
      run_steps(h, 1);
    }
    DevCtl t;
    CK(cudaMemcpy(&t, h->ctl, sizeof t, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 16; ++k) out16[k] = t.trace[k];
    t.trace_on = 0;
    h2d(h, h->ctl, &t, sizeof t);
  });
}

int gmaco_set_timing(gmaco_engine* h, int32_t enabled) {
  if (!h) return GMACO_EVALIDATION;
  h->timing = enabled != 0;
  return GMACO_OK;
}

int gmaco_last_timing(gmaco_engine* h, double* walk_ms, double* step_ms, int64_t* walk_launches) {
  if (!h) return GMACO_EVALIDATION;
  if (walk_ms) *walk_ms = h->last_walk_ms;
  if (step_ms) *step_ms = h->last_step_ms;
  if (walk_launches) *walk_launches = h->last_walk_launches;
  return GMACO_OK;
}

const char* gmaco_last_error(const gmaco_engine* h) { return h ? h->err.c_str() : g_create_err.c_str(); }

void gmaco_destroy(gmaco_engine* h) { delete h; }

}  // extern "C"
