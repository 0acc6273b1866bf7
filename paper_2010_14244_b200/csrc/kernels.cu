// kernels.cu — sm_100a kernels of one GMACO-P engine step.
//
// Stage map (engine.cpp:352-400 sequential_step):
//   B   k_decide<Dist>  reference routing decision per vehicle
//       k_colony<Dist>  colony: K ants per vehicle walk to the destination
//   C,D,E1 k_signals    density sample, green assignment, FIFO discharge
//   E2  k_move          motion, arrivals, edge-load histogram, next n_t
//   E3  k_e3            enqueue commit in ascending vid + signal timers
//   F   k_scoped        sibling-scoped MACO replay (decrement_siblings_only)
//   F+G k_edges         MACO fold / deposit + evaporation + next-step weights
// The whole step is free of floating-point atomics: every cross-thread
// reduction is an integer sum/min/max, so results are bit-deterministic.
// Floating-point expressions use explicit _rn intrinsics (and the library is
// built with -fmad=false) so they round exactly like the reference's
// FMA-free x86-64 build.

#include <cooperative_groups.h>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.cuh"
#include "gmaco.h"
#include "kernels.h"

namespace gmaco {

namespace cg = cooperative_groups;
constexpr int kTailCoop = 128;
constexpr int kSigCtas = 8;  // walk-kernel CTAs running stages C, D, E1 (e1_in_walk)

// ---------------------------------------------------------------------------
// counter-based RNG (rng.hpp:21-56) and Philox4x32-10
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t h = mix64(seed);
  h = mix64(h ^ a);
  h = mix64(h ^ b);
  return mix64(h ^ c);
}
__device__ __forceinline__ double to_unit(uint64_t bits) {
  return __dmul_rn((double)(bits >> 11), 0x1.0p-53);
}
// Philox4x32-10 (Salmon et al., SC'11).  One call serves two hops: the
// counter is (step, vehicle, ant, hop/2) and hop&1 selects the 64-bit half.
__device__ __forceinline__ uint4 philox4(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}
// Same function with the key schedule precomputed on the host:
// rk[2r], rk[2r+1] = key words of round r (kernel-parameter constants).
__device__ __forceinline__ uint4 philox4_rk(uint4 c, const uint32_t* rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ rk[2 * r], lo1, hi0 ^ c.w ^ rk[2 * r + 1], lo0);
  }
  return c;
}
// Rounds [R0, R1) of philox4_rk, so callers can interleave a block's rounds
// with independent dependent chains (warps issue in order).
template <int R0, int R1>
__device__ __forceinline__ void philox_rounds(uint4& c, const uint32_t* rk) {
#pragma unroll
  for (int r = R0; r < R1; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ rk[2 * r], lo1, hi0 ^ c.w ^ rk[2 * r + 1], lo0);
  }
}
__device__ __forceinline__ uint64_t philox_half(uint4 o, int32_t hop) {
  return (hop & 1) ? (((uint64_t)o.z << 32) | o.w) : (((uint64_t)o.x << 32) | o.y);
}
// Ant uniform: REFERENCE keying reduces to RngKey{seed, vid, step} of the
// reference ACO decision at ant 0 hop 0 (routing.cpp:97-98).
__device__ __forceinline__ double ant_uniform(int rng, uint64_t seed, int64_t step, int32_t vid,
                                              int32_t ant, int32_t hop) {
  if (rng == 1) {
    const uint64_t a = (uint64_t)(uint32_t)vid | ((uint64_t)(uint32_t)ant << 32);
    const uint64_t b = (uint64_t)step | ((uint64_t)(uint32_t)hop << 40);
    return to_unit(draw(seed, 5, a, b));
  }
  const uint4 o = philox4(make_uint4((uint32_t)step, (uint32_t)vid, (uint32_t)ant, (uint32_t)hop >> 1),
                          (uint32_t)seed, (uint32_t)(seed >> 32));
  return to_unit(philox_half(o, hop));
}

// ---------------------------------------------------------------------------
// distance service
// ---------------------------------------------------------------------------
template <int DK>
struct Target {
  int32_t dest;
  int32_t rd, cd, cols;
  int64_t len;
  const int64_t* __restrict__ trow;
  __device__ __forceinline__ Target(const DevDist& d, int32_t dst) : dest(dst) {
    if (DK == 1) {
      cols = d.cols;
      rd = dst / d.cols;
      cd = dst - rd * d.cols;
      len = d.grid_len;
      trow = nullptr;
    } else {
      const int32_t slot = d.slot_of ? d.slot_of[dst] : dst;
      trow = slot < 0 ? nullptr : d.table + (size_t)slot * d.n;
    }
  }
  __device__ __forceinline__ int64_t dist(int32_t x) const {
    if (DK == 1) {
      const int32_t r = x / cols, c = x - r * cols;
      return (int64_t)(abs(r - rd) + abs(c - cd)) * len;
    }
    return trow ? __ldg(trow + x) : kInf;
  }
};

// Candidate scan of node x (candidate_neighbors, routing.cpp:16-30) as
// register bitmasks over the row's slot offsets (ascending neighbour id).
struct Row {
  int32_t first, deg;
  uint32_t reach, closer, sp;  // reachable / strictly closer / on a shortest path
  int64_t dx;
};

template <int DK>
__device__ __forceinline__ Row scan_row(const DevGraph& g, const Target<DK>& t, int32_t x) {
  Row r;
  const int2 ri = __ldg(g.row + x);
  r.first = ri.x;
  r.deg = 0;
  r.dx = t.dist(x);
  r.reach = r.closer = r.sp = 0u;
  for (int i = 0; i < ri.y; ++i) {  // ri.y = row span; ELL rows may hold holes (col -1)
    const int32_t nb = __ldg(g.col + r.first + i);
    if (nb < 0) continue;
    ++r.deg;
    const int64_t dn = t.dist(nb);
    if (dn == kInf) continue;
    r.reach |= 1u << i;
    if (dn < r.dx) r.closer |= 1u << i;
  }
  return r;
}

// Dijkstra hop: smallest neighbour on a shortest path (greedy_hop,
// net.cpp:387-395; next_node_dijkstra, routing.cpp:117-125).
template <int DK>
__device__ __forceinline__ int32_t dijkstra_pick(const DevGraph& g, const Target<DK>& t, int32_t x) {
  const int64_t dx = t.dist(x);
  if (dx == kInf) return -1;
  const int2 ri = __ldg(g.row + x);
  for (int i = 0; i < ri.y; ++i) {
    const int32_t s = ri.x + i;
    const int32_t nb = __ldg(g.col + s);
    if (nb < 0) continue;
    const int64_t dn = t.dist(nb);
    if (dn == kInf) continue;
    if (__ldg(g.len + s) + dn == dx) return s;
  }
  return -1;
}

// ACO roulette over candidate mask (routing.cpp:88-113): sequential
// left-to-right total and cumulative sums, u·total point, uniform fallback.
__device__ __forceinline__ int32_t roulette_pick(const double* __restrict__ W, int32_t first,
                                                 uint32_t cand, double u) {
  double total = 0.0;
  int c = 0;
  for (uint32_t m = cand; m; m &= m - 1) {
    total = __dadd_rn(total, W[first + __ffs(m) - 1]);
    ++c;
  }
  int pick_i = c - 1;
  if (total <= 0.0 || !isfinite(total)) {
    int p = (int)__dmul_rn(u, (double)c);
    pick_i = p < c - 1 ? p : c - 1;
  } else {
    const double point = __dmul_rn(u, total);
    double cum = 0.0;
    int i = 0;
    for (uint32_t m = cand; m; m &= m - 1, ++i) {
      cum = __dadd_rn(cum, W[first + __ffs(m) - 1]);
      if (point < cum) {
        pick_i = i;
        break;
      }
    }
  }
  uint32_t m = cand;
  for (int i = 0; i < pick_i; ++i) m &= m - 1;
  return first + __ffs(m) - 1;
}

// MACO min-pheromone with deviation (routing.cpp:32-75).
__device__ __forceinline__ int32_t maco_pick(const DevWorld& w, int32_t first, uint32_t cand,
                                             int64_t n_t, bool* deviated) {
  int32_t prim = -1, c = 0;
  int64_t tp = 0;
  for (uint32_t m = cand; m; m &= m - 1, ++c) {
    const int32_t s = first + __ffs(m) - 1;
    const int64_t t = w.tau[s];
    if (prim < 0 || t < tp) {
      prim = s;
      tp = t;
    }
  }
  bool trigger = false;
  if (c >= 2) {
    if (w.p.deviation_mode == 0)
      trigger = n_t > w.p.deviation_threshold;
    else
      trigger = (int64_t)w.occ_cur[prim] > w.p.deviation_threshold;
  }
  *deviated = trigger;
  if (!trigger) return prim;
  // second: initial = candidate 1 if primary is candidate 0 else candidate 0
  const int32_t c0 = first + __ffs(cand) - 1;
  const uint32_t rest = cand & (cand - 1);
  int32_t second = prim == c0 ? first + __ffs(rest) - 1 : c0;
  int64_t ts = w.tau[second];
  for (uint32_t m = cand; m; m &= m - 1) {
    const int32_t s = first + __ffs(m) - 1;
    if (s == prim || s == second) continue;
    const int64_t t = w.tau[s];
    if (t < ts) {
      second = s;
      ts = t;
    }
  }
  return second;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_min(DevCtl* c, int i) {
  if (c->trace_on) atomicMin(&c->trace[i], gtimer());
}
__device__ __forceinline__ void trace_max(DevCtl* c, int i) {
  if (c->trace_on) atomicMax(&c->trace[i], gtimer());
}

// finer stage stamps (tools/stage_trace.py), compiled in with -DGMACO_TRACE_FINE
#ifdef GMACO_TRACE_FINE
#define TRACE_FINE(i) trace_max(w.ctl, i)
#else
#define TRACE_FINE(i) (void)0
#endif

// atom.add with acquire-release semantics at GPU scope (last-block detection
// without a separate full fence)
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ bool skip_step(const DevCtl* ctl) {
  return ctl->done || ctl->step >= ctl->stop_at;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* smem) {
  // Reconverge first: a warp whose lanes arrive from divergent work (e.g.
  // one lane running a vehicle's epilogue) otherwise lets the waiting lanes'
  // shuffle starve it — measured ~10 us per step on C1 (K = 20) without this.
  __syncwarp();
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  T r = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)((blockDim.x + 31) >> 5); ++i) r += smem[i];
  return r;  // valid in thread 0
}

// Bulk L2 prefetch (TMA engine, cp.async.bulk.prefetch.L2) of every array
// the rest of the step touches, issued by one block at the start of the walk
// so stages C..G find their state in L2.  Fire-and-forget: no completion wait.
__device__ __forceinline__ void bulk_prefetch(const void* p, size_t bytes, int lane, int lanes) {
  const char* c = static_cast<const char*>(p);
  const size_t n = bytes & ~size_t(15);
  constexpr size_t kChunk = 1 << 16;
  for (size_t off = (size_t)lane * kChunk; off < n; off += (size_t)lanes * kChunk) {
    const uint32_t sz = (uint32_t)min(n - off, kChunk);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c + off), "r"(sz) : "memory");
  }
}

__device__ void prefetch_tail_state(const DevWorld& w) {
  const size_t V = w.p.V, Q = (size_t)w.p.S * kPhases, S = w.p.S, M = w.g.M;
  const int lane = threadIdx.x, lanes = blockDim.x;
  const DevVehicles& v = w.v;
  const DevSignals& g = w.s;
  bulk_prefetch(v.state, V, lane, lanes);
  bulk_prefetch(v.on_edge, 4 * V, lane, lanes);
  bulk_prefetch(v.at_node, 4 * V, lane, lanes);
  bulk_prefetch(v.dest, 4 * V, lane, lanes);
  bulk_prefetch(v.progress, 8 * V, lane, lanes);
  bulk_prefetch(v.advance, 8 * V, lane, lanes);
  bulk_prefetch(v.latency_debt, 8 * V, lane, lanes);
  bulk_prefetch(v.driving, 8 * V, lane, lanes);
  bulk_prefetch(v.depart, 8 * V, lane, lanes);
  bulk_prefetch(v.joined, 8 * V, lane, lanes);
  bulk_prefetch(v.queued, 8 * V, lane, lanes);
  bulk_prefetch(v.qnext, 4 * V, lane, lanes);
  bulk_prefetch(g.qlen, 4 * Q, lane, lanes);
  bulk_prefetch(g.qhead, 4 * Q, lane, lanes);
  bulk_prefetch(g.qtail, 4 * Q, lane, lanes);
  bulk_prefetch(g.arr_head, 4 * Q, lane, lanes);
  bulk_prefetch(g.head_wait, 8 * Q, lane, lanes);
  bulk_prefetch(g.rem, 8 * Q, lane, lanes);
  bulk_prefetch(g.green, 4 * S, lane, lanes);
  bulk_prefetch(g.cursor, 4 * S, lane, lanes);
  bulk_prefetch(g.lanes, 4 * S, lane, lanes);
  bulk_prefetch(g.node, 4 * S, lane, lanes);
  bulk_prefetch(g.el_s, 8 * S, lane, lanes);
  bulk_prefetch(g.el_steps, 8 * S, lane, lanes);
  bulk_prefetch(w.tau, 8 * M, lane, lanes);
  bulk_prefetch(w.occ_new, 4 * M, lane, lanes);
  bulk_prefetch(w.dep, 8 * M, lane, lanes);
  bulk_prefetch(w.g.slot_edge, 4 * M, lane, lanes);
  bulk_prefetch(w.g.bind, 4 * M, lane, lanes);
  bulk_prefetch(w.g.len, 8 * M, lane, lanes);
  bulk_prefetch(w.g.eta_beta, 8 * M, lane, lanes);
}

// Five block-wide sums with a single barrier; valid in thread 0.
struct Sum5 {
  long long v[7];  // ant_steps, candidates, degree_sum, routes, decisions, active(next), unfinished
};
__device__ __forceinline__ Sum5 block_sum5(Sum5 x, long long (*smem)[32]) {
  __syncwarp();  // reconverge first (see block_sum)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    long long a = x.v[k];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if (lane == 0) smem[k][wid] = a;
  }
  __syncthreads();
  Sum5 r{};
  if (threadIdx.x == 0)
    for (int k = 0; k < 7; ++k)
      for (int i = 0; i < (int)((blockDim.x + 31) >> 5); ++i) r.v[k] += smem[k][i];
  return r;
}

__device__ __forceinline__ void flush_counters(DevCtl* c, const Sum5& t) {
  if (t.v[0]) atomicAdd((unsigned long long*)&c->ant_steps, (unsigned long long)t.v[0]);
  if (t.v[1]) atomicAdd((unsigned long long*)&c->candidates, (unsigned long long)t.v[1]);
  if (t.v[2]) atomicAdd((unsigned long long*)&c->degree_sum, (unsigned long long)t.v[2]);
  if (t.v[3]) atomicAdd((unsigned long long*)&c->vehicle_routes, (unsigned long long)t.v[3]);
  if (t.v[4]) {
    atomicAdd((unsigned long long*)&c->decisions, (unsigned long long)t.v[4]);
    atomicAdd((unsigned long long*)&c->dcount, (unsigned long long)t.v[4]);
  }
  if (t.v[5]) atomicAdd((unsigned long long*)&c->n_next, (unsigned long long)t.v[5]);
  if (t.v[6]) atomicAdd((unsigned long long*)&c->unfinished, (unsigned long long)t.v[6]);
}

// Vehicle takes edge `slot` (engine.cpp:207-216).
__device__ __forceinline__ void take_edge(const DevWorld& w, int32_t vid, int32_t slot, bool deviated,
                                          int32_t from) {
  const DevVehicles& v = w.v;
  // every load ahead of the first store (the compiler may not move a load
  // past a possibly aliasing store): one memory round trip, not one per field
  const int64_t overshoot = v.overshoot[vid];
  const int64_t debt = v.latency_debt[vid];
  const int32_t ndec = v.decisions[vid];
  const int32_t ndev = deviated ? v.deviations[vid] : 0;
  const int32_t k = w.p.record_paths ? v.path_n[vid] : 0;
  const int64_t plen = v.path_len_mm[vid];
  const int64_t elen = w.g.len[slot];
  if (w.p.sharded) v.dec_rec[vid] = slot | (deviated ? GMACO_REC_DEVIATED : 0);
  v.state[vid] = kOnEdge;
  v.on_edge[vid] = slot;
  v.progress[vid] = overshoot;
  v.overshoot[vid] = 0;
  v.latency_debt[vid] = debt + w.p.latency_us;
  v.decisions[vid] = ndec + 1;
  if (deviated) v.deviations[vid] = ndev + 1;
  if (w.p.record_paths) {
    if (k < w.p.path_cap) {
      v.path[(size_t)vid * w.p.path_cap + k] = slot;
      v.path_n[vid] = k + 1;
    } else {
      atomicExch(&w.ctl->error, 1);  // path buffer overflow → host error
    }
  }
  v.path_len_mm[vid] = plen + elen;
  if (w.p.algorithm == 2 || w.p.algorithm == 3) {  // MACO commit bookkeeping
    const int32_t key = w.p.siblings_only ? from : slot;
    v.dec_next[vid] = atomicExch(&w.dec_head[key], vid);
  }
}

// ---------------------------------------------------------------------------
// B: reference decision kernel (dijkstra / aco / maco), one thread per vehicle
// ---------------------------------------------------------------------------
// One vehicle's stage B (engine.cpp:175-217): activation, the routing
// decision, its bookkeeping; adds to the block's counters.
template <int DK>
__device__ __forceinline__ void decide_vehicle(const DevWorld& w, int32_t vid, int64_t step, long long& decided,
                                               long long& cands, long long& degs) {
  const DevVehicles& v = w.v;
  // the vehicle's words in one round of loads, ahead of any store
  uint8_t st = v.state[vid];
  const int64_t depart = v.depart[vid];
  int32_t x = v.at_node[vid];
  const int32_t origin = v.origin[vid];
  const int32_t dest = v.dest[vid];
  if (w.p.sharded) v.dec_rec[vid] = -1;
  if (st == kPending && depart == step) {  // engine.cpp:177-180
    st = kAtNode;
    v.state[vid] = kAtNode;
    v.at_node[vid] = origin;
    x = origin;
  }
  if (w.p.need_positions) v.dflag[vid] = 0;
  if (st != kAtNode) return;
  const Target<DK> t(w.d, dest);
  int32_t slot = -1;
  bool dev = false;
  if (w.p.algorithm == 0) {
    slot = dijkstra_pick<DK>(w.g, t, x);
  } else {
    const Row r = scan_row<DK>(w.g, t, x);
    degs += r.deg;
    const uint32_t cand = (w.p.progress_filter && r.closer) ? r.closer : r.reach;
    if (cand) {
      cands += __popc(cand);
      if (w.p.algorithm == 1) {
        const double u = to_unit(draw(w.p.seed, 5, (uint64_t)vid, (uint64_t)step));
        slot = roulette_pick(w.weight, r.first, cand, u);
      } else {
        slot = maco_pick(w, r.first, cand, w.ctl->n_t, &dev);
      }
    }
  }
  if (slot < 0) {
    v.state[vid] = kRetired;  // engine.cpp:202-205
    if (w.p.sharded) v.dec_rec[vid] = -2;
  } else {
    take_edge(w, vid, slot, dev, x);
    if (w.p.need_positions) v.dflag[vid] = 1;
    decided = 1;
  }
}

__device__ __forceinline__ void flush_decide_counters(const DevWorld& w, long long decided, long long cands,
                                                      long long degs, long long* red) {
  const long long d = block_sum(decided, red);
  const long long c = block_sum(cands, red);
  const long long g = block_sum(degs, red);
  if (threadIdx.x == 0 && d) {
    atomicAdd((unsigned long long*)&w.ctl->dcount, (unsigned long long)d);
    atomicAdd((unsigned long long*)&w.ctl->decisions, (unsigned long long)d);
    atomicAdd((unsigned long long*)&w.ctl->ant_steps, (unsigned long long)d);
  }
  if (threadIdx.x == 0 && (c || g)) {
    atomicAdd((unsigned long long*)&w.ctl->candidates, (unsigned long long)c);
    atomicAdd((unsigned long long*)&w.ctl->degree_sum, (unsigned long long)g);
  }
}

template <int DK>
__global__ void __launch_bounds__(256) k_decide(DevWorld w) {
  if (skip_step(w.ctl)) return;
  if (blockIdx.x == 0 && w.p.prefetch) prefetch_tail_state(w);
  __shared__ long long red[32];
  // sharded: this rank decides vehicles [shard_lo, shard_hi); the others'
  // records arrive with the exchange (k_apply_remote)
  const int32_t vid = w.p.shard_lo + blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t step = w.ctl->step;
  long long decided = 0, cands = 0, degs = 0;
  if (vid < w.p.shard_hi) decide_vehicle<DK>(w, vid, step, decided, cands, degs);
  flush_decide_counters(w, decided, cands, degs, red);
}

// ---------------------------------------------------------------------------
// B (colony): K ants per vehicle, one thread per ant; best tour by
// (cost, ant) via a shared-memory 64-bit atomicMin; the winner replays its
// walk (counter RNG) to materialize the tour.
// ---------------------------------------------------------------------------
constexpr uint64_t kCostCap = (1ull << 53) - 1;

struct WalkOut {
  int64_t cost;
  int32_t hops;
  bool first_ok;
  long long steps, cands, degs;
};

template <int DK, bool kFilter>
__device__ __forceinline__ WalkOut ant_walk(const DevWorld& w, const Target<DK>& t, int32_t vid,
                                            int32_t ant, int32_t start, int64_t step,
                                            int32_t* __restrict__ tour) {
  WalkOut o{0, 0, false, 0, 0, 0};
  const int32_t dest = t.dest;
  const int32_t max_hops = w.p.max_hops;
  const int32_t hop_limit = w.p.hop_limit;
  int32_t tabu[kTabu];
  int32_t ntabu = 0, tpos = 0;
  if (!kFilter) {
    tabu[0] = start;
    ntabu = 1;
    tpos = 1;
  }
  int32_t x = start;
  while (x != dest && (hop_limit == 0 || o.hops < hop_limit)) {
    if (o.hops >= max_hops) {
      o.cost = kInf;
      return o;
    }
    const Row r = scan_row<DK>(w.g, t, x);
    uint32_t cand;
    if (kFilter) {
      cand = r.closer ? r.closer : r.reach;
    } else {
      cand = r.reach;
      for (uint32_t m = cand; m; m &= m - 1) {
        const int i = __ffs(m) - 1;
        const int32_t nb = __ldg(w.g.col + r.first + i);
        for (int k = 0; k < ntabu; ++k)
          if (tabu[k] == nb) cand &= ~(1u << i);
      }
    }
    o.degs += r.deg;
    if (!cand) {
      o.cost = kInf;
      return o;
    }
    if (o.hops == 0) o.first_ok = true;
    o.cands += __popc(cand);
    const double u = ant_uniform(w.p.rng, w.p.seed, step, vid, ant, o.hops);
    const int32_t s = roulette_pick(w.weight, r.first, cand, u);
    o.cost += w.ecost[s];
    x = __ldg(w.g.col + s);
    if (tour) tour[o.hops] = s;
    o.hops++;
    o.steps++;
    if (!kFilter) {
      tabu[tpos] = x;
      tpos = (tpos + 1) % kTabu;
      if (ntabu < kTabu) ntabu++;
    }
  }
  return o;
}

// E2 (motion) of one vehicle; defined with the other per-entity stage bodies.
// Colony walks run it for each vehicle right after that vehicle's stage B.
// The words E2 reads of a vehicle on an edge and of that edge, all loaded in
// one round (MoveWords::load) so that motion is one memory round trip.
struct MoveWords {
  int64_t debt, progress, advance, lat_steps, driving, len;
  int32_t reached, bind;
  __device__ __forceinline__ void load(const DevWorld& w, int32_t vid, int32_t slot) {
    const DevVehicles& v = w.v;
    debt = v.latency_debt[vid];
    progress = v.progress[vid];
    advance = v.advance[vid];
    lat_steps = v.lat_steps[vid];
    driving = v.driving[vid];
    len = w.g.len[slot];
    reached = w.g.col[slot];
    bind = w.g.bind[slot];
  }
};

// E2 (engine.cpp:221-261) for a vehicle whose state words are in registers:
// st, depart, its edge slot and dest, and -- when st == kOnEdge -- MoveWords.
__device__ __forceinline__ void veh_move_core(const DevWorld& w, int32_t vid, int64_t step, uint8_t st,
                                              int64_t depart, int32_t slot, int32_t dest, const MoveWords& m,
                                              long long& active, long long& unfinished) {
  const DevVehicles& v = w.v;
  if (st == kOnEdge) {
    const int64_t prog = m.progress + m.advance;
    const int64_t L = m.len;
    if (m.debt >= w.p.dt_us) {
      v.latency_debt[vid] = m.debt - w.p.dt_us;
      v.lat_steps[vid] = m.lat_steps + 1;
    } else {
      v.driving[vid] = m.driving + 1;
      if (prog < L) {
        v.progress[vid] = prog;
      } else {
        if (m.reached == dest) {
          st = kArrived;
          v.progress[vid] = prog;
          v.arrive[vid] = step + 1;
          if (w.p.deposit == 0 && (w.p.algorithm == 1 || w.p.algorithm == 4)) {
            const int32_t n = v.path_n[vid];
            if (n > 0) {
              const double km = __ddiv_rn((double)v.path_len_mm[vid], 1e6);
              const int64_t amount = llround(__dmul_rn(__ddiv_rn(w.p.deposit_q, km), 1e6));
              const int32_t* path = v.path + (size_t)vid * w.p.path_cap;
              for (int i = 0; i < n; ++i) atomicAdd((unsigned long long*)&w.dep[path[i]], (unsigned long long)amount);
            }
          }
        } else if (m.bind >= 0) {
          st = kQueued;
          v.at_node[vid] = m.reached;
          v.queued_phase[vid] = m.bind & 7;
          v.joined[vid] = step + 1;
          v.progress[vid] = 0;
          v.arr_next[vid] = atomicExch(&w.s.arr_head[m.bind], vid);
          if (w.p.e1_in_walk) atomicAdd(w.s.arr_cnt + (step & 1) * (int64_t)w.p.S * kPhases + m.bind, 1);
        } else {
          st = kAtNode;
          v.at_node[vid] = m.reached;
          v.overshoot[vid] = prog - L;
          v.progress[vid] = 0;
        }
        v.state[vid] = st;
      }
    }
    if (st == kOnEdge) atomicAdd(&w.occ_new[slot], 1);
  }
  active += st == kAtNode || st == kOnEdge || st == kQueued || st == kReleased ||
            (st == kPending && depart == step + 1);
  unfinished += st != kArrived && st != kRetired;
}

// E2 for a vehicle whose state words are in registers (st, depart, on_edge,
// dest): one round of loads (the edge's words included), then the stores.
__device__ __forceinline__ void veh_move_from(const DevWorld& w, int32_t vid, int64_t step, uint8_t st,
                                              int64_t depart, int32_t slot, int32_t dest, long long& active,
                                              long long& unfinished) {
  MoveWords m{};
  if (st == kOnEdge) m.load(w, vid, slot);
  veh_move_core(w, vid, step, st, depart, slot, dest, m, active, unfinished);
}

// E2 for one vehicle: its state words, then the edge's and the motion words
// (two memory round trips).
__device__ __forceinline__ void veh_move(const DevWorld& w, int32_t vid, long long& active, long long& unfinished) {
  const DevVehicles& v = w.v;
  const int64_t step = w.ctl->step;
  const uint8_t st = v.state[vid];
  const int64_t depart = v.depart[vid];
  const int32_t slot = v.on_edge[vid];
  const int32_t dest = v.dest[vid];
  veh_move_from(w, vid, step, st, depart, slot, dest, active, unfinished);
}


// Winner epilogue: plan bookkeeping, best-tour deposit (exact int64 sums,
// deposit_amount pheromone.cpp:73-78) and, at a node, the first hop.
__device__ __forceinline__ void finish_colony(const DevWorld& w, int32_t vid, int32_t start,
                                              const int32_t* tour, int32_t hops, bool deciding, int64_t step) {
  const DevVehicles& v = w.v;
  v.plan_n[vid] = hops;
  v.plan_step[vid] = step;
  const bool done = hops > 0 && w.g.col[tour[hops - 1]] == v.dest[vid];
  v.plan_done[vid] = done;
  if (done && w.p.deposit == 1) {
    int64_t len = 0;
    for (int i = 0; i < hops; ++i) len += w.g.len[tour[i]];
    const double km = __ddiv_rn((double)len, 1e6);
    const int64_t amount = llround(__dmul_rn(__ddiv_rn(w.p.deposit_q, km), 1e6));
    for (int i = 0; i < hops; ++i) atomicAdd((unsigned long long*)&w.dep[tour[i]], (unsigned long long)amount);
  }
  if (deciding) take_edge(w, vid, tour[0], false, start);
}

template <int DK, bool kFilter>
__global__ void __launch_bounds__(1024) k_colony(DevWorld w) {
  if (skip_step(w.ctl)) return;
  if (blockIdx.x == 0 && w.p.prefetch) prefetch_tail_state(w);
  constexpr int kMaxVpb = 256;
  __shared__ unsigned long long best[kMaxVpb];
  __shared__ int32_t start_s[kMaxVpb];
  __shared__ uint8_t deciding_s[kMaxVpb];
  __shared__ long long red5[7][32];
  const int K = w.p.ants;
  const int vpb = blockDim.x / K;
  const int lv = threadIdx.x / K;
  const int ant = threadIdx.x - lv * K;
  const int32_t vid = w.p.shard_lo + blockIdx.x * vpb + lv;
  const bool live = lv < vpb && vid < w.p.shard_hi;
  const int64_t step = w.ctl->step;
  const DevVehicles& v = w.v;

  long long act = 0, unf = 0;  // next step's count_active / unfinished (fused motion)
  if (live && ant == 0) {
    // the vehicle's words in one round of loads, ahead of any store (the
    // prologue runs beside the table staging and must not outlast it)
    uint8_t st = v.state[vid];
    const int64_t depart = v.depart[vid];
    int32_t at = v.at_node[vid];
    const int32_t origin = v.origin[vid];
    const int32_t on_edge = v.on_edge[vid];
    const int32_t dest = v.dest[vid];
    if (st == kPending && depart == step) {  // engine.cpp:177-180
      st = kAtNode;
      at = origin;
      v.state[vid] = kAtNode;
      v.at_node[vid] = origin;
    }
    int32_t start = -1;
    const bool deciding = st == kAtNode;
    if (deciding)
      start = at;
    else if (w.p.replan_all && (st == kQueued || st == kReleased))  // kReleased: queued at stage B
      start = at;
    else if (w.p.replan_all && st == kOnEdge)
      start = w.g.col[on_edge];
    if (start >= 0 && start == dest) {
      v.plan_n[vid] = 0;
      v.plan_step[vid] = step;
      v.plan_done[vid] = 0;
      start = -1;
    }
    start_s[lv] = start;
    deciding_s[lv] = deciding;
    if (w.p.sharded) v.dec_rec[vid] = -1;
    if (start < 0) veh_move(w, vid, act, unf);  // E2 now: stage B leaves this vehicle untouched
    best[lv] = ~0ull;
  }
  __syncthreads();
  long long steps = 0, cands = 0, degs = 0, routes = 0, decided = 0;
  int32_t start = -1;
  WalkOut o{};
  if (live) {
    start = start_s[lv];
    if (start >= 0) {
      const Target<DK> t(w.d, v.dest[vid]);
      int32_t* tour = w.p.scratch_mode
                          ? v.scratch + ((size_t)vid * w.p.ants + ant) * (size_t)w.p.plan_cap
                          : nullptr;
      o = ant_walk<DK, kFilter>(w, t, vid, ant, start, step, tour);
      steps = o.steps;
      cands = o.cands;
      degs = o.degs;
      const uint64_t c = o.cost >= (int64_t)kCostCap ? kCostCap : (uint64_t)o.cost;
      atomicMin(&best[lv], (c << 10) | (uint64_t)ant);
    }
  }
  __syncthreads();
  if (live && start >= 0 && ant == (int)(best[lv] & 1023u)) {
    const bool deciding = deciding_s[lv];
    if (!o.first_ok) {
      v.plan_n[vid] = 0;
      v.plan_step[vid] = step;
      v.plan_done[vid] = 0;
      if (deciding) {
        v.state[vid] = kRetired;
        if (w.p.sharded) v.dec_rec[vid] = -2;
      }
    } else {
      int32_t* tour;
      int32_t hops;
      if (w.p.scratch_mode) {
        tour = v.scratch + ((size_t)vid * w.p.ants + ant) * (size_t)w.p.plan_cap;
        hops = o.hops;
        v.plan_ant[vid] = ant;
      } else {
        const Target<DK> t(w.d, v.dest[vid]);
        tour = v.plan + (size_t)vid * w.p.plan_cap;
        hops = ant_walk<DK, kFilter>(w, t, vid, ant, start, step, tour).hops;
      }
      finish_colony(w, vid, start, tour, hops, deciding, step);
      routes = 1;
      decided = deciding;
    }
    veh_move(w, vid, act, unf);  // E2 right after this vehicle's stage B
  }
  const Sum5 t = block_sum5(Sum5{{steps, cands, degs, routes, decided, act, unf}}, red5);
  if (threadIdx.x == 0) flush_counters(w.ctl, t);
}

// ---------------------------------------------------------------------------
// B (colony) fast path: ELL-4 rows (out-degree <= 4), progress filter on.
// One thread per ant.  Per hop the thread issues ONE round of independent
// row loads — 4 neighbour keys (16 B), 4 roulette weights (32 B), 4 tour
// costs (32 B) — then decides in registers: candidate mask, sequential
// left-to-right roulette (routing.cpp:88-113), Philox draw shared by two
// hops.  Grid distances come from packed (row<<16|col) keys, so the filter
// needs no division and no distance table.  Same semantics as k_colony.
// ---------------------------------------------------------------------------
template <int DK>
__global__ void __launch_bounds__(256) k_colony_ell4(DevWorld w) {
  if (skip_step(w.ctl)) return;
  if (blockIdx.x == 0 && w.p.prefetch) prefetch_tail_state(w);
  constexpr int kMaxVpb = 256;
  __shared__ unsigned long long best[kMaxVpb];
  __shared__ int32_t start_s[kMaxVpb];
  __shared__ uint8_t deciding_s[kMaxVpb];
  __shared__ long long red5[7][32];
  const int K = w.p.ants;
  const int vpb = blockDim.x / K;
  const int lv = threadIdx.x / K;
  const int ant = threadIdx.x - lv * K;
  const int32_t vid = w.p.shard_lo + blockIdx.x * vpb + lv;
  const bool live = lv < vpb && vid < w.p.shard_hi;
  const int64_t step = w.ctl->step;
  const DevVehicles& v = w.v;

  long long act = 0, unf = 0;  // next step's count_active / unfinished (fused motion)
  if (live && ant == 0) {
    // the vehicle's words in one round of loads, ahead of any store (the
    // prologue runs beside the table staging and must not outlast it)
    uint8_t st = v.state[vid];
    const int64_t depart = v.depart[vid];
    int32_t at = v.at_node[vid];
    const int32_t origin = v.origin[vid];
    const int32_t on_edge = v.on_edge[vid];
    const int32_t dest = v.dest[vid];
    if (st == kPending && depart == step) {  // engine.cpp:177-180
      st = kAtNode;
      at = origin;
      v.state[vid] = kAtNode;
      v.at_node[vid] = origin;
    }
    int32_t start = -1;
    const bool deciding = st == kAtNode;
    if (deciding)
      start = at;
    else if (w.p.replan_all && (st == kQueued || st == kReleased))  // kReleased: queued at stage B
      start = at;
    else if (w.p.replan_all && st == kOnEdge)
      start = w.g.col[on_edge];
    if (start >= 0 && start == dest) {
      v.plan_n[vid] = 0;
      v.plan_step[vid] = step;
      v.plan_done[vid] = 0;
      start = -1;
    }
    start_s[lv] = start;
    deciding_s[lv] = deciding;
    if (w.p.sharded) v.dec_rec[vid] = -1;
    if (start < 0) veh_move(w, vid, act, unf);  // E2 now: stage B leaves this vehicle untouched
    best[lv] = ~0ull;
  }
  __syncthreads();
  long long steps = 0, cands = 0, degs = 0, routes = 0, decided = 0;
  int32_t start = -1, hops = 0;
  int64_t cost = 0;
  bool first_ok = false;
  int32_t* tour = nullptr;
  if (live) start = start_s[lv];
  if (live && start >= 0) {
    const int32_t dest = v.dest[vid];
    const int32_t max_hops = w.p.max_hops, hop_limit = w.p.hop_limit;
    const uint32_t k0 = (uint32_t)w.p.seed, k1 = (uint32_t)(w.p.seed >> 32);
    const int rng = w.p.rng;
    const int4* __restrict__ keys = reinterpret_cast<const int4*>(w.g.key);
    const double2* __restrict__ W2 = reinterpret_cast<const double2*>(w.weight);
    const longlong2* __restrict__ C2 = reinterpret_cast<const longlong2*>(w.ecost);
    if (w.p.scratch_mode) tour = v.scratch + ((size_t)vid * K + ant) * (size_t)w.p.plan_cap;
    // destination / current position
    int32_t cols = 0, rd = 0, cd = 0, rx = 0, cx = 0;
    const int64_t* __restrict__ trow = nullptr;
    if (DK == 1) {
      cols = w.d.cols;
      rd = dest / cols;
      cd = dest - rd * cols;
      rx = start / cols;
      cx = start - rx * cols;
    } else {
      const int32_t slot = w.d.slot_of ? w.d.slot_of[dest] : dest;
      trow = slot < 0 ? nullptr : w.d.table + (size_t)slot * w.d.n;
    }
    int32_t x = start;
    uint4 rnd = make_uint4(0, 0, 0, 0);
    while (x != dest && (hop_limit == 0 || hops < hop_limit)) {
      if (hops >= max_hops) {
        cost = kInf;
        break;
      }
      const int4 kk = keys[x];
      const double2 wa = W2[2 * x], wb = W2[2 * x + 1];
      const longlong2 ca = C2[2 * x], cb = C2[2 * x + 1];
      const int32_t kv[4] = {kk.x, kk.y, kk.z, kk.w};  // constant-indexed only (unrolled)
      uint32_t reach = 0, closer = 0;
      int deg = 0;
      if (DK == 1) {
        const int32_t dx = abs(rx - rd) + abs(cx - cd);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (kv[i] < 0) continue;
          ++deg;
          reach |= 1u << i;
          const int32_t dn = abs((kv[i] >> 16) - rd) + abs((kv[i] & 0xffff) - cd);
          if (dn < dx) closer |= 1u << i;
        }
      } else {
        if (trow) {
          const int64_t dx = __ldg(trow + x);
          int64_t dn[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) dn[i] = kv[i] >= 0 ? __ldg(trow + kv[i]) : kInf;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (kv[i] < 0) continue;
            ++deg;
            if (dn[i] == kInf) continue;
            reach |= 1u << i;
            if (dn[i] < dx) closer |= 1u << i;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) deg += kv[i] >= 0;
        }
      }
      degs += deg;
      const uint32_t cand = closer ? closer : reach;
      if (!cand) {
        cost = kInf;
        break;
      }
      if (hops == 0) first_ok = true;
      cands += __popc(cand);
      double u;
      if (rng == 1) {
        u = to_unit(draw(w.p.seed, 5, (uint64_t)(uint32_t)vid | ((uint64_t)(uint32_t)ant << 32),
                         (uint64_t)step | ((uint64_t)(uint32_t)hops << 40)));
      } else {
        if ((hops & 1) == 0)
          rnd = philox4(make_uint4((uint32_t)step, (uint32_t)vid, (uint32_t)ant, (uint32_t)hops >> 1), k0, k1);
        u = to_unit(philox_half(rnd, hops));
      }
      // sequential left-to-right roulette over the candidates (register-only)
      const double w0 = (cand & 1u) ? wa.x : 0.0, w1 = (cand & 2u) ? wa.y : 0.0;
      const double w2 = (cand & 4u) ? wb.x : 0.0, w3 = (cand & 8u) ? wb.y : 0.0;
      // adding an exact 0.0 for a non-candidate leaves every partial sum unchanged
      const double s0 = w0, s1 = __dadd_rn(s0, w1), s2 = __dadd_rn(s1, w2), total = __dadd_rn(s2, w3);
      const int c = __popc(cand);
      int pick = 31 - __clz(cand);  // default: last candidate
      if (total <= 0.0 || !isfinite(total)) {
        int p = (int)__dmul_rn(u, (double)c);
        p = p < c - 1 ? p : c - 1;
        uint32_t m = cand;
        if (p >= 1) m &= m - 1;
        if (p >= 2) m &= m - 1;
        if (p >= 3) m &= m - 1;
        pick = __ffs(m) - 1;
      } else {
        const double point = __dmul_rn(u, total);
        // first candidate i whose cumulative sum exceeds point
        if ((cand & 8u) && point < total) pick = 3;
        if ((cand & 4u) && point < s2) pick = 2;
        if ((cand & 2u) && point < s1) pick = 1;
        if ((cand & 1u) && point < s0) pick = 0;
      }
      const int64_t cpk = pick == 0 ? ca.x : pick == 1 ? ca.y : pick == 2 ? cb.x : cb.y;
      cost += cpk;
      if (tour) tour[hops] = 4 * x + pick;
      const int32_t nk = pick == 0 ? kk.x : pick == 1 ? kk.y : pick == 2 ? kk.z : kk.w;
      if (DK == 1) {
        rx = nk >> 16;
        cx = nk & 0xffff;
        x = rx * cols + cx;
      } else {
        x = nk;
      }
      ++hops;
      ++steps;
    }
    const uint64_t cc = cost >= (int64_t)kCostCap ? kCostCap : (uint64_t)cost;
    atomicMin(&best[lv], (cc << 10) | (uint64_t)ant);
  }
  __syncthreads();
  if (live && start >= 0 && ant == (int)(best[lv] & 1023u)) {
    const bool deciding = deciding_s[lv];
    if (!first_ok) {
      v.plan_n[vid] = 0;
      v.plan_step[vid] = step;
      v.plan_done[vid] = 0;
      if (deciding) {
        v.state[vid] = kRetired;
        if (w.p.sharded) v.dec_rec[vid] = -2;
      }
    } else {
      if (w.p.scratch_mode) {
        v.plan_ant[vid] = ant;
      } else {  // replay the winner with the generic walker to materialize its tour
        tour = v.plan + (size_t)vid * w.p.plan_cap;
        const Target<DK> t(w.d, v.dest[vid]);
        hops = ant_walk<DK, true>(w, t, vid, ant, start, step, tour).hops;
      }
      finish_colony(w, vid, start, tour, hops, deciding, step);
      routes = 1;
      decided = deciding;
    }
    veh_move(w, vid, act, unf);  // E2 right after this vehicle's stage B
  }
  const Sum5 t = block_sum5(Sum5{{steps, cands, degs, routes, decided, act, unf}}, red5);
  if (threadIdx.x == 0) flush_counters(w.ctl, t);
}

// ---------------------------------------------------------------------------
// B (colony) on general graphs, ant-queue form (scratch mode).  Long and
// uneven walks (C4: ~1000 hops, heavy tail) make any CTA-wide barrier wait
// for the slowest ant, so the step runs as three kernels:
//   k_colony_pro  one thread per vehicle: departure, walk start, fused
//                 motion of non-walkers, walking-vehicle list;
//   k_colony_q    persistent: every lane pulls (vehicle, ant) items from a
//                 global counter and advances its ant ONE HOP per loop trip,
//                 so a lane whose ant finished fetches the next item at once
//                 (no reconvergence on walk length); argmin via atomicMin on
//                 the packed (cost, ant) key;
//   k_colony_epi  one warp per vehicle: winner's tour from scratch, exact
//                 int64 deposits strided over the warp, take_edge, motion.
// Semantics identical to k_colony_csr / k_colony (routing.cpp:16-30, 88-113).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_colony_pro(DevWorld w) {
  if (skip_step(w.ctl)) return;
  __shared__ long long red5[7][32];
  const DevVehicles& v = w.v;
  const int64_t step = w.ctl->step;
  // walk order (destination-major, see gmaco_capi.cpp): the walking list, and
  // so the queue, visits vehicles bound for one target together
  const int32_t slot = w.p.shard_lo + blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t vid = (w.v.walk_order && slot < w.p.shard_hi) ? w.v.walk_order[slot] : slot;
  long long act = 0, unf = 0;
  bool walking = false;
  if (slot < w.p.shard_hi) {
    // the vehicle's words in one round of loads, ahead of any store (the
    // prologue runs beside the table staging and must not outlast it)
    uint8_t st = v.state[vid];
    const int64_t depart = v.depart[vid];
    int32_t at = v.at_node[vid];
    const int32_t origin = v.origin[vid];
    const int32_t on_edge = v.on_edge[vid];
    const int32_t dest = v.dest[vid];
    if (st == kPending && depart == step) {  // engine.cpp:177-180
      st = kAtNode;
      at = origin;
      v.state[vid] = kAtNode;
      v.at_node[vid] = origin;
    }
    int32_t start = -1;
    const bool deciding = st == kAtNode;
    if (deciding)
      start = at;
    else if (w.p.replan_all && (st == kQueued || st == kReleased))  // kReleased: queued at stage B
      start = at;
    else if (w.p.replan_all && st == kOnEdge)
      start = w.g.col[on_edge];
    if (start >= 0 && start == dest) {
      v.plan_n[vid] = 0;
      v.plan_step[vid] = step;
      v.plan_done[vid] = 0;
      start = -1;
    }
    if (w.p.sharded) v.dec_rec[vid] = -1;
    v.walk_start[vid] = start;

    if (start >= 0) {
      v.walk_dec[vid] = deciding;
      v.best_key[vid] = ~0ull;
      walking = true;
    } else {
      veh_move(w, vid, act, unf);
    }
  }
  // warp-aggregated append to the walking-vehicle list (order is immaterial:
  // every per-vehicle result is independent of processing order)
  const unsigned m = __ballot_sync(0xffffffffu, walking);
  if (m) {
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(&w.ctl->q_walkers, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (walking) v.walkers[base + __popc(m & ((1u << lane) - 1u))] = vid;
  }
  const Sum5 t = block_sum5(Sum5{{0, 0, 0, 0, 0, act, unf}}, red5);
  if (threadIdx.x == 0) flush_counters(w.ctl, t);
}

// Programmatic dependent launch (sm_90+): the dependent grid waits here for
// the full completion (and memory flush) of the grid it depends on.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

// 256-bit read-only global load (sm_100a LDG.256): two slot records per
// instruction, halving L1 wavefronts for lane-divergent rows.
__device__ __forceinline__ void ld256(const int4* p, int4& a, int4& b) {
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

__device__ __forceinline__ double rec_weight(const int4* r) {
  const int4 v = __ldg(r);
  return __hiloint2double(v.y, v.x);
}

// One hop of the queue walker is ONE dependent round trip: the row's filter
// bits plus the 16-B slot records {weight, head node, head row} of its first
// 8 slots (rows start 64-B aligned) are issued together; the pick is register-local, so the next row is known
// at once.  Rows wider than 8 slots (rare on road graphs) finish the roulette
// from global memory (L1-hot).
__global__ void __launch_bounds__(128, 6) k_colony_q(DevWorld w) {
  constexpr int W8 = 8;
  if (skip_step(w.ctl)) return;
  const DevVehicles& v = w.v;
  const int K = w.p.ants;
  const int64_t step = w.ctl->step;
  const unsigned long long total = w.ctl->q_walkers * (unsigned long long)K;
  const int32_t max_hops = w.p.max_hops, hop_limit = w.p.hop_limit;
  const int4* __restrict__ R = w.rec;
  const int32_t ell = w.g.ell;  // 8 (ELL-8 rows) or 0 (4-aligned CSR rows)
  const bool vec_tour = (w.p.plan_cap & 3) == 0;
  int4 tb = make_int4(0, 0, 0, 0);
  long long steps = 0, cands = 0, degs = 0;
  // current ant
  int32_t vid = 0, ant = 0, dmeta = 0, first = 0, span = 0, deg = 0, hops = 0;
  int64_t cost = 0;
  bool first_ok = false, active = false;
  const uint32_t* fb = nullptr;
  int32_t* tp = nullptr;
  uint4 rnd = make_uint4(0, 0, 0, 0);
  // Grouped form (K divides 32): K consecutive lanes own one vehicle's
  // colony and fetch the next vehicle together once all K ants finished, so a
  // vehicle's ants walk side by side (shared rows hit L1, same-node loads
  // coalesce).  Otherwise every lane fetches single ants.
  const bool grouped = K <= 32 && (32 % K) == 0;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = grouped ? (K == 32 ? 0xffffffffu : ((1u << K) - 1u) << (lane / K * K)) : (1u << lane);
  bool drained = false;  // this lane's (group's) queue fetch came back empty
  bool any_idle = true;  // warp-uniform: some lane finished its ant (a group may refetch)
  uint32_t trip = 0;     // warp-uniform loop trip count
  for (;;) {
    // full-warp votes: drained lanes stay in the loop (idle) until the whole
    // warp is drained, so no vote needs a partial mask; the fetch votes run
    // only after a lane of the warp went idle, and only on even trips (the
    // warp's ants share hop parity: one Philox block per pair for all)
    bool fetch = false;
    const bool even_trip = (trip++ & 1u) == 0;
    if (any_idle && even_trip) {
      fetch = !active && !drained;
      if (grouped) {
        const unsigned idle = __ballot_sync(0xffffffffu, !active);
        fetch = !drained && (idle & gmask) == gmask;
      }
      unsigned long long a = 0;
      if (fetch) {
        if (grouped) {  // the whole group is fetching: one atomic for K ants
          unsigned long long b = 0;
          if (lane == __ffs(gmask) - 1) b = atomicAdd(&w.ctl->q_next, (unsigned long long)K);
          a = __shfl_sync(gmask, b, __ffs(gmask) - 1) + (unsigned long long)(lane - (__ffs(gmask) - 1));
        } else {
          a = atomicAdd(&w.ctl->q_next, 1ull);
        }
      }
      const bool out = fetch && a >= total;  // group-uniform (total is a multiple of K)
      drained |= out;
      if (__all_sync(0xffffffffu, drained)) break;
      if (fetch && !out) {
        vid = v.walkers[a / K];
        ant = (int32_t)(a % K);
        const int32_t x0 = v.walk_start[vid];
        const int32_t dest = v.dest[vid];
        const int32_t tslot = w.d.slot_of ? w.d.slot_of[dest] : dest;
        fb = tslot < 0 ? nullptr : w.d.fbits + (size_t)tslot * w.d.fbw;
        const int2 r0 = __ldg(w.g.row + x0);
        first = r0.x;
        span = r0.y;
        deg = __ldg(w.g.deg + x0);
        // the destination's row descriptor: rows have unique starts, so a hop
        // reaches dest iff the picked record's descriptor equals it
        dmeta = (int32_t)(((uint32_t)__ldg(&w.g.row[dest].x) >> 2) << 5) | __ldg(w.g.deg + dest);
        tp = v.scratch + ((size_t)vid * K + ant) * (size_t)w.p.plan_cap;
        hops = 0;
        cost = 0;
        first_ok = false;
        active = true;
      }
    }
    any_idle = __any_sync(0xffffffffu, !active);
    if (!active) continue;  // idle lane waiting for its group (grouped form)
    bool fin = false;
    if (hops >= max_hops) {
      cost = kInf;
      fin = true;
    } else {
      // ---- the hop's single round trip ----
      uint32_t lo = 0, hi = 0;
      if (fb) {
        lo = __ldg(fb + (first >> 5));
        if ((first & 31) + span > 32) hi = __ldg(fb + (first >> 5) + 1);  // row crosses a word
      }
      int4 rc[W8];  // slot records: weight, int32 edge cost, head row (span is a multiple of 4)
#pragma unroll
      for (int i = 0; i < W8; i += 2) {
        if (i < span)
          ld256(R + first + i, rc[i], rc[i + 1]);
        else
          rc[i] = rc[i + 1] = make_int4(0, 0, -1, 0);
      }
      double wv[W8];
#pragma unroll
      for (int i = 0; i < W8; ++i) wv[i] = __hiloint2double(rc[i].y, rc[i].x);
      // closer bits only (see DevDist::fbits)
      const uint32_t cand = __funnelshift_r(lo, hi, first & 31) & ((1u << span) - 1u);
      degs += deg;
      if (!cand) {
        cost = kInf;
        fin = true;
      } else {
        if (hops == 0) first_ok = true;
        cands += __popc(cand);
        double u;
        if (w.p.rng == 1) {
          u = to_unit(draw(w.p.seed, 5, (uint64_t)(uint32_t)vid | ((uint64_t)(uint32_t)ant << 32),
                           (uint64_t)step | ((uint64_t)(uint32_t)hops << 40)));
        } else {
          if ((hops & 1) == 0)
            rnd = philox4_rk(make_uint4((uint32_t)step, (uint32_t)vid, (uint32_t)ant, (uint32_t)hops >> 1),
                             w.p.rk);
          u = to_unit(philox_half(rnd, hops));
        }
        // sequential left-to-right roulette over the candidates; the running
        // sums are kept: the cumulative pass of routing.cpp:104-110 adds the
        // same weights in the same order, so its values ARE these prefixes
        double total_w = 0.0;
        double pre[W8];
        int c = 0;
#pragma unroll
        for (int i = 0; i < W8; ++i) {
          if (cand & (1u << i)) {
            total_w = __dadd_rn(total_w, wv[i]);
            ++c;
          }
          pre[i] = total_w;
        }
        const uint32_t wide = cand >> W8;  // slots 8.. of a wide row (rare)
        for (uint32_t m = wide; m; m &= m - 1) {
          total_w = __dadd_rn(total_w, rec_weight(R + first + W8 + __ffs(m) - 1));
          ++c;
        }
        int pick = 31 - __clz(cand);
        if (total_w <= 0.0 || !isfinite(total_w)) {
          const int pp = min((int)__dmul_rn(u, (double)c), c - 1);
          uint32_t mm = cand;
          for (int j = 0; j < pp; ++j) mm &= mm - 1;
          pick = __ffs(mm) - 1;
        } else {
          const double point = __dmul_rn(u, total_w);
          // first candidate whose prefix exceeds the point (independent compares)
          uint32_t hit = 0;
#pragma unroll
          for (int i = 0; i < W8; ++i) hit |= (point < pre[i] ? 1u : 0u) << i;
          hit &= cand;
          const bool found = hit != 0;
          if (found) pick = __ffs(hit) - 1;
          double cum = pre[W8 - 1];
          for (uint32_t m = found ? 0u : wide; m; m &= m - 1) {
            const int i = W8 + __ffs(m) - 1;
            cum = __dadd_rn(cum, rec_weight(R + first + i));
            if (point < cum) {
              pick = i;
              break;
            }
          }
        }
        int32_t ec = 0, meta = 0;
        if (pick < W8) {
#pragma unroll
          for (int i = 0; i < W8; ++i)
            if (i == pick) {
              ec = rc[i].z;
              meta = rc[i].w;
            }
        } else {
          const int4 r = __ldg(R + first + pick);
          ec = r.z;
          meta = r.w;
        }
        const int32_t sl = first + pick;
        // int32 edge cost from the record; -1 marks a cost >= 2^31 (exact
        // value in the int64 table, rare)
        cost += ec >= 0 ? (int64_t)ec : w.ecost[sl];
        // tour: 4 hops per 16-B streaming store (evict-first: the tours are
        // read once, by the epilogue) when the scratch stride allows
        tb.x = (hops & 3) == 0 ? sl : tb.x;
        tb.y = (hops & 3) == 1 ? sl : tb.y;
        tb.z = (hops & 3) == 2 ? sl : tb.z;
        tb.w = (hops & 3) == 3 ? sl : tb.w;
        if (!vec_tour)
          __stcs(tp + hops, sl);
        else if ((hops & 3) == 3)
          __stcs(reinterpret_cast<int4*>(tp + hops - 3), tb);
        fin = meta == dmeta || (hop_limit != 0 && hops + 1 >= hop_limit);
        first = (int32_t)(((uint32_t)meta >> 5) << 2);
        deg = meta & 31;
        span = ell ? ell : (deg + 3) & ~3;
        ++hops;
        ++steps;
      }
    }
    if (fin) {
      if (vec_tour)  // flush the partial 4-hop tour buffer
        for (int j = hops & ~3; j < hops; ++j) tp[j] = (j & 3) == 0 ? tb.x : (j & 3) == 1 ? tb.y : tb.z;
      const uint64_t cc = cost >= (int64_t)kCostCap ? kCostCap : (uint64_t)cost;
      v.ant_hops[(size_t)vid * K + ant] = first_ok ? hops : -1;
      atomicMin(&v.best_key[vid], (cc << 10) | (uint64_t)ant);
      active = false;
    }
  }
  // per-warp counter flush (lanes leave the loop at different times)
  __syncwarp();
  for (int o = 16; o > 0; o >>= 1) {
    steps += __shfl_xor_sync(0xffffffffu, steps, o);
    cands += __shfl_xor_sync(0xffffffffu, cands, o);
    degs += __shfl_xor_sync(0xffffffffu, degs, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (steps) atomicAdd((unsigned long long*)&w.ctl->ant_steps, (unsigned long long)steps);
    if (cands) atomicAdd((unsigned long long*)&w.ctl->candidates, (unsigned long long)cands);
    if (degs) atomicAdd((unsigned long long*)&w.ctl->degree_sum, (unsigned long long)degs);
  }
}

// ---------------------------------------------------------------------------
// Ant-queue walker over per-target candidate rows (DevTT): the same queue,
// grouped fetch and argmin as k_colony_q, but a hop loads only its
// candidates' records (one LDG.256 for <= 2 candidates, no filter word) and
// the roulette runs over c <= 4 registers.  Tours hold record indices
// (k_colony_epi maps the winner's to slots).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 8) k_colony_qt(DevWorld w) {
  if (skip_step(w.ctl)) return;
  const DevVehicles& v = w.v;
  const int K = w.p.ants;
  const int64_t step = w.ctl->step;
  const unsigned long long total = w.ctl->q_walkers * (unsigned long long)K;
  const int32_t max_hops = w.p.max_hops, hop_limit = w.p.hop_limit, n = w.g.n;
  const bool vec_tour = (w.p.plan_cap & 3) == 0;
  uint32_t steps = 0, cands = 0, degs = 0;  // per-thread (widened at the flush)
  int32_t vid = 0, ant = 0, dmeta = 0, meta = 0, hops = 0, tbase = 0;
  int64_t cost = 0;
  bool active = false;
  const int4* tt = w.tt.rec;
  int32_t* tp = nullptr;
  int4 tb = make_int4(0, 0, 0, 0);
  uint4 rnd = make_uint4(0, 0, 0, 0);
  const bool grouped = K <= 32 && (32 % K) == 0;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = grouped ? (K == 32 ? 0xffffffffu : ((1u << K) - 1u) << (lane / K * K)) : (1u << lane);
  bool drained = false;
  bool any_idle = true;  // warp-uniform: some lane finished its ant (a group may refetch)
  uint32_t trip = 0;     // warp-uniform loop trip count
  for (;;) {
    // full-warp votes (drained lanes idle in the loop until the warp drains);
    // the fetch votes run only after a lane of the warp went idle, and only on
    // even trips: every ant then takes hop h on a trip of h's parity, so the
    // Philox block (one per hop pair) is computed by the whole warp together,
    // every other trip, instead of whenever either of its groups needs one
    bool fetch = false;
    const bool even_trip = (trip++ & 1u) == 0;
    if (any_idle && even_trip) {
      fetch = !active && !drained;
      if (grouped) {
        const unsigned idle = __ballot_sync(0xffffffffu, !active);
        fetch = !drained && (idle & gmask) == gmask;
      }
      unsigned long long a = 0;
      if (fetch) {
        if (grouped) {  // the whole group is fetching: one atomic for K ants
          unsigned long long b = 0;
          if (lane == __ffs(gmask) - 1) b = atomicAdd(&w.ctl->q_next, (unsigned long long)K);
          a = __shfl_sync(gmask, b, __ffs(gmask) - 1) + (unsigned long long)(lane - (__ffs(gmask) - 1));
        } else {
          a = atomicAdd(&w.ctl->q_next, 1ull);
        }
      }
      const bool out = fetch && a >= total;  // group-uniform (total is a multiple of K)
      drained |= out;
      if (__all_sync(0xffffffffu, drained)) break;
      if (fetch && !out) {
        vid = v.walkers[a / K];
        ant = (int32_t)(a % K);
        const int32_t x0 = v.walk_start[vid];
        const int32_t dest = v.dest[vid];
        const int32_t tslot = w.d.slot_of ? w.d.slot_of[dest] : dest;
        if (tslot < 0) {  // no table: the zero row (no candidate) fails the ant at once
          tbase = 0;
          meta = 0;
          dmeta = -1;
        } else {
          tbase = (int32_t)__ldg(w.tt.base + tslot);
          const uint32_t* mt = w.tt.meta + (size_t)tslot * n;
          meta = (int32_t)__ldg(mt + x0);
          dmeta = (int32_t)__ldg(mt + dest);  // metas identify rows: a hop reaches dest iff it picks dest's
        }
        tt = w.tt.rec + tbase;
        tp = v.scratch + ((size_t)vid * K + ant) * (size_t)w.p.plan_cap;
        hops = 0;
        cost = 0;
        active = true;
      }
    }
    any_idle = __any_sync(0xffffffffu, !active);
    if (!active) continue;  // idle lane waiting for its group (grouped form)
    bool fin = false;
    {  // (max_hops >= 1: an ant is failed on the hop that reaches max_hops, below)
      // ---- the hop's single round trip: the candidates' records ----
      const uint32_t off2 = ((uint32_t)meta >> 8) << 1;
      const int c = (meta >> 4) & 15;
      const int4* rp = tt + off2;
      int4 rc[4];
      ld256(rp, rc[0], rc[1]);
      if (c > 2)
        ld256(rp + 2, rc[2], rc[3]);
      else
        rc[2] = rc[3] = make_int4(0, 0, 0, 0);
      degs += meta & 15;
      if (c == 0) {
        cost = kInf;
        fin = true;
      } else {
        cands += c;
        double u;
        if (w.p.rng == 1) {
          u = to_unit(draw(w.p.seed, 5, (uint64_t)(uint32_t)vid | ((uint64_t)(uint32_t)ant << 32),
                           (uint64_t)step | ((uint64_t)(uint32_t)hops << 40)));
        } else {
          if ((hops & 1) == 0)
            rnd = philox4_rk(make_uint4((uint32_t)step, (uint32_t)vid, (uint32_t)ant, (uint32_t)hops >> 1),
                             w.p.rk);
          u = to_unit(philox_half(rnd, hops));
        }
        // sequential left-to-right roulette (routing.cpp:100-113) over the c
        // candidates; the kept prefixes are the cumulative pass's values
        double total_w = 0.0, pre[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < c) total_w = __dadd_rn(total_w, __hiloint2double(rc[i].y, rc[i].x));
          pre[i] = total_w;
        }
        for (int i = 4; i < c; ++i) total_w = __dadd_rn(total_w, rec_weight(rp + i));  // rare wide rows
        int pick = c - 1;
        if (total_w <= 0.0 || !isfinite(total_w)) {
          pick = min((int)__dmul_rn(u, (double)c), c - 1);
        } else {
          const double point = __dmul_rn(u, total_w);
          uint32_t hit = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) hit |= (i < c && point < pre[i] ? 1u : 0u) << i;
          if (hit) {
            pick = __ffs(hit) - 1;
          } else {
            double cum = pre[3];
            for (int i = 4; i < c; ++i) {
              cum = __dadd_rn(cum, rec_weight(rp + i));
              if (point < cum) {
                pick = i;
                break;
              }
            }
          }
        }
        int32_t ec = 0, nm = 0;
        if (pick < 4) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (i == pick) {
              ec = rc[i].z;
              nm = rc[i].w;
            }
        } else {
          const int4 r = __ldg(rp + pick);
          ec = r.z;
          nm = r.w;
        }
        const int32_t ri = tbase + (int32_t)off2 + pick;  // record index (k_colony_epi maps it to the slot)
        // int32 edge cost; -1 marks a cost >= 2^31 (exact value in the int64 table, rare)
        if (__builtin_expect(ec < 0, 0))
          cost += w.ecost[w.tt.sm[ri].x];
        else
          cost += ec;
        // tour: 4 hops per 16-B streaming store (evict-first: read once, by the epilogue)
        tb.x = (hops & 3) == 0 ? ri : tb.x;
        tb.y = (hops & 3) == 1 ? ri : tb.y;
        tb.z = (hops & 3) == 2 ? ri : tb.z;
        tb.w = (hops & 3) == 3 ? ri : tb.w;
        if (!vec_tour)
          __stcs(tp + hops, ri);
        else if ((hops & 3) == 3)
          __stcs(reinterpret_cast<int4*>(tp + hops - 3), tb);
        fin = nm == dmeta || (hop_limit != 0 && hops + 1 >= hop_limit);
        if (!fin && hops + 1 >= max_hops) {  // tour cap reached short of dest: the ant fails
          cost = kInf;
          fin = true;
        }
        meta = nm;
        ++hops;
        ++steps;
      }
    }
    if (fin) {
      if (vec_tour)  // flush the partial 4-hop tour buffer
        for (int j = hops & ~3; j < hops; ++j) tp[j] = (j & 3) == 0 ? tb.x : (j & 3) == 1 ? tb.y : tb.z;
      const uint64_t cc = cost >= (int64_t)kCostCap ? kCostCap : (uint64_t)cost;
      // (the first hop had candidates iff any hop was made: max_hops >= 1)
      v.ant_hops[(size_t)vid * K + ant] = hops > 0 ? hops : -1;
      atomicMin(&v.best_key[vid], (cc << 10) | (uint64_t)ant);
      active = false;
    }
  }
  __syncwarp();
  unsigned long long ws = steps, wc = cands, wd = degs;
  for (int o = 16; o > 0; o >>= 1) {
    ws += __shfl_xor_sync(0xffffffffu, ws, o);
    wc += __shfl_xor_sync(0xffffffffu, wc, o);
    wd += __shfl_xor_sync(0xffffffffu, wd, o);
  }
  if (lane == 0) {
    const unsigned long long steps = ws, cands = wc, degs = wd;
    if (steps) atomicAdd((unsigned long long*)&w.ctl->ant_steps, (unsigned long long)steps);
    if (cands) atomicAdd((unsigned long long*)&w.ctl->candidates, (unsigned long long)cands);
    if (degs) atomicAdd((unsigned long long*)&w.ctl->degree_sum, (unsigned long long)degs);
  }
}

__global__ void __launch_bounds__(256) k_colony_epi(DevWorld w) {
  griddep_launch_dependents();  // let the tail's CTAs launch early (they wait for our completion)
  if (skip_step(w.ctl)) return;
  if (blockIdx.x == gridDim.x - 1) {  // dedicated prefetch block
    if (w.p.prefetch) prefetch_tail_state(w);
    if (threadIdx.x == 0) {  // the queue walk is complete: re-arm the queue
      w.ctl->q_walkers = 0;
      w.ctl->q_next = 0;
    }
    return;
  }
  __shared__ long long red5[7][32];
  const DevVehicles& v = w.v;
  const int64_t step = w.ctl->step;
  const int lane = threadIdx.x & 31;
  // this rank's vehicles, in walk order when one is set (by-target shards)
  const int32_t slot = w.p.shard_lo + blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int32_t vid = (w.v.walk_order && slot < w.p.shard_hi) ? w.v.walk_order[slot] : slot;
  long long routes = 0, decided = 0, act = 0, unf = 0;
  const int32_t start = slot < w.p.shard_hi ? v.walk_start[vid] : -1;
  if (start >= 0) {
    const int K = w.p.ants;
    const bool deciding = v.walk_dec[vid];
    const int ant = (int)(v.best_key[vid] & 1023u);
    const int32_t hops = v.ant_hops[(size_t)vid * K + ant];
    if (hops < 0) {  // no candidate at the first hop
      if (lane == 0) {
        v.plan_n[vid] = 0;
        v.plan_step[vid] = step;
        v.plan_done[vid] = 0;
        if (deciding) {
          v.state[vid] = kRetired;
          if (w.p.sharded) v.dec_rec[vid] = -2;
        }
      }
    } else {
      int32_t* tour = v.scratch + ((size_t)vid * K + ant) * (size_t)w.p.plan_cap;
      long long len = 0;
      if (w.tt.sl) {  // per-target walker: record indices -> {slot, length} (one gather per hop)
        int i = lane;
        for (; i + 96 < hops; i += 128) {  // four gathers in flight per lane
          const int32_t r0 = tour[i], r1 = tour[i + 32], r2 = tour[i + 64], r3 = tour[i + 96];
          const int2 q0 = w.tt.sl[r0], q1 = w.tt.sl[r1], q2 = w.tt.sl[r2], q3 = w.tt.sl[r3];
          tour[i] = q0.x;
          tour[i + 32] = q1.x;
          tour[i + 64] = q2.x;
          tour[i + 96] = q3.x;
          len += (long long)q0.y + q1.y + q2.y + q3.y;
        }
        for (; i < hops; i += 32) {
          const int2 q = w.tt.sl[tour[i]];
          tour[i] = q.x;
          len += q.y;
        }
        __syncwarp();
      } else {
        if (w.tt.rec) {  // per-target walker: the tour holds record indices -> slots
          for (int i = lane; i < hops; i += 32) tour[i] = w.tt.sm[tour[i]].x;
          __syncwarp();
        }
        if (w.p.deposit == 1)
          for (int i = lane; i < hops; i += 32) len += w.g.len[tour[i]];
      }
      const bool done = hops > 0 && w.g.col[tour[hops - 1]] == v.dest[vid];
      if (done && w.p.deposit == 1) {  // finish_colony's deposit, strided over the warp
        for (int o = 16; o > 0; o >>= 1) len += __shfl_xor_sync(0xffffffffu, len, o);
        const double km = __ddiv_rn((double)len, 1e6);
        const int64_t amount = llround(__dmul_rn(__ddiv_rn(w.p.deposit_q, km), 1e6));
        int i = lane;
        for (; i + 96 < hops; i += 128) {  // four slot loads in flight before the fire-and-forget adds
          const int32_t s0 = tour[i], s1 = tour[i + 32], s2 = tour[i + 64], s3 = tour[i + 96];
          atomicAdd((unsigned long long*)&w.dep[s0], (unsigned long long)amount);
          atomicAdd((unsigned long long*)&w.dep[s1], (unsigned long long)amount);
          atomicAdd((unsigned long long*)&w.dep[s2], (unsigned long long)amount);
          atomicAdd((unsigned long long*)&w.dep[s3], (unsigned long long)amount);
        }
        for (; i < hops; i += 32) atomicAdd((unsigned long long*)&w.dep[tour[i]], (unsigned long long)amount);
      }
      if (lane == 0) {
        v.plan_ant[vid] = ant;
        v.plan_n[vid] = hops;
        v.plan_step[vid] = step;
        v.plan_done[vid] = done;
        if (deciding) take_edge(w, vid, tour[0], false, start);
        routes = 1;
        decided = deciding;
      }
    }
    if (lane == 0) veh_move(w, vid, act, unf);
  }
  const Sum5 t = block_sum5(Sum5{{0, 0, 0, routes, decided, act, unf}}, red5);
  if (threadIdx.x == 0) flush_counters(w.ctl, t);
}

// ---------------------------------------------------------------------------
// B (colony) on general graphs (CSR or ELL-8 rows, distance tables, progress
// filter on).  One thread per ant.  The candidate filter (routing.cpp:16-30)
// is read from precomputed {closer, reach} bitmaps of the destination's table
// row instead of gathering every neighbour's distance, and each slot carries
// its head node's row descriptor, so a hop is two dependent round trips:
// (filter bits + the row's weights, issued together), then (chosen slot's
// head, next row descriptor, edge cost).  The decision is register-only
// (sequential left-to-right roulette, routing.cpp:88-113).  Same semantics
// as k_colony.
// ---------------------------------------------------------------------------
template <int MAXD, bool kScratch>
__global__ void __launch_bounds__(256) k_colony_csr(DevWorld w) {
  if (skip_step(w.ctl)) return;
  if (blockIdx.x == gridDim.x - 1) {  // dedicated prefetch block
    if (w.p.prefetch) prefetch_tail_state(w);
    return;
  }
  constexpr int kMaxVpb = 256;
  __shared__ unsigned long long best[kMaxVpb];
  __shared__ int32_t start_s[kMaxVpb];
  __shared__ uint8_t deciding_s[kMaxVpb];
  __shared__ long long red5[7][32];
  const int K = w.p.ants;
  const int vpb = blockDim.x / K;
  const int lv = threadIdx.x / K;
  const int ant = threadIdx.x - lv * K;
  const int32_t vid = w.p.shard_lo + blockIdx.x * vpb + lv;
  const bool live = lv < vpb && vid < w.p.shard_hi;
  const int64_t step = w.ctl->step;
  const DevVehicles& v = w.v;
  long long act = 0, unf = 0;
  if (live && ant == 0) {
    // the vehicle's words in one round of loads, ahead of any store (the
    // prologue runs beside the table staging and must not outlast it)
    uint8_t st = v.state[vid];
    const int64_t depart = v.depart[vid];
    int32_t at = v.at_node[vid];
    const int32_t origin = v.origin[vid];
    const int32_t on_edge = v.on_edge[vid];
    const int32_t dest = v.dest[vid];
    if (st == kPending && depart == step) {  // engine.cpp:177-180
      st = kAtNode;
      at = origin;
      v.state[vid] = kAtNode;
      v.at_node[vid] = origin;
    }
    int32_t start = -1;
    const bool deciding = st == kAtNode;
    if (deciding)
      start = at;
    else if (w.p.replan_all && (st == kQueued || st == kReleased))  // kReleased: queued at stage B
      start = at;
    else if (w.p.replan_all && st == kOnEdge)
      start = w.g.col[on_edge];
    if (start >= 0 && start == dest) {
      v.plan_n[vid] = 0;
      v.plan_step[vid] = step;
      v.plan_done[vid] = 0;
      start = -1;
    }
    start_s[lv] = start;
    deciding_s[lv] = deciding;
    if (w.p.sharded) v.dec_rec[vid] = -1;
    if (start < 0) veh_move(w, vid, act, unf);
    best[lv] = ~0ull;
  }
  __syncthreads();
  long long steps = 0, cands = 0, degs = 0, routes = 0, decided = 0;
  int32_t start = -1;
  bool first_ok = false;
  int32_t hops = 0;
  if (live) start = start_s[lv];
  if (live && start >= 0) {
    const int32_t dest = v.dest[vid];
    const int32_t tslot = w.d.slot_of ? w.d.slot_of[dest] : dest;
    const int64_t* __restrict__ trow = tslot < 0 ? nullptr : w.d.table + (size_t)tslot * w.d.n;
    const int32_t max_hops = w.p.max_hops, hop_limit = w.p.hop_limit;
    int32_t* tp = kScratch ? v.scratch + ((size_t)vid * K + ant) * (size_t)w.p.plan_cap : nullptr;
    int64_t cost = 0;
    int32_t x = start;
    const uint32_t* __restrict__ fb = tslot < 0 ? nullptr : w.d.fbits + (size_t)tslot * w.d.fbw;
    const int2 r0 = __ldg(w.g.row + start);
    int32_t first = r0.x, span = r0.y, deg = __ldg(w.g.deg + start);
    uint4 rnd = make_uint4(0, 0, 0, 0);
    while (x != dest && (hop_limit == 0 || hops < hop_limit)) {
      if (hops >= max_hops) {
        cost = kInf;
        break;
      }
      // round trip 1: the row's filter bits and weights (independent loads)
      uint32_t cand = 0;  // closer bits only (see DevDist::fbits)
      if (fb) {
        const uint32_t lo = __ldg(fb + (first >> 5)), hi = __ldg(fb + (first >> 5) + 1);
        cand = __funnelshift_r(lo, hi, first & 31) & ((1u << span) - 1u);
      }
      double wv[MAXD];
#pragma unroll
      for (int i = 0; i < MAXD; ++i) wv[i] = i < span ? w.weight[first + i] : 0.0;
      degs += deg;
      if (!cand) {
        cost = kInf;
        break;
      }
      if (hops == 0) first_ok = true;
      cands += __popc(cand);
      double u;
      if (w.p.rng == 1) {
        u = to_unit(draw(w.p.seed, 5, (uint64_t)(uint32_t)vid | ((uint64_t)(uint32_t)ant << 32),
                         (uint64_t)step | ((uint64_t)(uint32_t)hops << 40)));
      } else {
        if ((hops & 1) == 0)
          rnd = philox4_rk(make_uint4((uint32_t)step, (uint32_t)vid, (uint32_t)ant, (uint32_t)hops >> 1), w.p.rk);
        u = to_unit(philox_half(rnd, hops));
      }
      // sequential left-to-right roulette over the candidates (registers only)
      double total = 0.0;
      int c = 0;
#pragma unroll
      for (int i = 0; i < MAXD; ++i)
        if (cand & (1u << i)) {
          total = __dadd_rn(total, wv[i]);
          ++c;
        }
      int pick = 31 - __clz(cand);  // default: last candidate
      if (total <= 0.0 || !isfinite(total)) {
        const int pp = min((int)__dmul_rn(u, (double)c), c - 1);
        uint32_t mm = cand;
        for (int j = 0; j < pp; ++j) mm &= mm - 1;
        pick = __ffs(mm) - 1;
      } else {
        const double point = __dmul_rn(u, total);
        double cum = 0.0;
        bool found = false;
#pragma unroll
        for (int i = 0; i < MAXD; ++i)
          if (!found && (cand & (1u << i))) {
            cum = __dadd_rn(cum, wv[i]);
            if (point < cum) {
              pick = i;
              found = true;
            }
          }
      }
      // round trip 2: the chosen slot's head node, its row descriptor, its cost
      const int32_t sl = first + pick;
      x = __ldg(w.g.col + sl);
      const int2 nr = __ldg(w.g.nrow + sl);
      cost += w.ecost[sl];
      if (kScratch) tp[hops] = sl;
      first = nr.x;
      span = nr.y & 0xff;
      deg = nr.y >> 8;
      ++hops;
      ++steps;
    }
    const uint64_t cc = cost >= (int64_t)kCostCap ? kCostCap : (uint64_t)cost;
    atomicMin(&best[lv], (cc << 10) | (uint64_t)ant);
  }
  __syncthreads();
  if (live && start >= 0 && ant == (int)(best[lv] & 1023u)) {
    const bool deciding = deciding_s[lv];
    if (!first_ok) {
      v.plan_n[vid] = 0;
      v.plan_step[vid] = step;
      v.plan_done[vid] = 0;
      if (deciding) {
        v.state[vid] = kRetired;
        if (w.p.sharded) v.dec_rec[vid] = -2;
      }
    } else {
      int32_t* tour;
      if (kScratch) {
        tour = v.scratch + ((size_t)vid * K + ant) * (size_t)w.p.plan_cap;
        v.plan_ant[vid] = ant;
      } else {  // replay the winner to materialize its tour
        tour = v.plan + (size_t)vid * w.p.plan_cap;
        const Target<0> t(w.d, v.dest[vid]);
        hops = ant_walk<0, true>(w, t, vid, ant, start, step, tour).hops;
      }
      finish_colony(w, vid, start, tour, hops, deciding, step);
      routes = 1;
      decided = deciding;
    }
    veh_move(w, vid, act, unf);
  }
  const Sum5 t = block_sum5(Sum5{{steps, cands, degs, routes, decided, act, unf}}, red5);
  if (threadIdx.x == 0) flush_counters(w.ctl, t);
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ size_t grid_staged_bytes_dev(const DevWorld& w) {
  return 16 * (size_t)w.g.M;  // the LatRec table (kSmem variant)
}
// B (colony) on a validated uniform lattice (GMACO_DIST_GRID, progress filter
// on).  The distance service is closed-form and the lattice is checked at
// create, so a node's candidate set needs no loads at all: the strictly
// closer neighbours are the one horizontal and the one vertical move toward
// the destination, and their ELL slots follow from the ascending-id row
// order [up, left, right, down].  A hop is then 1-2 weight loads, a 2-way
// sequential roulette and one tour-cost load — identical decisions to
// k_colony / k_colony_ell4 (same candidate order, same arithmetic).
// ---------------------------------------------------------------------------
// Tour materialization of the lattice walker:
//   kTourReplay  — the winner re-walks (counter RNG) into v.plan;
//   kTourScratch — every ant writes its slots to v.scratch, the plan is the
//                  winner's row;
//   kTourBits    — one bit per hop (vertical or horizontal move), 64 hops
//                  per word in a register, full words flushed to SMEM
//                  (bit_words per ant); the winner's tour is rebuilt
//                  arithmetically (prefix popcounts) into v.plan.  No
//                  per-hop global stores.
// degree_sum and two-candidate counters of a monotone lattice walk from its
// move bits (hop i: word i/64, bit 63-(i%64); 1 = vertical), equal to summing
// per hop: rows change only on vertical moves, so the hops standing on the
// start row are those before the first vertical move and the hops on the
// final row those after the last one (a hop counts the node it departs from,
// so the first vertical move still stands on the start row; rows strictly
// between are interior);
// columns likewise with horizontal moves.  A hop has two candidates while
// both vertical and horizontal distance remain: hop i <= the index of the
// RV-th vertical and of the RH-th horizontal move (n when not made).
__device__ __forceinline__ void walk_counters_from_bits(const unsigned long long* wb, int32_t n, int32_t RV,
                                                        int32_t RH, int32_t rx, int32_t cx, int32_t dr, int32_t dc,
                                                        int32_t rows, int32_t cols, int32_t& idegs,
                                                        int32_t& n_two) {
  if (n <= 0) return;
  int32_t nv = 0, fv = -1, lv = -1, fh = -1, lh = -1;
  const int32_t words = (n + 63) >> 6;
  for (int32_t j = 0; j < words; ++j) {
    const unsigned long long wv = wb[j];
    const int32_t valid = min(64, n - 64 * j);
    const unsigned long long mask = valid == 64 ? ~0ull : (~0ull << (64 - valid));
    const unsigned long long wh = ~wv & mask;
    nv += __popcll(wv);
    if (wv) {
      if (fv < 0) fv = 64 * j + __clzll(wv);
      lv = 64 * j + 63 - (__ffsll((long long)wv) - 1);
    }
    if (wh) {
      if (fh < 0) fh = 64 * j + __clzll(wh);
      lh = 64 * j + 63 - (__ffsll((long long)wh) - 1);
    }
  }
  const int32_t nh = n - nv;
  auto border_r = [&](int32_t r) { return (r == 0) + (r == rows - 1); };
  auto border_c = [&](int32_t c) { return (c == 0) + (c == cols - 1); };
  int32_t sub = 0;
  if (nv == 0) {
    sub += n * border_r(rx);
  } else {
    sub += (fv + 1) * border_r(rx) + (n - 1 - lv) * border_r(rx + dr * nv);  // hop fv departs from row rx
  }
  if (nh == 0) {
    sub += n * border_c(cx);
  } else {
    sub += (fh + 1) * border_c(cx) + (n - 1 - lh) * border_c(cx + dc * nh);
  }
  idegs += 4 * n - sub;
  const int32_t cv = RV == 0 ? 0 : (nv >= RV ? lv + 1 : n);  // nv == RV: the RV-th vertical move is the last
  const int32_t chh = RH == 0 ? 0 : (nh >= RH ? lh + 1 : n);
  n_two += min(cv, chh);
}

enum { kTourReplay = 0, kTourScratch = 1, kTourBits = 2 };

// kOneVeh: the CTA holds exactly one vehicle's colony (threads == K, K a
// multiple of 32), so its per-vehicle barrier is the literal id 1: ptxas then
// reserves 2 named barriers instead of 16, which would otherwise cap the SM
// at 4 resident CTAs.
// C, D, E1 of one signal (defined with the tail stages below)
template <bool kConcurrent = false>
__device__ __forceinline__ long long sig_cde1(const DevWorld& w, int32_t s);

template <bool kSmem, int kTour, bool kOneVeh = false>
__global__ void __launch_bounds__(256, 2) k_colony_grid(DevWorld w) {
  griddep_launch_dependents();  // let the tail's CTAs launch early (they wait for our completion)
  // Block layout: [kSigCtas signal CTAs (e1_in_walk)][prefetch CTA][walk CTAs].
  // The special CTAs come first so the block scheduler dispatches them at
  // once: placed last, they started only when the final wave of walk CTAs was
  // dispatched and held the kernel's end ~17 us past the last walk (C3).
  const int nsig = w.p.e1_in_walk ? kSigCtas : 0;
  const int K = w.p.ants;
  const int vpb = blockDim.x / K;
  const int lv = threadIdx.x / K;
  const int ant = threadIdx.x - lv * K;
  const int32_t slot = w.p.shard_lo + ((int)blockIdx.x - nsig - 1) * vpb + lv;  // walk slot; the vehicle via the balance order
  const bool live = (int)blockIdx.x > nsig && lv < vpb && slot < w.p.shard_hi;
  // the walk slot's vehicle is loaded in the same memory round trip as the
  // control block (its load does not depend on the step check below)
  const int32_t vid = (w.v.walk_order && live) ? w.v.walk_order[slot] : slot;
  // Stage this step's LatRec table in shared memory with one TMA bulk copy
  // (cp.async.bulk) completing on an mbarrier, issued first thing: it does
  // not wait for the step check's round trip, and the prologue below
  // overlaps it.  (The table is the previous tail's output, complete at
  // launch: this kernel is not a programmatic dependent.)
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ __align__(8) uint64_t stage_bar;
  const bool stages = kSmem && (int)blockIdx.x > nsig;
  if (stages && threadIdx.x == 0) {
    const uint32_t bR = 16u * (uint32_t)w.g.M;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&stage_bar);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(dyn_smem);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bR) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(w.lrec), "r"(bR), "r"(bar) : "memory");
  }
  if (skip_step(w.ctl)) {
    if (stages && threadIdx.x == 0) {  // the copy lands before the CTA's shared memory is released
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&stage_bar);
      asm volatile(
          "{\n .reg .pred p;\n WAITS_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAITS_%=;\n}" ::"r"(bar)
          : "memory");
    }
    return;
  }
  if ((int)blockIdx.x == nsig) {  // dedicated prefetch block: stages C..G's state into L2
    if (w.p.prefetch) prefetch_tail_state(w);
    if (threadIdx.x == 0) TRACE_FINE(11);  // prefetch CTA done
    return;
  }
  if (w.p.e1_in_walk) {  // stages C, D, E1, concurrent with B
    const int sb = (int)blockIdx.x;
    if (sb < kSigCtas) {
      __shared__ long long redq[32];
      long long qt = 0;
      for (int32_t s = sb * blockDim.x + threadIdx.x; s < w.p.S; s += kSigCtas * blockDim.x)
        qt += sig_cde1<true>(w, s);
      qt = block_sum(qt, redq);
      if (threadIdx.x == 0 && qt) atomicAdd((unsigned long long*)&w.ctl->qtotal, (unsigned long long)qt);
      if (threadIdx.x == 0) TRACE_FINE(15);  // signal CTA done
      return;
    }
  }
  if (threadIdx.x == 0) {
    trace_min(w.ctl, 0);
    TRACE_FINE(7);  // the last walk CTA's start
  }
  constexpr int kMaxVpb = 256;
  __shared__ unsigned long long best[kMaxVpb];
  __shared__ int32_t start_s[kMaxVpb];
  __shared__ int32_t done_s[kMaxVpb];
  __shared__ uint8_t deciding_s[kMaxVpb];
  __shared__ long long red5[7][32];
  // move-bit words [blockDim][bit_words] after the staged tables (kTourBits)
  const int64_t step = w.ctl->step;
  const DevVehicles& v = w.v;
  const LatRec* __restrict__ R = kSmem ? reinterpret_cast<const LatRec*>(dyn_smem) : w.lrec;
  const int nw = w.p.bit_words;
  unsigned long long* const bits_w =
      reinterpret_cast<unsigned long long*>(dyn_smem + (kSmem ? grid_staged_bytes_dev(w) : 0));
  long long act = 0, unf = 0;  // next step's count_active / unfinished (fused motion)
  // a vehicle that does not walk moves (E2) after the block barrier below,
  // beside the walks, from the words its prologue loaded
  bool move_later = false;
  uint8_t st = 0;
  int64_t depart = 0;
  int32_t on_edge = 0, dest = 0;
  if (live && ant == 0) {
    // the vehicle's words in one round of loads, ahead of any store (the
    // prologue runs beside the table staging and must not outlast it)
    st = v.state[vid];
    depart = v.depart[vid];
    int32_t at = v.at_node[vid];
    const int32_t origin = v.origin[vid];
    on_edge = v.on_edge[vid];
    dest = v.dest[vid];
    if (st == kPending && depart == step) {  // engine.cpp:177-180
      st = kAtNode;
      at = origin;
      v.state[vid] = kAtNode;
      v.at_node[vid] = origin;
    }
    int32_t start = -1;
    const bool deciding = st == kAtNode;
    if (deciding)
      start = at;
    else if (w.p.replan_all && (st == kQueued || st == kReleased))  // kReleased: queued at stage B
      start = at;
    else if (w.p.replan_all && st == kOnEdge)
      start = w.g.col[on_edge];
    if (start >= 0 && start == dest) {
      v.plan_n[vid] = 0;
      v.plan_step[vid] = step;
      v.plan_done[vid] = 0;
      start = -1;
    }
    start_s[lv] = start;
    deciding_s[lv] = deciding;
    if (w.p.sharded) v.dec_rec[vid] = -1;
    move_later = start < 0;  // E2 below: stage B leaves this vehicle untouched
    done_s[lv] = 0;
    best[lv] = ~0ull;
  }
  __syncthreads();
  if (threadIdx.x == 0) TRACE_FINE(10);  // vehicle prologue done
  if (move_later) veh_move_from(w, vid, step, st, depart, on_edge, dest, act, unf);
  if (kSmem) {  // TMA tables landed (phase 0 of the staging mbarrier)
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&stage_bar);
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(bar)
        : "memory");
  }
  if (threadIdx.x == 0) trace_max(w.ctl, 1);
  long long steps = 0, cands = 0, degs = 0, routes = 0, decided = 0;
  int32_t start = -1, hops = 0;
  int64_t cost = 0;
  int32_t* tour = nullptr;
  if (live) start = start_s[lv];
  if (live && start >= 0) {
    int64_t lsum = 0;  // the walk's congestion loads (tour cost = len * (hops + lsum))
    const int32_t dest = v.dest[vid];
    const int32_t cols = w.d.cols;
    const int32_t rd = dest / cols, cd = dest - rd * cols;
    const int32_t rx = start / cols, cx = start - rx * cols;
    // The walk is monotone: the signs of (rd - rx, cd - cx) never flip and
    // every hop removes one unit of Manhattan distance, so the hop count is
    // known up front (the generic loop's x != dest / hop_limit / max_hops
    // tests collapse to this count and a failure flag).
    const int dc = cd > cx ? 1 : -1, dr = rd > rx ? 1 : -1;
    int32_t rem_h = abs(cd - cx), rem_v = abs(rd - rx);
    int32_t n = rem_h + rem_v;
    if (w.p.hop_limit && n > w.p.hop_limit) n = w.p.hop_limit;
    const bool capped = n > w.p.max_hops;  // generic walker fails at hop max_hops
    if (capped) n = w.p.max_hops;
    int32_t* tp = kTour == kTourScratch ? v.scratch + ((size_t)vid * K + ant) * (size_t)w.p.plan_cap : nullptr;
    tour = tp;
    int32_t idegs = 0;
    const int32_t rows = w.d.rows;
    int32_t rr = rx, cq = cx;
    int32_t n_two = 0;  // hops with two candidates (candidates = n + n_two)
    unsigned long long mbits = 0;  // move_v per hop of the current 64-hop word
    int32_t hb = 0, wj = 0;        // hops in the current word, words flushed
    // Direction-slotted lattice rows: slot 4x+{0,1,2,3} = {up, left, right,
    // down} (holes at the border), i.e. ascending neighbour id.  With the
    // walk direction fixed, the candidate slots are per-walk constants: when
    // both moves remain, the first candidate is "up" if moving up, else the
    // horizontal move.
    const int off_h = dc > 0 ? 2 : 1, off_v = dr > 0 ? 3 : 0;
    const int step_h = dc, step_v = dr * cols;
    const bool v_first = dr < 0;
    const int quad = (dr > 0 ? 2 : 0) | (dc > 0 ? 1 : 0);
    int32_t x = start;
    // the walk's record index and its per-hop steps (lrec_index)
    int32_t ri = lrec_index(w, start, quad);
    const int32_t ri_h = w.lrec_stride ? dr * rows : step_h * 4, ri_v = w.lrec_stride ? dr * (rows + 1) : step_v * 4;
    // One hop as straight-line predicated code (no branches: the compiler can
    // interleave the next Philox block and the two hops of a pair).  The
    // roulette (routing.cpp:100-113) over the hop's <= 2 candidates is the
    // integer compare against the node's tabulated threshold (LatRec): the
    // first candidate (vertical when moving up) iff the draw's top 53 bits
    // are below it; a single candidate is taken without a draw.
    int32_t l32 = 0;  // loads of the current (<= 64-hop) segment, flushed into lsum
    auto hop = [&](uint64_t bits) -> unsigned {
      const bool two = (rem_h > 0) & (rem_v > 0);
      // the record in one 16-B load: {thr lo, thr hi, lv, lh}
      const uint4 r = reinterpret_cast<const uint4*>(R)[ri];
      const unsigned long long thr = ((unsigned long long)r.y << 32) | r.x;
      const bool first = (bits >> 11) < thr;
      const unsigned mv = two ? (unsigned)(first == v_first) : (unsigned)(rem_h == 0);
      l32 += (int32_t)(mv ? r.z : r.w);
      if (kTour == kTourScratch) *tp++ = 4 * x + (mv ? off_v : off_h);
      if (kTour != kTourBits) {  // move-bit walks derive both counters after the walk
        // out-degree of x on the validated full lattice (degree_sum counter)
        idegs += (rr > 0) + (rr < rows - 1) + (cq > 0) + (cq < cols - 1);
        n_two += two;
        rr += mv ? dr : 0;
        cq += mv ? 0 : dc;
      }
      if (kTour == kTourScratch) x += mv ? step_v : step_h;
      ri += mv ? ri_v : ri_h;
      rem_v -= mv;
      rem_h -= mv ^ 1u;
      return mv;
    };
    // move bits: 64 hops per word, first hop of a word at bit 63
    if (w.p.rng == 1) {
      for (int32_t h = 0; h < n; ++h) {
        const unsigned mv = hop(draw(w.p.seed, 5, (uint64_t)(uint32_t)vid | ((uint64_t)(uint32_t)ant << 32),
                                     (uint64_t)step | ((uint64_t)(uint32_t)h << 40)));
        if (kTour == kTourBits) {
          mbits = (mbits << 1) | mv;
          if (++hb == 64) {
            bits_w[threadIdx.x * nw + wj++] = mbits;
            hb = 0;
          }
        }
        if ((h & 63) == 63) {
          lsum += l32;
          l32 = 0;
        }
      }
    } else {
      // hop pair (2p, 2p+1) uses Philox block p; block p+1 is computed in the
      // same basic block, so its independent chain fills the hops' latency.
      // One inner loop per 64-hop word (32 pairs): the word's bits and loads
      // are flushed after it, not tested for every hop.
      uint4 cur = philox4_rk(make_uint4((uint32_t)step, (uint32_t)vid, (uint32_t)ant, 0u), w.p.rk);
      const int32_t pairs = n >> 1;
      for (int32_t p0 = 0; p0 < pairs; p0 += 32) {
        const int32_t pe = min(pairs, p0 + 32);
        unsigned long long mb = 0;
        for (int32_t p = p0; p < pe; ++p) {
          // next block's rounds split across the pair's two dependent hops
          uint4 nxt = make_uint4((uint32_t)step, (uint32_t)vid, (uint32_t)ant, (uint32_t)p + 1u);
          philox_rounds<0, 5>(nxt, w.p.rk);
          const unsigned m0 = hop(((uint64_t)cur.x << 32) | cur.y);
          philox_rounds<5, 10>(nxt, w.p.rk);
          const unsigned m1 = hop(((uint64_t)cur.z << 32) | cur.w);
          mb = (mb << 2) | (m0 << 1) | m1;
          cur = nxt;
        }
        lsum += l32;
        l32 = 0;
        if (kTour == kTourBits) {
          if (pe - p0 == 32) {
            bits_w[threadIdx.x * nw + wj++] = mb;
          } else {
            mbits = mb;
            hb = 2 * (pe - p0);
          }
        }
      }
      if (n & 1) {
        const unsigned mv = hop(((uint64_t)cur.x << 32) | cur.y);
        mbits = (mbits << 1) | mv;
        ++hb;
      }
    }
    lsum += l32;
    if (kTour == kTourBits) {
      if (hb) bits_w[threadIdx.x * nw + wj] = mbits << (64 - hb);  // left-aligned
      walk_counters_from_bits(bits_w + threadIdx.x * nw, n, abs(rd - rx), abs(cd - cx), rx, cx, dr, dc, rows, cols,
                              idegs, n_two);
    }
    if (ant == 0) TRACE_FINE(8);  // walk loop done (all ants of a vehicle walk n hops)
    cost = (int64_t)w.d.grid_len * ((int64_t)n + lsum);  // = the sum of the hops' len * (1 + load)
    if (capped) cost = kInf;
    hops = n;
    steps = n;
    degs = idegs;
    cands = n + n_two;
    const uint64_t cc = cost >= (int64_t)kCostCap ? kCostCap : (uint64_t)cost;
    atomicMin(&best[lv], (cc << 10) | (uint64_t)ant);
    if (kTour == kTourBits && (K & 31) == 0) {
      if (ant == 32) TRACE_FINE(12);  // the vehicle's second warp's walk done
      if (kOneVeh)
        asm volatile("bar.sync 1, %0;" ::"r"(K) : "memory");
      else
        asm volatile("bar.sync %0, %1;" ::"r"(1 + lv), "r"(K) : "memory");
      if (ant == 0) TRACE_FINE(13);  // past the vehicle's barrier
      if (ant < 32) {
        const int winner = (int)(best[lv] & 1023u);
        const unsigned long long* wb = bits_w + (size_t)(lv * K + winner) * nw;
        const bool reached = hops == abs(rd - rx) + abs(cd - cx);
        const bool dep = reached && w.p.deposit == 1;
        const int64_t amount = dep ? w.dep_amount[hops] : 0;
        int32_t* plan = v.plan + (size_t)vid * w.p.plan_cap;
        int32_t before = 0;  // vertical moves in the words before word j
        for (int32_t j = 0; 64 * j < hops; ++j) {
          const unsigned long long word = wb[j];
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int32_t r = ant + 32 * t, i = 64 * j + r;
            if (i < hops) {
              const int32_t nv = before + (r ? __popcll(word >> (64 - r)) : 0);  // vertical moves before hop i
              const int32_t y = start + step_v * nv + step_h * (i - nv);
              const unsigned mv = (unsigned)(word >> (63 - r)) & 1u;
              const int32_t sl = 4 * y + (mv ? off_v : off_h);
              plan[i] = sl;
              if (dep) atomicAdd((unsigned long long*)&w.dep[sl], (unsigned long long)amount);
            }
          }
          before += __popcll(word);
        }
        if (ant == 0) {
          TRACE_FINE(14);  // tour rebuilt, deposits issued
          const bool deciding = deciding_s[lv];
          v.plan_n[vid] = hops;
          v.plan_step[vid] = step;
          v.plan_done[vid] = reached && hops > 0;
          if (deciding) {
            const unsigned mv0 = (unsigned)(wb[0] >> 63) & 1u;
            take_edge(w, vid, 4 * start + (mv0 ? off_v : off_h), false, start);
          }
          veh_move(w, vid, act, unf);  // E2 right after this vehicle's stage B
          routes = 1;
          decided = deciding;
          TRACE_FINE(9);  // vehicle epilogue done
        }
      }
    } else {
    // best tour by (cost, ant); the vehicle's LAST ant to finish runs the
    // epilogue, so no block barrier couples different vehicles' walk lengths
    __threadfence_block();
    if (atomicAdd(&done_s[lv], 1) == K - 1) {
      __threadfence_block();
      const int winner = (int)(best[lv] & 1023u);
      const bool deciding = deciding_s[lv];
      // Lattice epilogue (finish_colony without re-reading the tour): every
      // ant walks the same hop count, edges have one length, and a walk
      // reaches the destination iff it was not cut short.
      const bool reached = hops == abs(rd - rx) + abs(cd - cx);
      const bool dep = reached && w.p.deposit == 1;
      const int64_t amount = dep ? w.dep_amount[hops] : 0;  // deposit_amount(hops * edge length)
      int32_t first = -1;
      if (kTour == kTourBits) {  // rebuild the winner's tour from its move bits
        tour = v.plan + (size_t)vid * w.p.plan_cap;
        const unsigned long long* wb = bits_w + (size_t)(lv * K + winner) * nw;
        int32_t y = start;
        for (int32_t i = 0; i < hops; ++i) {
          const unsigned mv = (unsigned)(wb[i >> 6] >> (63 - (i & 63))) & 1u;
          const int32_t sl = 4 * y + (mv ? off_v : off_h);
          tour[i] = sl;
          if (dep) atomicAdd((unsigned long long*)&w.dep[sl], (unsigned long long)amount);
          y += mv ? step_v : step_h;
          if (i == 0) first = sl;
        }
      } else {
        if (kTour == kTourScratch) {
          v.plan_ant[vid] = winner;
          tour = v.scratch + ((size_t)vid * K + winner) * (size_t)w.p.plan_cap;
        } else {  // replay the winner to materialize its tour
          tour = v.plan + (size_t)vid * w.p.plan_cap;
          const Target<1> t(w.d, v.dest[vid]);
          hops = ant_walk<1, true>(w, t, vid, winner, start, step, tour).hops;
        }
        if (dep) {
          int32_t i = 0;
          for (; i + 4 <= hops; i += 4) {  // independent loads, pipelined
            const int32_t a0 = tour[i], a1 = tour[i + 1], a2 = tour[i + 2], a3 = tour[i + 3];
            atomicAdd((unsigned long long*)&w.dep[a0], (unsigned long long)amount);
            atomicAdd((unsigned long long*)&w.dep[a1], (unsigned long long)amount);
            atomicAdd((unsigned long long*)&w.dep[a2], (unsigned long long)amount);
            atomicAdd((unsigned long long*)&w.dep[a3], (unsigned long long)amount);
          }
          for (; i < hops; ++i) atomicAdd((unsigned long long*)&w.dep[tour[i]], (unsigned long long)amount);
        }
        if (hops > 0) first = tour[0];
      }
      v.plan_n[vid] = hops;
      v.plan_step[vid] = step;
      v.plan_done[vid] = reached && hops > 0;
      if (deciding) take_edge(w, vid, first, false, start);
      routes = 1;
      decided = deciding;
      veh_move(w, vid, act, unf);  // E2 right after this vehicle's stage B
    }
    }
  }
  const Sum5 t = block_sum5(Sum5{{steps, cands, degs, routes, decided, act, unf}}, red5);
  if (threadIdx.x == 0) {
    flush_counters(w.ctl, t);
    trace_max(w.ctl, 2);
  }
}

// ---------------------------------------------------------------------------
// C, D, E1: one thread per signal (engine.cpp:219-252, signals.cpp:62-135)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int order_position(const DevParams& p, int ph) {
  for (int i = 0; i < kPhases; ++i)
    if (p.order[i] == ph) return i;
  return 0;
}
__device__ __forceinline__ int next_in_order(const DevParams& p, int cursor) {
  return p.order[(order_position(p, cursor) + 1) % kPhases];
}

__device__ int select_phase(const DevParams& p, const int32_t* q, const double* hw, int cursor) {
  if (p.controller == 0) return next_in_order(p, cursor);
  if (p.controller == 1) {
    const int pos = order_position(p, cursor);
    for (int i = 0; i < kPhases; ++i) {
      const int ph = p.order[(pos + i) % kPhases];
      if (q[ph] > 0) return ph;
    }
    return next_in_order(p, cursor);
  }
  int best = -1;
  for (int ph = 0; ph < kPhases; ++ph)
    if (q[ph] > p.th_max && (best == -1 || q[ph] > q[best])) best = ph;
  if (best != -1) return best;
  for (int ph = 0; ph < kPhases; ++ph)
    if (hw[ph] > p.t_max && (best == -1 || hw[ph] > hw[best])) best = ph;
  if (best != -1) return best;
  for (int ph = 0; ph < kPhases; ++ph)
    if (q[ph] > 0 && (best == -1 || q[ph] > q[best])) best = ph;
  if (best != -1) return best;
  return next_in_order(p, cursor);
}

// C, D, E1 for one signal: density sample (returned), green assignment at an
// epoch (engine.cpp:223-239, assign_green signals.cpp:111-117), FIFO
// discharge (signals.cpp:119-135, engine.cpp:241-252).
template <bool kConcurrent>
__device__ __forceinline__ long long sig_cde1(const DevWorld& w, int32_t s) {
  const DevSignals& S = w.s;
  int32_t q[kPhases];
  double hw[kPhases];
  long long qt = 0;
#pragma unroll
  for (int ph = 0; ph < kPhases; ++ph) {
    q[ph] = S.qlen[s * kPhases + ph];
    hw[ph] = S.head_wait[s * kPhases + ph];
    qt += q[ph];
  }
  int green = S.green[s];
  if (!(S.el_s[s] < w.p.green_duration_s)) {
    green = select_phase(w.p, q, hw, S.cursor[s]);
    S.green[s] = green;
    S.cursor[s] = green;
    S.el_s[s] = 0.0;
    S.el_steps[s] = 0;
    S.rem[s * kPhases + green] = 0.0;
  }
  const int k = s * kPhases + green;
  double rem = S.rem[k];
  rem = __dadd_rn(rem, __dmul_rn(__dmul_rn(w.p.saturation_flow, (double)S.lanes[s]), w.p.dt_s));
  int budget = (int)floor(rem);
  rem = __dsub_rn(rem, (double)budget);
  S.rem[k] = rem;
  int32_t len = 0;  // q[green] without dynamic register indexing
#pragma unroll
  for (int ph = 0; ph < kPhases; ++ph)
    if (ph == green) len = q[ph];
  if (budget > 0 && len > 0) {
    int32_t head = S.qhead[k];
    const int64_t step = w.ctl->step;
    const int32_t node = S.node[s];
    while (budget > 0 && len > 0) {
      const int32_t vid = head;
      head = w.v.qnext[vid];
      --len;
      --budget;
      w.v.queued[vid] += step - w.v.joined[vid] + 1;
      if (kConcurrent) {  // stage B may be reading this vehicle: Queued until the tail
        w.v.state[vid] = kReleased;
        w.v.rel[atomicAdd(&w.ctl->nrel, 1)] = vid;
      } else {
        w.v.state[vid] = kAtNode;
      }
      w.v.at_node[vid] = node;
      w.v.queued_phase[vid] = -1;
    }
    S.qhead[k] = len ? head : -1;
    if (!len) S.qtail[k] = -1;
    S.qlen[k] = len;
  }
  if (len == 0) S.head_wait[k] = 0.0;
  if (kConcurrent) {  // F+G's queue loads without waiting for E3 (DevSignals::qlen_e1)
    const int64_t Q = (int64_t)w.p.S * kPhases;
    int32_t* nxt = S.arr_cnt + ((w.ctl->step + 1) & 1) * Q;  // next step's arrival counters
#pragma unroll
    for (int ph = 0; ph < kPhases; ++ph) {
      S.qlen_e1[s * kPhases + ph] = ph == green ? len : q[ph];
      nxt[s * kPhases + ph] = 0;
    }
  }
  return qt;
}

// E2 for one vehicle: motion (engine.cpp:254-295), arrival deposit (ACO,
// engine.cpp:341-346; per-edge sum-then-clamp equals sequential clamping for
// amounts >= 0), queue arrival push, occupancy histogram (engine.cpp:316-322)
// and the next step's count_active / unfinished contributions.
// E3 for one signal: enqueue commit in ascending vid (engine.cpp:297-301) and
// timers (engine.cpp:303-314).  This step's arrivals all share joined =
// step+1, larger than every queued key, so FIFO order = old queue then the
// arrivals by ascending vid.
__device__ __forceinline__ void sig_e3(const DevWorld& w, int32_t s) {
  const DevSignals& S = w.s;
  const int64_t now = w.ctl->step + 1;
  const int k0 = s * kPhases;
  // one round of independent loads for all 8 queues, then the (rare)
  // arrival chains, then one round of head lookups for head_wait
  int32_t chain[kPhases], len[kPhases], head[kPhases];
  const int64_t e = S.el_steps[s] + 1;  // loaded with the queue words, ahead of the stores
#pragma unroll
  for (int ph = 0; ph < kPhases; ++ph) {
    chain[ph] = S.arr_head[k0 + ph];
    len[ph] = S.qlen[k0 + ph];
    head[ph] = S.qhead[k0 + ph];
  }
#pragma unroll
  for (int ph = 0; ph < kPhases; ++ph) {
    if (chain[ph] < 0) continue;
    const int k = k0 + ph;
    S.arr_head[k] = -1;
    int32_t tail = S.qtail[k];
    int32_t hd = head[ph], n = len[ph];
    int32_t last = -1;
    for (;;) {  // append chain members in ascending vid (selection; chains are short)
      int32_t best = INT32_MAX;
      for (int32_t c = chain[ph]; c >= 0; c = w.v.arr_next[c])
        if (c > last && c < best) best = c;
      if (best == INT32_MAX) break;
      w.v.qnext[best] = -1;
      if (tail < 0)
        hd = best;
      else
        w.v.qnext[tail] = best;
      tail = best;
      ++n;
      last = best;
    }
    S.qhead[k] = hd;
    S.qtail[k] = tail;
    S.qlen[k] = n;
    head[ph] = hd;
    len[ph] = n;
  }
  int64_t joined[kPhases];
#pragma unroll
  for (int ph = 0; ph < kPhases; ++ph) joined[ph] = len[ph] ? w.v.joined[head[ph]] : 0;
#pragma unroll
  for (int ph = 0; ph < kPhases; ++ph)
    S.head_wait[k0 + ph] = len[ph] == 0 ? 0.0 : __dmul_rn((double)(now - joined[ph]), w.p.dt_s);
  S.el_steps[s] = e;
  S.el_s[s] = __dmul_rn((double)e, w.p.dt_s);
}

// E3 for one queue k = s * kPhases + ph: the per-queue body of sig_e3, for
// the one-pass colony tail (one thread per queue, so a signal's queues with
// arrivals no longer chain their round trips one after another).  A kept
// head's joined step is loaded beside the arrival chain: appends do not move
// a non-empty queue's head, and a queue that was empty gets an arrival head,
// whose joined step is now (veh_move_core).
__device__ __forceinline__ void queue_e3(const DevWorld& w, int32_t k) {
  const DevSignals& S = w.s;
  const int64_t now = w.ctl->step + 1;
  const int32_t s = k / kPhases;
  const bool first = k == s * kPhases;  // the signal's phase-0 queue also advances its clock
  const int32_t chain = S.arr_head[k];
  const int32_t len0 = S.qlen[k], head0 = S.qhead[k], tail0 = S.qtail[k];
  const int64_t e = first ? S.el_steps[s] + 1 : 0;
  const int64_t jh = len0 ? w.v.joined[head0] : now;
  int32_t n = len0;
  if (chain >= 0) {
    S.arr_head[k] = -1;
    int32_t hd = head0, tail = tail0, last = -1;
    for (;;) {  // append chain members in ascending vid (selection; chains are short)
      int32_t best = INT32_MAX;
      for (int32_t c = chain; c >= 0; c = w.v.arr_next[c])
        if (c > last && c < best) best = c;
      if (best == INT32_MAX) break;
      w.v.qnext[best] = -1;
      if (tail < 0)
        hd = best;
      else
        w.v.qnext[tail] = best;
      tail = best;
      ++n;
      last = best;
    }
    S.qhead[k] = hd;
    S.qtail[k] = tail;
    S.qlen[k] = n;
  }
  S.head_wait[k] = n == 0 ? 0.0 : __dmul_rn((double)(now - jh), w.p.dt_s);
  if (first) {
    S.el_steps[s] = e;
    S.el_s[s] = __dmul_rn((double)e, w.p.dt_s);
  }
}

// F (scoped MACO) for one decision node: replay the step's decisions at that
// node in ascending vid (apply_maco_update_scoped, pheromone.cpp:48-59).
__device__ __forceinline__ void node_scoped(const DevWorld& w, int32_t u) {
  const int32_t chain = w.dec_head[u];
  if (chain < 0) return;
  w.dec_head[u] = -1;
  const int2 ri = w.g.row[u];
  int32_t last = -1;
  for (;;) {
    int32_t best = INT32_MAX;
    for (int32_t c = chain; c >= 0; c = w.v.dec_next[c])
      if (c > last && c < best) best = c;
    if (best == INT32_MAX) break;
    last = best;
    const int32_t chosen = w.v.on_edge[best];
    for (int i = 0; i < ri.y; ++i) {
      const int32_t s = ri.x + i;
      if (w.g.col[s] < 0) continue;  // ELL hole
      const int64_t t = w.tau[s];
      w.tau[s] = s == chosen ? min(w.p.tau_hi, t + w.p.inc) : max(w.p.tau_lo, t - w.p.dec);
    }
  }
}

// The lattice walker's roulette threshold (LatRec): the least k in
// [0, 2^53] with !(fl(fl(k * 2^-53) * (wa + wb)) < wa), i.e. the walk takes
// the first candidate iff its draw's top 53 bits are below it.  The product
// is monotone in k, so the boundary is exact from a quotient estimate
// confirmed by probes, or else by bisection.  A total
// that is not positive and finite picks uniformly (routing.cpp:100-104):
// the second candidate iff floor(2u) >= 1, i.e. k >= 2^52.
__device__ __forceinline__ unsigned long long lattice_threshold(double wa, double wb) {
  const double total = __dadd_rn(wa, wb);
  if (!((total > 0.0) & (total <= 1.7976931348623157e308))) return 1ull << 52;
  const unsigned long long kEnd = 1ull << 53;
  // a lattice border's hole (weight 0) on either side: never first (u *
  // total >= 0 >= wa), or always first for a normal wa (fl(u * wa) < wa for
  // every u <= 1 - 2^-53; not so for a subnormal one); the zero dividend
  // would otherwise take the division's slow path
  if (wa <= 0.0) return 0;
  if (wb == 0.0 && wa >= 2.2250738585072014e-308) return kEnd;
  auto first_d = [&](double kd) { return __dmul_rn(__dmul_rn(kd, 0x1.0p-53), total) < wa; };  // kd integral
  auto first = [&](unsigned long long k) { return first_d((double)k); };
  // estimate k0 = floor(wa / total * 2^53); the boundary is within k0 - 1
  // .. k0 + 1 up to rounding noise, settled by four independent probes
  const double r = __dmul_rn(__ddiv_rn(wa, total), 0x1.0p53);
  const double kf = !(r > 0.0) ? 0.0 : (r >= 0x1.0p53 ? 0x1.0p53 : floor(r));
  const unsigned long long k = (unsigned long long)kf;
  const bool pmm = k < 2 || first_d(__dadd_rn(kf, -2.0));
  const bool pm = k == 0 || first_d(__dadd_rn(kf, -1.0));
  const bool p0 = k < kEnd && first_d(kf);
  const bool p1 = k + 1 < kEnd && first_d(__dadd_rn(kf, 1.0));
  if (pm && !p0) return k;
  if (p0 && !p1) return k + 1;
  if (k > 0 && pmm && !pm) return k - 1;
  // otherwise bisect a window around k0 when it brackets the boundary, else
  // all of [0, 2^53] (subnormal products round coarsely, so the boundary can
  // lie far from the quotient): at most 53 probes
  unsigned long long lo = k > 4 ? k - 4 : 0, hi = k + 5 < kEnd ? k + 5 : kEnd;
  if (!((lo == 0 || first(lo - 1)) && (hi == kEnd || !first(hi)))) {
    lo = 0;
    hi = kEnd;
  }
  while (lo < hi) {
    const unsigned long long mid = lo + ((hi - lo) >> 1);
    if (first(mid))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// The four LatRec of node s / 4 from its four slots' next-step weights and
// loads: lane s & 3 of the quad writes quadrant q = s & 3 (rows grow: q & 2,
// cols grow: q & 1; slots {up, left, right, down}).  Every lane of the quad
// calls it together (s & 3 == lane & 3: callers stride by whole warps).
__device__ __forceinline__ void lattice_quad(const DevWorld& w, int64_t s, double wt, int32_t load) {
  const unsigned lane = threadIdx.x & 31u, base = lane & ~3u;
  const unsigned qm = 0xFu << base;
  const unsigned q = (unsigned)s & 3u;
  const bool down = q & 2u, right = q & 1u;
  const int ov = (int)base + (down ? 3 : 0), oh = (int)base + (right ? 2 : 1);
  const double wv = __shfl_sync(qm, wt, ov), wh = __shfl_sync(qm, wt, oh);
  const int32_t lv = __shfl_sync(qm, load, ov), lh = __shfl_sync(qm, load, oh);
  // moving up, "up" is the first slot (arguments selected first: one inlined
  // threshold chain per lane, not two divergent ones)
  const double wa = down ? wh : wv, wb = down ? wv : wh;
  const unsigned long long thr = lattice_threshold(wa, wb);
  reinterpret_cast<uint4*>(w.lrec)[lrec_index(w, (int32_t)(s >> 2), (int)q)] =
      make_uint4((uint32_t)thr, (uint32_t)(thr >> 32), (uint32_t)lv, (uint32_t)lh);
}

// F + G for one slot: MACO fold (fold_maco_edge, parallel.cpp:77-92) or exact
// deposit sum-then-clamp, evaporation (pheromone.cpp:61-67), colony
// congestion term, occupancy hand-off, next step's weight / tour cost
// (routing.cpp:90-94).  Returns the slot's occupancy (for the running max).
// A slot's words that no step changes (the graph's) and the step parity,
// loaded by a programmatic-dependent tail before it waits for the walk:
// the slot's F+G is then one memory round trip after the wait, not two.
struct SlotStatic {
  double eta;
  int64_t len;
  int32_t bind;
  int32_t par;
  __device__ __forceinline__ void load(const DevWorld& w, int32_t s) {
    const int alg = w.p.algorithm;
    const bool aco = alg == 1 || alg == 4;
    eta = aco ? w.g.eta_beta[s] : 0.0;
    len = aco ? w.g.len[s] : 0;
    bind = (alg == 4 && w.p.congestion) ? w.g.bind[s] : -1;
    par = (int32_t)(w.ctl->step & 1);  // (finalize of the previous step wrote it)
  }
};

__device__ __forceinline__ int32_t slot_fg(const DevWorld& w, int32_t s, double* wt_out = nullptr,
                                           int32_t* load_out = nullptr, const SlotStatic* pre = nullptr) {
  const DevParams& p = w.p;
  const int alg = p.algorithm;
  const bool aco = alg == 1 || alg == 4;
  // every load that does not depend on another is issued here, ahead of the
  // stores below (the compiler may not move a load past a possibly aliasing
  // store): the slot's chain is two memory round trips instead of four
  int64_t t = w.tau[s];
  const int32_t occ = w.occ_new[s];
  const int64_t d = aco ? w.dep[s] : 0;
  const double eta = pre ? pre->eta : (aco ? w.g.eta_beta[s] : 0.0);
  const int64_t len = pre ? pre->len : (aco ? w.g.len[s] : 0);
  const int32_t b = pre ? pre->bind : ((alg == 4 && p.congestion) ? w.g.bind[s] : -1);
  const int64_t par = (b >= 0 && p.e1_in_walk) ? (pre ? pre->par : (w.ctl->step & 1)) : 0;
  int32_t q = 0;  // the queue's length after E3
  if (b >= 0)
    q = p.e1_in_walk ? w.s.qlen_e1[b] + w.s.arr_cnt[par * (int64_t)p.S * kPhases + b] : w.s.qlen[b];
  if ((alg == 2 || alg == 3) && !p.siblings_only) {
    const int64_t D = w.ctl->dcount;
    const int32_t chain = w.dec_head[s];
    int64_t done = 0;
    if (chain >= 0) {
      w.dec_head[s] = -1;
      int32_t last = -1;
      for (;;) {
        int32_t best = INT32_MAX;
        for (int32_t c = chain; c >= 0; c = w.v.dec_next[c])
          if (c > last && c < best) best = c;
        if (best == INT32_MAX) break;
        last = best;
        const int64_t pos = w.v.pos[best];
        const int64_t gap = pos - done;
        if (gap > 0) t = max(p.tau_lo, t - gap * p.dec);
        t = min(p.tau_hi, t + p.inc);
        done = pos + 1;
      }
    }
    const int64_t gap = D - done;
    if (gap > 0) t = max(p.tau_lo, t - gap * p.dec);
  } else if (aco) {
    if (d) {
      t = min(p.tau_hi, t + d);
      w.dep[s] = 0;
    }
  }
  const int64_t scaled = (int64_t)floor(__dmul_rn(p.one_minus_rho, (double)t));
  t = max(p.tau_lo, scaled);
  if (alg == 4 && p.cong_evap && occ > 0) t = max(p.tau_lo, t - p.dec * (int64_t)occ);
  w.tau[s] = t;
  w.occ_cur[s] = occ;
  w.occ_new[s] = 0;
  if (aco) {
    double wt = __dmul_rn(tau_alpha(w, t), eta);
    int64_t cost = len;
    if (alg == 4 && p.congestion) {
      const int32_t load = occ + q;
      wt = __dmul_rn(wt, __ddiv_rn(1.0, __dadd_rn(1.0, (double)load)));
      cost = cost + cost * (int64_t)load;
      if (load_out) *load_out = load;
    }
    if (wt_out) *wt_out = wt;
    w.weight[s] = wt;
    if (w.rec) {  // slot record {weight, int32 cost (-1: >= 2^31, see ecost)}
      *reinterpret_cast<double*>(w.rec + s) = wt;
      w.rec[s].z = cost <= INT32_MAX ? (int32_t)cost : -1;
    }
    w.ecost[s] = cost;
    if (w.ecost32) w.ecost32[s] = (int32_t)cost;  // bound checked on the host
  }
  return occ;
}

// Step finalize (engine.cpp:399 ++step, finished() engine.cpp:146-152).
__device__ __forceinline__ void finalize_step(const DevWorld& w) {
  DevCtl* c = w.ctl;
  c->blocks_done = 0;
  if (c->max_occ_acc > c->max_occ) c->max_occ = c->max_occ_acc;
  c->qsamples += w.p.S;
  c->n_t = c->n_next;
  c->n_next = 0;
  c->nrel = 0;
  c->dcount = 0;
  const int64_t step = c->step + 1;
  c->step = step;
  c->done = (step >= w.p.max_steps || c->unfinished == 0) ? 1 : 0;
  c->unfinished = 0;
}

// The snapshot gather by one block (the step's finalizing block; small
// worlds only, see gmaco_step_snapshot): every requested field of the
// post-step vehicle state into mapped pinned memory.
__device__ __forceinline__ void block_snapshot(const PackDesc* d) {
  const int n = d->n;
  for (int k = 0; k < n; ++k) {
    const PackField f = d->f[k];
    const bool vec = ((reinterpret_cast<uintptr_t>(f.src) | reinterpret_cast<uintptr_t>(f.dst)) & 15) == 0;
    size_t done = 0;
    if (vec) {
      const size_t n16 = f.bytes / 16;
      for (size_t i = threadIdx.x; i < n16; i += blockDim.x)
        reinterpret_cast<uint4*>(f.dst)[i] = reinterpret_cast<const uint4*>(f.src)[i];
      done = n16 * 16;
    }
    for (size_t i = done + threadIdx.x; i < f.bytes; i += blockDim.x)
      static_cast<char*>(f.dst)[i] = static_cast<const char*>(f.src)[i];
  }
}

__device__ __forceinline__ int32_t block_max(int32_t m, int32_t* smax) {
  __syncwarp();  // reconverge first (see block_sum)
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 1; i < (int)((blockDim.x + 31) >> 5); ++i) m = max(m, smax[i]);
  return m;  // valid in thread 0
}

// ---------------------------------------------------------------------------
// multi-kernel tail (large worlds): one thread per entity per stage
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_signals(DevWorld w) {
  if (skip_step(w.ctl)) return;
  __shared__ long long red[32];
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  long long qt = s < w.p.S ? sig_cde1(w, s) : 0;
  qt = block_sum(qt, red);
  if (threadIdx.x == 0 && qt) atomicAdd((unsigned long long*)&w.ctl->qtotal, (unsigned long long)qt);
}

__global__ void __launch_bounds__(256) k_move(DevWorld w) {
  if (skip_step(w.ctl)) return;
  __shared__ long long red[32];
  const int32_t vid = blockIdx.x * blockDim.x + threadIdx.x;
  long long active = 0, unfinished = 0;
  if (vid < w.p.V) veh_move(w, vid, active, unfinished);
  active = block_sum(active, red);
  unfinished = block_sum(unfinished, red);
  if (threadIdx.x == 0) {
    if (active) atomicAdd((unsigned long long*)&w.ctl->n_next, (unsigned long long)active);
    if (unfinished) atomicAdd((unsigned long long*)&w.ctl->unfinished, (unsigned long long)unfinished);
  }
}

__global__ void __launch_bounds__(256) k_e3(DevWorld w) {
  if (skip_step(w.ctl)) return;
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < w.p.S) sig_e3(w, s);
}

__global__ void __launch_bounds__(256) k_scoped(DevWorld w) {
  if (skip_step(w.ctl)) return;
  const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < w.g.n) node_scoped(w, u);
}

// LatRec table from the current weights and tour costs (create,
// gmaco_set_pheromone): cost = len * (1 + load) on the uniform lattice.
__global__ void __launch_bounds__(256) k_lattice_rec(DevWorld w) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= w.g.M) return;  // (whole quads: M = 4 n)
  const bool live = w.g.slot_edge[s] >= 0;
  const double wt = live ? w.weight[s] : 0.0;
  const int32_t load = live ? (int32_t)(w.ecost[s] / w.d.grid_len - 1) : 0;
  lattice_quad(w, s, wt, load);
}

cudaError_t launch_lattice_rec(const DevWorld& w, cudaStream_t st) {
  if (!w.lrec) return cudaSuccess;
  k_lattice_rec<<<(unsigned)((w.g.M + 255) / 256), 256, 0, st>>>(w);
  return cudaGetLastError();
}

// gmaco_debug_roulette_threshold: lattice_threshold over a batch.
__global__ void k_threshold_batch(int32_t count, const double* wa, const double* wb, unsigned long long* out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = lattice_threshold(wa[i], wb[i]);
}

cudaError_t launch_threshold_batch(int32_t count, const double* wa, const double* wb, uint64_t* out,
                                   cudaStream_t st) {
  if (count > 0)
    k_threshold_batch<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(count, wa, wb,
                                                                        reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

// The last block to finish finalizes the step.
__global__ void __launch_bounds__(256) k_edges(DevWorld w) {
  if (skip_step(w.ctl)) {
    if (blockIdx.x == 0 && w.snap) block_snapshot(w.snap);  // a no-op step still snapshots the state
    return;
  }
  __shared__ int32_t smax[32];
  __shared__ bool is_last;
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  double wt = 0.0;
  int32_t load = 0;
  const int32_t occ = (s < w.g.M && w.g.slot_edge[s] >= 0) ? slot_fg(w, s, &wt, &load) : 0;
  if (w.lrec && s < w.g.M) lattice_quad(w, s, wt, load);  // (M = 4 n on a lattice: whole quads)
  const int32_t m = block_max(occ, smax);
  if (threadIdx.x == 0) {
    if (m > 0) atomicMax(&w.ctl->max_occ_acc, m);
    is_last = atom_add_acq_rel(&w.ctl->blocks_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) finalize_step(w);  // the kernel's completion publishes it
  if (is_last && w.snap) block_snapshot(w.snap);  // (is_last is block-uniform)
}

// ---------------------------------------------------------------------------
// Sharded runs: apply the other ranks' decisions (after the exchange) to the
// replicated vehicle state — activation (engine.cpp:177-180), then the
// decision's bookkeeping (engine.cpp:202-216) or retirement.
// ---------------------------------------------------------------------------
// A vehicle another rank plans (its decision record arrives with the exchange).
__device__ __forceinline__ bool is_remote(const DevWorld& w, int32_t vid) {
  return w.v.owner ? w.v.owner[vid] != w.p.rank : !(vid >= w.p.shard_lo && vid < w.p.shard_hi);
}

__global__ void __launch_bounds__(256) k_apply_remote(DevWorld w) {
  if (skip_step(w.ctl)) return;
  __shared__ long long red[32];
  const int32_t vid = blockIdx.x * blockDim.x + threadIdx.x;
  long long applied = 0;
  if (vid < w.p.V && is_remote(w, vid)) {
    const DevVehicles& v = w.v;
    const int64_t step = w.ctl->step;
    if (v.state[vid] == kPending && v.depart[vid] == step) {
      v.state[vid] = kAtNode;
      v.at_node[vid] = v.origin[vid];
    }
    const int32_t rec = v.dec_rec[vid];
    if (rec >= 0) {
      take_edge(w, vid, rec & ~GMACO_REC_DEVIATED, (rec & GMACO_REC_DEVIATED) != 0, v.at_node[vid]);
      applied = 1;
    } else if (rec == -2) {
      v.state[vid] = kRetired;
    }
    // network-wide MACO fold: remote decisions take their positions too
    if (w.p.need_positions) v.dflag[vid] = rec >= 0 ? 1 : 0;
  }
  // the fold's decision total D (fold_maco_edge's total_decisions) is global
  applied = block_sum(applied, red);
  if (threadIdx.x == 0 && applied) atomicAdd((unsigned long long*)&w.ctl->dcount, (unsigned long long)applied);
}

// colony mode: a remote vehicle's decision, then its motion (E2) and the
// next step's counts, exactly as the walk kernel does for its own shard
__device__ __forceinline__ void apply_remote_one(const DevWorld& w, int32_t vid, long long& act, long long& unf) {
  const DevVehicles& v = w.v;
  const int64_t step = w.ctl->step;
  if (v.state[vid] == kPending && v.depart[vid] == step) {
    v.state[vid] = kAtNode;
    v.at_node[vid] = v.origin[vid];
  }
  const int32_t rec = v.dec_rec[vid];
  if (rec >= 0)
    take_edge(w, vid, rec, false, v.at_node[vid]);
  else if (rec == -2)
    v.state[vid] = kRetired;
  veh_move(w, vid, act, unf);
}

__global__ void __launch_bounds__(256) k_apply_remote_move(DevWorld w) {
  if (skip_step(w.ctl)) return;
  __shared__ long long red[32];
  const int32_t vid = blockIdx.x * blockDim.x + threadIdx.x;
  long long act = 0, unf = 0;
  if (vid < w.p.V && is_remote(w, vid)) apply_remote_one(w, vid, act, unf);
  act = block_sum(act, red);
  unf = block_sum(unf, red);
  if (threadIdx.x == 0) {
    if (act) atomicAdd((unsigned long long*)&w.ctl->n_next, (unsigned long long)act);
    if (unf) atomicAdd((unsigned long long*)&w.ctl->unfinished, (unsigned long long)unf);
  }
}

// ---------------------------------------------------------------------------
// cooperative tail (one launch for stages C..G): E1 (signals) and E2 (motion)
// touch disjoint vehicles — queued vs on-edge — and disjoint queue fields
// (E1: qhead/qnext/qlen, E2: arrival stacks), so they run concurrently;
// grid.sync() orders E3 after E2 and F+G after E3.  Launched with the
// cooperative attribute, which guarantees co-residency of the grid.
// ---------------------------------------------------------------------------
// MACO fold positions of the vehicles [c0, c1) of this block: the exclusive
// prefix of dflag, offset by the decisions of the blocks before it (bsum,
// published before the last grid barrier).
__device__ __forceinline__ void chunk_positions(const DevWorld& w, int64_t c0, int64_t c1, long long* red) {
  long long off = 0;
  for (int64_t b = threadIdx.x; b < blockIdx.x; b += blockDim.x) off += w.v.bsum[b];
  off = block_sum(off, red);
  __shared__ long long s_off;
  __shared__ int32_t wsum[kTailCoop / 32];
  if (threadIdx.x == 0) s_off = off;
  __syncthreads();
  long long base = s_off;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t t0 = c0; t0 < c1; t0 += blockDim.x) {
    const int64_t i = t0 + threadIdx.x;
    const int32_t f = i < c1 ? w.v.dflag[i] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f != 0);
    if (lane == 0) wsum[wid] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kTailCoop / 32; ++k) {
      before += k < wid ? wsum[k] : 0;
      total += wsum[k];
    }
    if (i < c1) w.v.pos[i] = (int32_t)(base + before + __popc(bal & ((1u << lane) - 1u)));
    base += total;
    __syncthreads();
  }
}

// The step's end: the running occupancy maximum, and either the last block to
// finish finalizes the step (no grid barrier) or the caller does after one.
template <bool kLastBlockFinalize>
__device__ __forceinline__ void step_end(const DevWorld& w, int32_t m, int32_t* smax) {
  m = block_max(m, smax);
  if (kLastBlockFinalize) {
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
      if (m > 0) atomicMax(&w.ctl->max_occ_acc, m);
      trace_max(w.ctl, 6);
      // release the block's stores, acquire every block's (see k_tail_coop)
      is_last = atom_add_acq_rel(&w.ctl->blocks_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (is_last && threadIdx.x == 0) finalize_step(w);  // the kernel's completion publishes it
    if (is_last && w.snap) block_snapshot(w.snap);  // (is_last is block-uniform)
  } else if (threadIdx.x == 0 && m > 0) {
    atomicMax(&w.ctl->max_occ_acc, m);
  }
}

// One reference-algorithm step on the cooperative grid (stages B..G):
// optional stage B, C, D, E1 || E2, E3 (+ the MACO fold positions), F+G.
// kLastBlockFinalize: the last block to finish finalizes the step; else the
// caller finalizes after a grid barrier (the persistent multi-step kernel).
template <int kDecideDK, bool kLastBlockFinalize>
__device__ __forceinline__ void ref_step(const DevWorld& w, cg::grid_group& grid) {
  __shared__ long long red[32];
  __shared__ int32_t smax[32];
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const DevParams& p = w.p;
  if (kDecideDK >= 0 && !p.siblings_only) {
    // Stage B fused (unsharded): TWO grid barriers per step.  Block b decides
    // the contiguous vehicle chunk [c0, c1) and publishes its decision count;
    // after barrier 1 it runs C, D, E1 || E2 and writes its chunk's fold
    // positions; after barrier 2, E3 and F+G run in one pass -- for the
    // reference algorithms F+G reads nothing E3 writes (no congestion term)
    // and E3 nothing F+G writes.
    const int64_t chunk = (p.V + gridDim.x - 1) / gridDim.x;
    const int64_t c0 = min((int64_t)p.V, (int64_t)blockIdx.x * chunk), c1 = min((int64_t)p.V, c0 + chunk);
    {
      const int64_t step = w.ctl->step;
      long long decided = 0, cands = 0, degs = 0;
      for (int64_t vid = c0 + threadIdx.x; vid < c1; vid += blockDim.x)
        decide_vehicle<kDecideDK < 0 ? 0 : kDecideDK>(w, (int32_t)vid, step, decided, cands, degs);
      flush_decide_counters(w, decided, cands, degs, red);  // (its block reductions order the dflag writes)
      if (p.need_positions) {
        long long cnt = 0;
        for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) cnt += w.v.dflag[i];
        cnt = block_sum(cnt, red);
        if (threadIdx.x == 0) w.v.bsum[blockIdx.x] = (int32_t)cnt;
      }
    }
    grid.sync();
    long long qt = 0, active = 0, unfinished = 0;
    for (int64_t i = gtid; i < (int64_t)p.S + p.V; i += gstride) {
      if (i < p.S)
        qt += sig_cde1(w, (int32_t)i);
      else
        veh_move(w, (int32_t)(i - p.S), active, unfinished);
    }
    qt = block_sum(qt, red);
    if (threadIdx.x == 0 && qt) atomicAdd((unsigned long long*)&w.ctl->qtotal, (unsigned long long)qt);
    active = block_sum(active, red);
    if (threadIdx.x == 0 && active) atomicAdd((unsigned long long*)&w.ctl->n_next, (unsigned long long)active);
    unfinished = block_sum(unfinished, red);
    if (threadIdx.x == 0 && unfinished)
      atomicAdd((unsigned long long*)&w.ctl->unfinished, (unsigned long long)unfinished);
    if (p.need_positions) chunk_positions(w, c0, c1, red);
    grid.sync();
    int32_t m = 0;
    const int64_t M = w.g.M;
    for (int64_t i = gtid; i < M + p.S; i += gstride) {
      if (i < M) {
        if (w.g.slot_edge[i] >= 0) m = max(m, slot_fg(w, (int32_t)i));
      } else {
        sig_e3(w, (int32_t)(i - M));
      }
    }
    step_end<kLastBlockFinalize>(w, m, smax);
    return;
  }
  if (kDecideDK >= 0) {
    // reference algorithms, unsharded: stage B in the same launch (one kernel
    // per step); decisions never see each other (engine.cpp:197-198)
    const int64_t step = w.ctl->step;
    long long decided = 0, cands = 0, degs = 0;
    for (int64_t vid = gtid; vid < p.V; vid += gstride)
      decide_vehicle<kDecideDK < 0 ? 0 : kDecideDK>(w, (int32_t)vid, step, decided, cands, degs);
    flush_decide_counters(w, decided, cands, degs, red);
    grid.sync();
  }
  // Network-wide MACO fold (fold_maco_edge, parallel.cpp:77-92): every
  // decision's position in ascending-vid order is the exclusive prefix of
  // dflag (set by stage B).  Block b scans the contiguous vehicle chunk
  // [c0, c1): its count is published before the first grid barrier, its
  // positions written before the second (F+G reads them after the third) --
  // no extra barrier and no library scan.
  const bool pos_scan = p.need_positions;
  const int64_t chunk = (p.V + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = min((int64_t)p.V, (int64_t)blockIdx.x * chunk), c1 = min((int64_t)p.V, c0 + chunk);
  if (pos_scan) {
    long long cnt = 0;
    for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) cnt += w.v.dflag[i];
    cnt = block_sum(cnt, red);
    if (threadIdx.x == 0) w.v.bsum[blockIdx.x] = (int32_t)cnt;
  }
  // C, D, E1 (signals) || E2 (vehicles)
  long long qt = 0, active = 0, unfinished = 0;
  for (int64_t i = gtid; i < (int64_t)p.S + p.V; i += gstride) {
    if (i < p.S)
      qt += sig_cde1(w, (int32_t)i);
    else
      veh_move(w, (int32_t)(i - p.S), active, unfinished);
  }
  qt = block_sum(qt, red);
  if (threadIdx.x == 0 && qt) atomicAdd((unsigned long long*)&w.ctl->qtotal, (unsigned long long)qt);
  active = block_sum(active, red);
  if (threadIdx.x == 0 && active) atomicAdd((unsigned long long*)&w.ctl->n_next, (unsigned long long)active);
  unfinished = block_sum(unfinished, red);
  if (threadIdx.x == 0 && unfinished)
    atomicAdd((unsigned long long*)&w.ctl->unfinished, (unsigned long long)unfinished);
  if (threadIdx.x == 0) trace_max(w.ctl, 4);
  grid.sync();
  // E3
  for (int64_t s = gtid; s < p.S; s += gstride) sig_e3(w, (int32_t)s);
  if (pos_scan) chunk_positions(w, c0, c1, red);  // (block-uniform loop bounds)
  if (p.siblings_only && (p.algorithm == 2 || p.algorithm == 3)) {
    grid.sync();
    for (int64_t u = gtid; u < w.g.n; u += gstride) node_scoped(w, (int32_t)u);
  }
  if (threadIdx.x == 0) trace_max(w.ctl, 5);
  grid.sync();
  // F + G
  int32_t m = 0;
  for (int64_t s = gtid; s < w.g.M; s += gstride)
    if (w.g.slot_edge[s] >= 0) m = max(m, slot_fg(w, (int32_t)s));
  step_end<kLastBlockFinalize>(w, m, smax);
}

// Persistent run of up to `nsteps` reference-algorithm steps in ONE
// cooperative launch (gmaco_run / multi-step gmaco_step, unsharded): a step
// is stage B .. G on the whole grid, then two grid barriers around the
// finalize; the loop ends at finished() (engine.cpp:146-152) or after nsteps.
template <int DK>
__global__ void __launch_bounds__(kTailCoop) k_run_coop(DevWorld w, int64_t nsteps) {
  cg::grid_group grid = cg::this_grid();
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  (void)gtid;
  for (int64_t k = 0; k < nsteps && !skip_step(w.ctl); ++k) {  // ctl is read after a barrier: grid-uniform
    ref_step<DK, true>(w, grid);  // the step's last block finalizes it
    grid.sync();
  }
}

template <bool kFusedMotion, int kDecideDK>
__global__ void __launch_bounds__(kTailCoop) k_tail_coop(DevWorld w) {
  // the first slot's static words, loaded while the walk still runs (PDL
  // early launch); nothing the walk writes is read before the wait below
  SlotStatic pre{};
  const int64_t gtid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool have_pre = kFusedMotion && w.p.e1_in_walk && gtid0 < w.g.M;
  if (have_pre) pre.load(w, (int32_t)gtid0);
  griddep_wait();  // PDL: the preceding kernel (walk) completed and its writes are visible
  if (skip_step(w.ctl)) {  // grid-uniform: ctl changes only in the finalize below
    if (blockIdx.x == 0 && w.snap) block_snapshot(w.snap);  // a no-op step still snapshots the state
    return;
  }
  cg::grid_group grid = cg::this_grid();
  if (threadIdx.x == 0) trace_min(w.ctl, 3);
  __shared__ long long red[32];
  __shared__ int32_t smax[32];
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const DevParams& p = w.p;
  if (kFusedMotion) {
    if (p.sharded) {
      // other ranks' vehicles (their decision records arrived with the
      // exchange): activation, decision bookkeeping, then motion — what the
      // walk kernel did for this rank's shard (k_apply_remote_move, folded
      // in to save a kernel boundary per step)
      long long act = 0, unf = 0;
      for (int64_t vid = gtid; vid < p.V; vid += gstride)
        if (is_remote(w, (int32_t)vid)) apply_remote_one(w, (int32_t)vid, act, unf);
      act = block_sum(act, red);
      if (threadIdx.x == 0 && act) atomicAdd((unsigned long long*)&w.ctl->n_next, (unsigned long long)act);
      unf = block_sum(unf, red);
      if (threadIdx.x == 0 && unf) atomicAdd((unsigned long long*)&w.ctl->unfinished, (unsigned long long)unf);
      grid.sync();
    }
    // colony mode: E2 already ran inside the walk kernel, so one pass per
    // signal does C, D, E1 (pops the FIFO head) and E3 (appends this step's
    // arrivals after it) — the reference order for each queue.  With
    // e1_in_walk, C, D, E1 ran beside the walk: E3 only, and the vehicles E1
    // released become AtNode
    long long qt = 0;
    if (p.e1_in_walk) {
      // E3 || F+G in one pass (F+G's queue loads come from qlen_e1 + the
      // arrival counters), the kReleased fix-up, and the last block to finish
      // finalizes the step: no grid-wide barrier at all
      // one index space (slots, then queues: E3 per queue) so that no thread
      // chains a queue's E3 after a slot's F+G when the grid covers both
      const int64_t M = w.g.M;
      int32_t m = 0;
      for (int64_t i = gtid; i < M + (int64_t)p.S * kPhases; i += gstride) {
        if (i < M) {
          double wt = 0.0;
          int32_t load = 0;
          m = max(m, slot_fg(w, (int32_t)i, &wt, &load, (have_pre && i == gtid) ? &pre : nullptr));
          if (w.lrec) lattice_quad(w, i, wt, load);  // (M = 4 n: whole quads take this branch)
        } else {
          queue_e3(w, (int32_t)(i - M));
        }
      }
#ifdef GMACO_TRACE_FINE
      __syncwarp();  // one stamp per warp: [4] slot warps done, [5] queue warps done
      if ((threadIdx.x & 31) == 0 && gtid < M + (int64_t)p.S * kPhases) TRACE_FINE(gtid < M ? 4 : 5);
#endif
      const int32_t nrel = w.ctl->nrel;
      for (int64_t i = gtid; i < nrel; i += gstride) w.v.state[w.v.rel[i]] = kAtNode;
      m = block_max(m, smax);
      __shared__ bool is_last;
      if (threadIdx.x == 0) {
        if (m > 0) atomicMax(&w.ctl->max_occ_acc, m);
        trace_max(w.ctl, 6);
        // release: the block's stores (ordered before thread 0 by block_max's
        // barrier) and its atomicMax; acquire: the last block sees every
        // block's, and its threads see them after the barrier below
        is_last = atom_add_acq_rel(&w.ctl->blocks_done, 1u) == gridDim.x - 1;
      }
      __syncthreads();
      if (is_last && threadIdx.x == 0) {
        finalize_step(w);  // the kernel's completion publishes it
      }
      if (is_last && w.snap) block_snapshot(w.snap);  // (is_last is block-uniform)
      return;
    } else {
      for (int64_t s = gtid; s < p.S; s += gstride) {
        qt += sig_cde1(w, (int32_t)s);
        sig_e3(w, (int32_t)s);
      }
    }
    qt = block_sum(qt, red);
    if (threadIdx.x == 0 && qt) atomicAdd((unsigned long long*)&w.ctl->qtotal, (unsigned long long)qt);
    if (threadIdx.x == 0) trace_max(w.ctl, 5);
    grid.sync();
    // every slot, ELL padding included: padding slots carry no decisions,
    // deposits or occupancy and no walk reads them, so skipping the
    // validity load only shortens the dependent chain
    int32_t m = 0;
    for (int64_t s = gtid; s < w.g.M; s += gstride) {
      double wt = 0.0;
      int32_t load = 0;
      m = max(m, slot_fg(w, (int32_t)s, &wt, &load));
      if (w.lrec) lattice_quad(w, s, wt, load);
    }
    m = block_max(m, smax);
    if (threadIdx.x == 0 && m > 0) atomicMax(&w.ctl->max_occ_acc, m);
    if (threadIdx.x == 0) trace_max(w.ctl, 6);
    grid.sync();
    if (gtid == 0) finalize_step(w);
    if (blockIdx.x == 0 && w.snap) block_snapshot(w.snap);
    return;
  }
  ref_step<kDecideDK, true>(w, grid);
}

// ---------------------------------------------------------------------------
// Batched next-hop query (gmaco_next_node): next_node_{dijkstra,aco,maco}
// over the current field, one thread per query.
// ---------------------------------------------------------------------------
template <int DK>
__global__ void k_next_node(DevWorld w, int algorithm, int count, const int32_t* cur, const int32_t* dst,
                            const uint64_t* entity, const uint64_t* stepk, int64_t n_t, int32_t* out_next,
                            int32_t* out_via, uint8_t* out_dev) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int32_t x = cur[i];
  const Target<DK> t(w.d, dst[i]);
  int32_t slot = -1;
  bool dev = false;
  if (algorithm == 0) {
    slot = dijkstra_pick<DK>(w.g, t, x);
  } else {
    const Row r = scan_row<DK>(w.g, t, x);
    const uint32_t cand = (w.p.progress_filter && r.closer) ? r.closer : r.reach;
    if (cand) {
      if (algorithm == 1) {
        // fresh weights from the current tau (no colony congestion factor)
        double total = 0.0;
        int c = 0;
        double wv[kMaxDegree];
        for (uint32_t m = cand; m; m &= m - 1, ++c) {
          const int32_t s = r.first + __ffs(m) - 1;
          wv[c] = __dmul_rn(tau_alpha(w, w.tau[s]), w.g.eta_beta[s]);
          total = __dadd_rn(total, wv[c]);
        }
        const double u = to_unit(draw(w.p.seed, 5, entity[i], stepk[i]));
        int pick_i = c - 1;
        if (total <= 0.0 || !isfinite(total)) {
          const int pp = (int)__dmul_rn(u, (double)c);
          pick_i = pp < c - 1 ? pp : c - 1;
        } else {
          const double point = __dmul_rn(u, total);
          double cum = 0.0;
          for (int j = 0; j < c; ++j) {
            cum = __dadd_rn(cum, wv[j]);
            if (point < cum) {
              pick_i = j;
              break;
            }
          }
        }
        uint32_t m = cand;
        for (int j = 0; j < pick_i; ++j) m &= m - 1;
        slot = r.first + __ffs(m) - 1;
      } else {
        slot = maco_pick(w, r.first, cand, n_t, &dev);
      }
    }
  }
  out_via[i] = slot < 0 ? -1 : w.g.slot_edge[slot];
  out_next[i] = slot < 0 ? -1 : w.g.col[slot];
  out_dev[i] = dev ? 1 : 0;
}

// ---------------------------------------------------------------------------
// launch plumbing
// ---------------------------------------------------------------------------
static inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
// stages C..G: latency-bound per-entity chains, so small blocks spread them
// over as many SMs as possible
constexpr int kTail = 64;

// Dynamic shared memory of the staged grid walker (0 = read from global):
// the LatRec table, 16 B per slot, when it fits 96 KiB.
size_t grid_smem_bytes(const DevWorld& w) {
  const size_t bytes = 16 * (size_t)w.g.M;
  return (w.lrec && !w.lrec_stride && bytes <= (96u << 10)) ? bytes : 0;
}

// Move-bit words of a CTA (kTourBits): [threads][bit_words] u64.
size_t grid_bits_bytes(const DevWorld& w, int threads) {
  return w.p.grid_bits ? (size_t)threads * w.p.bit_words * 8 : 0;
}

// Shared-memory carveout of the non-staged lattice walker: just enough SMEM
// for the register-limited number of CTAs per SM (move-bit words + static
// arrays), the rest stays L1 for the weight / cost gathers.  Without it the
// driver favours L1 and the move-bit words cap residency (5 CTAs instead of 12
// on C5).
cudaError_t configure_grid_carveout(const DevWorld& w) {
  if (!w.p.grid_bits || grid_smem_bytes(w)) return cudaSuccess;
  const int K = w.p.ants, threads = (K % 32 == 0) ? K : 256;
  cudaFuncAttributes fa{};
  const bool one = threads == K;
  cudaError_t e = one ? cudaFuncGetAttributes(&fa, k_colony_grid<false, kTourBits, true>)
                      : cudaFuncGetAttributes(&fa, k_colony_grid<false, kTourBits>);
  if (e != cudaSuccess) return e;
  const int regs_blocks = 65536 / std::max(1, fa.numRegs * threads);
  const size_t per_block = fa.sharedSizeBytes + grid_bits_bytes(w, threads) + 1024;  // + per-CTA reserve
  const size_t need = per_block * std::max(1, std::min(regs_blocks, 32));
  const int pct = (int)std::min<size_t>(100, (need * 100 + (228u << 10) - 1) / (228u << 10));
  return one ? cudaFuncSetAttribute(k_colony_grid<false, kTourBits, true>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, pct)
             : cudaFuncSetAttribute(k_colony_grid<false, kTourBits>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

cudaError_t configure_kernels() {
  for (auto f : {k_colony_grid<true, kTourBits>, k_colony_grid<true, kTourScratch>, k_colony_grid<true, kTourReplay>,
                 k_colony_grid<false, kTourBits>, k_colony_grid<false, kTourBits, true>}) {
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 << 10);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Grid size of the cooperative tail: enough 128-thread blocks for the
// largest stage, capped at what is co-resident on the device.
int coop_tail_blocks(const DevWorld& w, int device) {
  int per_sm = 0, sms = 0, coop = 0;
  if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device) != cudaSuccess || !coop) return 0;
  // the variant that will be launched (colony worlds run the fused one)
  cudaError_t oe;
  if (w.p.algorithm == 4) {
    oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tail_coop<true, -1>, kTailCoop, 0);
  } else {  // the variants a reference-algorithm step may launch (with / without the fused stage B)
    int a = 0, b = 0, c = 0, d = 0, e = 0;
    oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_tail_coop<false, -1>, kTailCoop, 0);
    if (oe == cudaSuccess) oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_tail_coop<false, 0>, kTailCoop, 0);
    if (oe == cudaSuccess) oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_tail_coop<false, 1>, kTailCoop, 0);
    if (oe == cudaSuccess) oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d, k_run_coop<0>, kTailCoop, 0);
    if (oe == cudaSuccess) oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&e, k_run_coop<1>, kTailCoop, 0);
    per_sm = std::min(std::min(a, std::min(b, c)), std::min(d, e));
  }
  if (oe != cudaSuccess || per_sm < 1) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  // (colony worlds: slots and signals share one pass, see k_tail_coop)
  const int64_t work = std::max<int64_t>((int64_t)w.p.S + w.p.V, w.g.M + (w.p.algorithm == 4 ? (int64_t)w.p.S * kPhases : 0));
  const int64_t want = (work + kTailCoop - 1) / kTailCoop;
  return (int)std::min<int64_t>(want, (int64_t)per_sm * sms);
}

__global__ void k_rec_weights(DevWorld w) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < w.g.M) {
    *reinterpret_cast<double*>(w.rec + s) = w.weight[s];
    const int64_t c = w.ecost[s];
    w.rec[s].z = c <= INT32_MAX ? (int32_t)c : -1;
  }
}

cudaError_t sync_rec_weights(const DevWorld& w, cudaStream_t st) {
  if (!w.rec) return cudaSuccess;
  k_rec_weights<<<blocks_for(w.g.M, 256), 256, 0, st>>>(w);
  return cudaGetLastError();
}

// Gathers several device arrays into mapped pinned host memory in one launch
// (the batched readback of gmaco_get_vehicles: one kernel + one sync instead
// of one copy per field).
__global__ void k_pack(PackDesc d) {
  const PackField f = d.f[blockIdx.y];
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(f.src) | reinterpret_cast<uintptr_t>(f.dst)) & 15) == 0;
  size_t done = 0;
  if (vec) {
    const size_t n16 = f.bytes / 16;
    for (size_t i = tid; i < n16; i += stride)
      reinterpret_cast<uint4*>(f.dst)[i] = reinterpret_cast<const uint4*>(f.src)[i];
    done = n16 * 16;
  }
  for (size_t i = done + tid; i < f.bytes; i += stride)
    static_cast<char*>(f.dst)[i] = static_cast<const char*>(f.src)[i];
}

cudaError_t launch_pack(const PackDesc& d, cudaStream_t st) {
  if (d.n <= 0) return cudaSuccess;
  size_t mx = 0;
  for (int i = 0; i < d.n; ++i) mx = std::max(mx, d.f[i].bytes);
  const unsigned bx = (unsigned)std::min<size_t>(std::max<size_t>((mx / 16 + 255) / 256, 1), 1024);
  k_pack<<<dim3(bx, d.n), 256, 0, st>>>(d);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Distance service on the device: exact multi-target
// shortest distances dist(x -> target) over the reversed graph, int64 mm.
// Frontier Bellman-Ford: every (target, node) whose distance dropped is
// relaxed along its in-edges with int64 atomicMin; a per-state in-queue flag
// dedups the next frontier.  Shortest distances are unique, so the table is
// identical to the reference's Dijkstra (net.cpp:359-437) whatever the
// relaxation order.  Tables are destination-major [T][n].
// ---------------------------------------------------------------------------
__global__ void k_sssp_fill(int64_t* D, size_t total) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x)
    D[i] = kInf;
}

__global__ void k_sssp_seed(int64_t* D, const int32_t* dests, int32_t T, int32_t n, uint32_t* cur) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint32_t item = (uint32_t)t * (uint32_t)n + (uint32_t)dests[t];
  D[item] = 0;
  cur[t] = item;
}

// All rounds in one persistent cooperative launch, near/far ordered
// (delta-stepping without per-bucket lists): states whose new distance is
// <= T go to the near frontier, others to a far pile; when the near frontier
// empties, T grows by delta and the far pile is split (entries already at
// <= T move to near, the rest are compacted).  Exactness does not depend on
// delta or on the processing order: every improvement is still relaxed.
// Lists: q[0]/q[1] near in/out, q[2]/q[3] far cur/next; cnt[0..3] their sizes.
__device__ __forceinline__ void sssp_append(uint32_t* list, uint32_t* n, uint32_t item) {
  cg::coalesced_group g = cg::coalesced_threads();
  uint32_t base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(n, (uint32_t)g.size());
  base = g.shfl(base, 0);
  list[base + g.thread_rank()] = item;
}

__global__ void __launch_bounds__(256) k_sssp_coop(SsspArgs a, uint32_t* q0, uint32_t* q1, uint32_t* q2,
                                                   uint32_t* q3, uint32_t* cnt, uint32_t count, int64_t delta) {
  cg::grid_group grid = cg::this_grid();
  uint32_t* nl[2] = {q0, q1};
  uint32_t* fl[2] = {q2, q3};
  int cur = 0, fcur = 0;
  int64_t T = delta;
  uint32_t nfar = 0;
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, gsz = gridDim.x * blockDim.x;
  for (;;) {
    if (count) {
      const uint32_t* in = nl[cur];
      for (uint32_t i = gtid; i < count; i += gsz) {
        const uint32_t item = in[i];
        const uint32_t t = item / (uint32_t)a.n, u = item - t * (uint32_t)a.n;
        a.inq[item] = 0;
        __threadfence();
        const int64_t du = *((volatile int64_t*)(a.D + item));
        int64_t* Drow = a.D + (size_t)t * a.n;
        for (int32_t k = a.rptr[u]; k < a.rptr[u + 1]; ++k) {
          const int32_t v = a.rsrc[k];
          const int64_t nd = du + a.rlen[k];
          if (nd < Drow[v]) {
            const long long old = atomicMin(reinterpret_cast<long long*>(Drow + v), (long long)nd);
            if (nd < old) __threadfence();
            if (nd < old && atomicExch(a.inq + (size_t)t * a.n + v, 1u) == 0u) {
              const uint32_t it = t * (uint32_t)a.n + (uint32_t)v;
              if (nd <= T)
                sssp_append(nl[cur ^ 1], cnt + (cur ^ 1), it);
              else
                sssp_append(fl[fcur], cnt + 2 + fcur, it);
            }
          }
        }
      }
      grid.sync();
      if (grid.thread_rank() == 0) cnt[cur] = 0;
      count = *((volatile uint32_t*)(cnt + (cur ^ 1)));
      nfar = *((volatile uint32_t*)(cnt + 2 + fcur));
      grid.sync();
      cur ^= 1;
      continue;
    }
    if (!nfar) break;  // both frontiers empty: done
    // near frontier empty: raise the threshold and split the far pile
    T += delta;
    const uint32_t* fin = fl[fcur];
    for (uint32_t i = gtid; i < nfar; i += gsz) {
      const uint32_t item = fin[i];
      if (*((volatile int64_t*)(a.D + item)) <= T)
        sssp_append(nl[cur], cnt + cur, item);
      else
        sssp_append(fl[fcur ^ 1], cnt + 2 + (fcur ^ 1), item);
    }
    grid.sync();
    if (grid.thread_rank() == 0) cnt[2 + fcur] = 0;
    count = *((volatile uint32_t*)(cnt + cur));
    nfar = *((volatile uint32_t*)(cnt + 2 + (fcur ^ 1)));
    grid.sync();
    fcur ^= 1;
  }
}

cudaError_t sssp_run_coop(const SsspArgs& a, uint32_t* const* q, uint32_t* cnt, uint32_t count, int64_t delta,
                          int device, cudaStream_t st) {
  int per_sm = 0, sms = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sssp_coop, 256, 0);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)std::max(1, per_sm * sms));
  lc.blockDim = dim3(256);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, k_sssp_coop, a, q[0], q[1], q[2], q[3], cnt, count, delta);
}

cudaError_t sssp_fill_seed(int64_t* D, size_t total, const int32_t* dests, int32_t T, int32_t n, uint32_t* cur,
                           cudaStream_t st) {
  k_sssp_fill<<<(unsigned)std::min<size_t>((total + 255) / 256, 148 * 32), 256, 0, st>>>(D, total);
  k_sssp_seed<<<blocks_for(T, 256), 256, 0, st>>>(D, dests, T, n, cur);
  return cudaGetLastError();
}

// Reachability bitmap of a distance table for the host's spawn:
// out[x * words + t/64] bit t%64 = D[t][x] != inf.  Threads run over x, so
// the loads of a table row are coalesced.
__global__ void k_reach_bits(const int64_t* D, int32_t T, int32_t n, int64_t words, uint64_t* out) {
  const int64_t total = (int64_t)n * words;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t wd = i / n, x = i - wd * n;
    uint64_t bits = 0;
    for (int b = 0; b < 64; ++b) {
      const int64_t t = wd * 64 + b;
      if (t >= T) break;
      if (D[t * n + x] != kInf) bits |= uint64_t(1) << b;
    }
    out[x * words + wd] = bits;
  }
}

cudaError_t build_reach_bits(const int64_t* D, int32_t T, int32_t n, int64_t words, uint64_t* out, cudaStream_t st) {
  const int64_t total = (int64_t)n * words;
  k_reach_bits<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32), 256, 0, st>>>(D, T, n, words, out);
  return cudaGetLastError();
}

// Progress-filter bitmaps from a device distance table (see DevDist::fbits).
__global__ void k_fbits(const int64_t* D, int32_t n, int32_t T, const int32_t* col, const int32_t* from, int32_t M,
                        int64_t fbw, uint32_t* fb) {
  const size_t total = (size_t)T * fbw;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const size_t t = idx / fbw;
    const int64_t wd = (int64_t)(idx - t * fbw);
    const int64_t* Dr = D + t * n;
    uint32_t out = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t s = wd * 32 + b;
      if (s >= M) break;
      const int32_t c = col[s];
      if (c < 0) continue;
      const int64_t dn = Dr[c];
      if (dn != kInf && dn < Dr[from[s]]) out |= 1u << b;
    }
    fb[idx] = out;
  }
}

cudaError_t build_fbits(const DevWorld& w, int32_t T, uint32_t* fb, cudaStream_t st) {
  const size_t total = (size_t)T * w.d.fbw;
  k_fbits<<<(unsigned)std::min<size_t>((total + 255) / 256, 148 * 32), 256, 0, st>>>(w.d.table, w.g.n, T, w.g.col,
                                                                                      w.g.slot_from, w.g.M, w.d.fbw, fb);
  return cudaGetLastError();
}

// ---- per-target candidate rows (DevTT) ------------------------------------
// (t, p) pairs run t-major over the row placement order `place`, so a
// target's table inherits the shared rows' locality.

// closer bits of node x's row toward table row t (DevDist::fbits)
__device__ __forceinline__ uint32_t row_closer_bits(const DevWorld& w, int64_t t, int32_t x) {
  const int2 r = w.g.row[x];
  const uint32_t* fb = w.d.fbits + (size_t)t * w.d.fbw;
  const uint32_t lo = fb[r.x >> 5], hi = fb[(r.x >> 5) + 1];
  return __funnelshift_r(lo, hi, r.x & 31) & (r.y >= 32 ? 0xffffffffu : ((1u << r.y) - 1u));
}

__global__ void k_tt_count(DevWorld w, int32_t T, const int32_t* place, int32_t* units) {
  const int64_t n = w.g.n, total = (int64_t)T * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / n;
    const int c = __popc(row_closer_bits(w, t, place[i - t * n]));
    units[i] = max(1, (c + 1) >> 1);  // record pairs; a candidate-free row still owns one
  }
}

// offs: exclusive sums of units (t-major, +1 leading zero pair); meta[t*n + x]
__global__ void k_tt_meta(DevWorld w, int32_t T, const int32_t* place, const int64_t* offs, uint32_t* meta,
                          int64_t* base, int64_t* cstart, int32_t nch) {
  const int64_t n = w.g.n, total = (int64_t)T * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / n, p = i - t * n;
    const int32_t x = place[p];
    const int c = __popc(row_closer_bits(w, t, x));
    const int64_t off = offs[i] - offs[t * n];
    meta[t * n + x] = ((uint32_t)off << 8) | ((uint32_t)c << 4) | (uint32_t)w.g.deg[x];
    const int64_t r = 2 * (offs[i] + 1);  // pair 0 is the zero row
    if (p == 0) {
      base[t] = r;
      if (t > 0) cstart[(t - 1) * (nch + 1) + nch] = r;  // end of the previous table
    }
    if (p % kTTChunk == 0) cstart[t * (nch + 1) + p / kTTChunk] = r;
  }
}

__global__ void k_tt_fill(DevWorld w, int32_t T, const int32_t* place, const int64_t* offs, const uint32_t* meta,
                          int4* rec, int2* sm, int2* sl) {
  const int64_t n = w.g.n, total = (int64_t)T * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / n;
    const int32_t x = place[i - t * n];
    uint32_t bits = row_closer_bits(w, t, x);
    const int c = __popc(bits);
    const int first = w.g.row[x].x;
    const int64_t r0 = 2 * (offs[i] + 1);
    const int pad = 2 * max(1, (c + 1) >> 1);
    for (int j = 0; j < pad; ++j) {
      int32_t s = -1, m = 0;
      if (bits) {  // candidates in slot (= ascending neighbour) order
        s = first + __ffs(bits) - 1;
        bits &= bits - 1;
        m = (int32_t)meta[t * n + w.g.col[s]];
      }
      rec[r0 + j] = make_int4(0, 0, 0, m);
      sm[r0 + j] = make_int2(s, m);
      if (sl) sl[r0 + j] = make_int2(s, s >= 0 ? (int32_t)w.g.len[s] : 0);
    }
  }
}

// Block b refreshes chunk b / T of table b % T: the T tables' records of one
// row chunk are rewritten by consecutive blocks, so the shared slot records
// they gather are read from DRAM once and hit L2 for the other tables.
__global__ void __launch_bounds__(256, 4) k_tt_refresh(DevWorld w) {
  const int32_t T = w.tt.own_t ? w.tt.T_own : w.tt.T, nch = w.tt.nch;
  const int32_t t = w.tt.own_t ? w.tt.own_t[blockIdx.x % T] : (int32_t)(blockIdx.x % T), ch = blockIdx.x / T;
  const int64_t* cs = w.tt.cstart + (int64_t)t * (nch + 1);
  const int64_t lo = cs[ch];
  const int32_t cnt = (int32_t)(cs[ch + 1] - lo);
  const int2* __restrict__ sm = w.tt.sm + lo;
  int4* __restrict__ out = w.tt.rec + lo;
  const int4* __restrict__ R = w.rec;
  constexpr int U = 8;  // records in flight per thread
  for (int32_t i0 = threadIdx.x; i0 < cnt; i0 += U * 256) {
    int2 q[U];
#pragma unroll
    for (int k = 0; k < U; ++k) q[k] = i0 + k * 256 < cnt ? sm[i0 + k * 256] : make_int2(-1, 0);
    int4 r[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (q[k].x >= 0) r[k] = __ldg(R + q[k].x);  // the shared slot record {weight, int32 cost, -}
#pragma unroll
    for (int k = 0; k < U; ++k)  // padding records too: whole 32-B sectors, no L2 fill reads
      if (i0 + k * 256 < cnt)
        out[i0 + k * 256] = q[k].x >= 0 ? make_int4(r[k].x, r[k].y, r[k].z, q[k].y) : make_int4(0, 0, 0, 0);
  }
}

// dist(origin_i -> dest_i) of every vehicle from a [row][n] distance table
// (walk-order keys at create).
__global__ void k_gather_dist(const int64_t* table, int32_t n, const int32_t* row, const int32_t* x, int32_t count,
                              int64_t* out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = row[i] < 0 ? INT64_MAX : table[(size_t)row[i] * n + x[i]];
}
cudaError_t gather_dist(const int64_t* table, int32_t n, const int32_t* row, const int32_t* x, int32_t count,
                        int64_t* out, cudaStream_t st) {
  k_gather_dist<<<blocks_for(count, 256), 256, 0, st>>>(table, n, row, x, count, out);
  return cudaGetLastError();
}

// By-target sharding exchange: this rank's records in its walk order into the
// allgather send buffer, then every rank's records back to their vehicles.
__global__ void k_rec_pack(DevWorld w, int32_t* send, int32_t pad) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < pad) send[i] = i < w.p.shard_hi ? w.v.dec_rec[w.v.walk_order[i]] : -1;
}
__global__ void k_rec_unpack(DevWorld w, const int32_t* recv, const int32_t* gath, int32_t count) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count && gath[i] >= 0) w.v.dec_rec[gath[i]] = recv[i];
}
cudaError_t rec_pack(const DevWorld& w, int32_t* send, int32_t pad, cudaStream_t st) {
  k_rec_pack<<<blocks_for(pad, 256), 256, 0, st>>>(w, send, pad);
  return cudaGetLastError();
}
cudaError_t rec_unpack(const DevWorld& w, const int32_t* recv, const int32_t* gath, int32_t count, cudaStream_t st) {
  k_rec_unpack<<<blocks_for(count, 256), 256, 0, st>>>(w, recv, gath, count);
  return cudaGetLastError();
}

cudaError_t tt_count(const DevWorld& w, int32_t T, const int32_t* place, int32_t* units, cudaStream_t st) {
  k_tt_count<<<148 * 32, 256, 0, st>>>(w, T, place, units);
  return cudaGetLastError();
}

cudaError_t tt_scan(const int32_t* units, int64_t* offs, int64_t count, cudaStream_t st) {
  size_t bytes = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, bytes, units, offs, count, st);
  if (e != cudaSuccess) return e;
  void* tmp = nullptr;
  if ((e = cudaMallocAsync(&tmp, std::max<size_t>(bytes, 1), st)) != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(tmp, bytes, units, offs, count, st);
  cudaFreeAsync(tmp, st);
  return e;
}

cudaError_t tt_build(const DevWorld& w, int32_t T, const int32_t* place, const int64_t* offs, uint32_t* meta,
                     int64_t* base, int64_t* cstart, int4* rec, int2* sm, int2* sl, cudaStream_t st) {
  k_tt_meta<<<148 * 32, 256, 0, st>>>(w, T, place, offs, meta, base, cstart, w.tt.nch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // the zero row (records 0-1)
  if ((e = cudaMemsetAsync(rec, 0, 2 * sizeof(int4), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(sm, 0xff, 2 * sizeof(int2), st)) != cudaSuccess) return e;
  if (sl && (e = cudaMemsetAsync(sl, 0xff, 2 * sizeof(int2), st)) != cudaSuccess) return e;
  k_tt_fill<<<148 * 32, 256, 0, st>>>(w, T, place, offs, meta, rec, sm, sl);
  return cudaGetLastError();
}

cudaError_t tt_refresh(const DevWorld& w, cudaStream_t st) {
  if (!w.tt.rec) return cudaSuccess;
  k_tt_refresh<<<(w.tt.own_t ? w.tt.T_own : w.tt.T) * w.tt.nch, 256, 0, st>>>(w);
  return cudaGetLastError();
}

int queue_blocks(const DevWorld& w, int device) {
  if (!w.p.ant_queue) return 0;
  int per_sm = 0, sms = 0;
  const cudaError_t oe = w.tt.rec ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_colony_qt, 128, 0)
                                  : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_colony_q, 128, 0);
  if (oe != cudaSuccess || per_sm < 1) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  return per_sm * sms;  // persistent: one full wave
}

void colony_shape(int ants, int* threads, int* vpb) {
  int t = ants <= 256 ? 256 : ((ants + 31) / 32) * 32;
  *threads = t;
  *vpb = t / ants;
}

// Reference algorithms run stage B inside the cooperative tail (one launch
// per step) unless the step is split around an exchange (sharding) or the
// device has no cooperative launch.
static bool fuse_decide(const DevWorld& w, const StepResources& r) {
  return w.p.algorithm != 4 && r.coop_blocks > 0 && r.part == 0 && !w.p.sharded;
}

cudaError_t launch_step(const DevWorld& w, const StepResources& r, cudaStream_t st,
                        cudaEvent_t walk_begin, cudaEvent_t walk_end) {
  const int V = w.p.V, S = w.p.S, n = w.g.n;
  const int VS = w.p.shard_hi - w.p.shard_lo;  // vehicles planned on this rank
  if (walk_begin) cudaEventRecordWithFlags(walk_begin, st, r.capturing ? cudaEventRecordExternal : 0);
  if (r.part == 2) goto tail;
  if (w.p.algorithm == 4 && w.d.kind == 1 && w.g.ell == 4 && w.p.progress_filter && w.p.ants <= 256 && w.lrec) {
    const size_t smem = grid_smem_bytes(w);
    const int mode = w.p.grid_bits ? kTourBits : (w.p.scratch_mode ? kTourScratch : kTourReplay);
    // staged tables: pack vehicles into 256-thread CTAs; otherwise one
    // vehicle's colony per CTA when it fills whole warps
    // (whole warps: the block reductions' full-mask shuffles need every lane
    // of the last warp to exist; threads past vpb * K are idle)
    const int threads = smem ? (((256 / w.p.ants) * w.p.ants + 31) & ~31) : ((w.p.ants % 32 == 0) ? w.p.ants : 256);
    // +1: prefetch CTA; + kSigCtas: stages C, D, E1 beside the walk (e1_in_walk)
    const unsigned grid = blocks_for(VS, threads / w.p.ants) + 1 + (w.p.e1_in_walk ? kSigCtas : 0);
    const size_t dyn = smem + grid_bits_bytes(w, threads);  // staged tables, then move-bit words
#define GMACO_GRID(SM, MODE) k_colony_grid<SM, MODE><<<grid, threads, dyn, st>>>(w)
    if (smem) {
      if (mode == kTourBits) GMACO_GRID(true, kTourBits);
      else if (mode == kTourScratch) GMACO_GRID(true, kTourScratch);
      else GMACO_GRID(true, kTourReplay);
    } else {
      if (mode == kTourBits && threads == w.p.ants)
        k_colony_grid<false, kTourBits, true><<<grid, threads, dyn, st>>>(w);
      else if (mode == kTourBits) GMACO_GRID(false, kTourBits);
      else if (mode == kTourScratch) GMACO_GRID(false, kTourScratch);
      else GMACO_GRID(false, kTourReplay);
    }
#undef GMACO_GRID
  } else if (w.p.algorithm == 4 && w.g.ell == 4 && w.p.progress_filter && w.p.ants <= 256) {
    // one vehicle's colony per block when it fills whole warps (no block
    // barrier couples different vehicles' walk lengths), else packed
    const int threads = (w.p.ants % 32 == 0) ? w.p.ants : 256, vpb = threads / w.p.ants;
    if (w.d.kind == 1)
      k_colony_ell4<1><<<blocks_for(VS, vpb), threads, 0, st>>>(w);
    else
      k_colony_ell4<0><<<blocks_for(VS, vpb), threads, 0, st>>>(w);
  } else if (w.p.ant_queue) {
    if (w.tt.rec) {
      k_tt_refresh<<<(w.tt.own_t ? w.tt.T_own : w.tt.T) * w.tt.nch, 256, 0, st>>>(w);  // this step's weights / costs
      k_colony_pro<<<blocks_for(VS, 256), 256, 0, st>>>(w);
      k_colony_qt<<<r.queue_blocks, 128, 0, st>>>(w);
    } else {
      k_colony_pro<<<blocks_for(VS, 256), 256, 0, st>>>(w);
      k_colony_q<<<r.queue_blocks, 128, 0, st>>>(w);
    }
    k_colony_epi<<<blocks_for(VS, 8) + 1, 256, 0, st>>>(w);  // +1: prefetch CTA
  } else if (w.p.csr_walker) {
    const int vpb = 256 / w.p.ants;
    const unsigned grid = blocks_for(VS, vpb) + 1;  // +1: prefetch CTA
    const int threads = (vpb * w.p.ants + 31) & ~31;  // whole warps (full-mask block reductions)
    if (w.p.max_degree <= 8) {
      if (w.p.scratch_mode) k_colony_csr<8, true><<<grid, threads, 0, st>>>(w);
      else k_colony_csr<8, false><<<grid, threads, 0, st>>>(w);
    } else {
      if (w.p.scratch_mode) k_colony_csr<16, true><<<grid, threads, 0, st>>>(w);
      else k_colony_csr<16, false><<<grid, threads, 0, st>>>(w);
    }
  } else if (w.p.algorithm == 4) {
    int threads, vpb;
    colony_shape(w.p.ants, &threads, &vpb);
    const unsigned grid = blocks_for(VS, vpb);
    if (w.d.kind == 1) {
      if (w.p.progress_filter)
        k_colony<1, true><<<grid, threads, 0, st>>>(w);
      else
        k_colony<1, false><<<grid, threads, 0, st>>>(w);
    } else {
      if (w.p.progress_filter)
        k_colony<0, true><<<grid, threads, 0, st>>>(w);
      else
        k_colony<0, false><<<grid, threads, 0, st>>>(w);
    }
  } else if (!fuse_decide(w, r)) {
    if (w.d.kind == 1)
      k_decide<1><<<blocks_for(V, 256), 256, 0, st>>>(w);
    else
      k_decide<0><<<blocks_for(V, 256), 256, 0, st>>>(w);
  }
  if (walk_end) cudaEventRecordWithFlags(walk_end, st, r.capturing ? cudaEventRecordExternal : 0);
  if (r.part == 1) return cudaGetLastError();
tail:
  const bool fused = w.p.algorithm == 4;  // colony walks run E2 themselves
  if (w.p.sharded) {
    if (r.exchange) {  // NCCL: decisions allgather + deposit allreduce (captured with the step)
      cudaError_t e = r.exchange(r.exchange_ctx, st);
      if (e != cudaSuccess) return e;
    }
    const bool coop_tail = r.coop_blocks > 0;
    if (fused && !coop_tail)  // (the cooperative tail applies remote vehicles itself)
      k_apply_remote_move<<<blocks_for(V, 256), 256, 0, st>>>(w);
    else if (!fused)
      k_apply_remote<<<blocks_for(V, 256), 256, 0, st>>>(w);
  }
  if (r.coop_blocks > 0) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(r.coop_blocks);
    lc.blockDim = dim3(kTailCoop);
    lc.dynamicSmemBytes = 0;
    lc.stream = st;
    // programmatic dependent launch: the tail's CTAs are scheduled while the
    // walk drains and wait in griddepcontrol.wait for its completion + memory
    cudaLaunchAttribute at[2];
    int na = 0;
    if (w.p.pdl) {
      at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    // the one-pass lattice colony tail (e1_in_walk, unsharded) has no grid
    // barrier (the last block finalizes), so it needs no cooperative launch
    if (!(fused && w.p.e1_in_walk && !w.p.sharded)) {
      at[na].id = cudaLaunchAttributeCooperative;
      at[na++].val.cooperative = 1;
    }
    lc.attrs = at;
    lc.numAttrs = na;
    if (fused) return cudaLaunchKernelEx(&lc, k_tail_coop<true, -1>, w);
    if (fuse_decide(w, r))  // stage B inside the cooperative tail: one launch per step
      return w.d.kind == 1 ? cudaLaunchKernelEx(&lc, k_tail_coop<false, 1>, w)
                           : cudaLaunchKernelEx(&lc, k_tail_coop<false, 0>, w);
    return cudaLaunchKernelEx(&lc, k_tail_coop<false, -1>, w);
  }
  if (S > 0) k_signals<<<blocks_for(S, kTail), kTail, 0, st>>>(w);
  if (!fused) k_move<<<blocks_for(V, kTail), kTail, 0, st>>>(w);
  if (S > 0) k_e3<<<blocks_for(S, kTail), kTail, 0, st>>>(w);
  if (w.p.algorithm == 2 || w.p.algorithm == 3) {
    if (w.p.siblings_only) {
      k_scoped<<<blocks_for(n, kTail), kTail, 0, st>>>(w);
    } else {
      size_t bytes = r.scan_temp_bytes;
      cudaError_t e = cub::DeviceScan::ExclusiveSum(r.scan_temp, bytes, w.v.dflag, w.v.pos, V, st);
      if (e != cudaSuccess) return e;
    }
  }
  k_edges<<<blocks_for(w.g.M, kTail), kTail, 0, st>>>(w);
  return cudaGetLastError();
}

// Persistent multi-step run (k_run_coop) for reference algorithms.
bool run_coop_ok(const DevWorld& w, const StepResources& r) { return fuse_decide(w, r); }

cudaError_t launch_run_coop(const DevWorld& w, const StepResources& r, int64_t nsteps, cudaStream_t st) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(r.coop_blocks);
  lc.blockDim = dim3(kTailCoop);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return w.d.kind == 1 ? cudaLaunchKernelEx(&lc, k_run_coop<1>, w, nsteps)
                       : cudaLaunchKernelEx(&lc, k_run_coop<0>, w, nsteps);
}

// Engine kernels enqueued per step by launch_step (library kernels such as
// the CUB scan and NCCL collectives are not counted).
int kernels_per_step(const DevWorld& w, const StepResources& r) {
  if (fuse_decide(w, r)) return 1;  // k_tail_coop with stage B
  int k = 1;                 // stage-B walk / decide
  if (w.p.ant_queue) k += 2; // k_colony_pro + k_colony_epi around k_colony_q
  if (w.tt.rec) k += 1;      // k_tt_refresh
  if (w.p.sharded && !(w.p.algorithm == 4 && r.coop_blocks > 0))
    k += 1;  // k_apply_remote[_move] (folded into the cooperative colony tail otherwise)
  if (w.v.owner && r.exchange) k += 2;  // by-target shards: k_rec_pack / k_rec_unpack around the allgather
  if (r.coop_blocks > 0) return k + 1;  // k_tail_coop
  if (w.p.S > 0) k += 2;     // k_signals, k_e3
  if (w.p.algorithm != 4) k += 1;  // k_move (colony walks run E2 themselves)
  if ((w.p.algorithm == 2 || w.p.algorithm == 3) && w.p.siblings_only) k += 1;  // k_scoped
  return k + 1;              // k_edges
}

size_t scan_temp_bytes(int V) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int32_t*)nullptr, (int32_t*)nullptr, V);
  return bytes;
}

cudaError_t launch_next_node(const DevWorld& w, int algorithm, int count, const int32_t* cur,
                             const int32_t* dst, const uint64_t* entity, const uint64_t* stepk, int64_t n_t,
                             int32_t* out_next, int32_t* out_via, uint8_t* out_dev, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  if (w.d.kind == 1)
    k_next_node<1><<<blocks_for(count, 128), 128, 0, st>>>(w, algorithm, count, cur, dst, entity, stepk,
                                                           n_t, out_next, out_via, out_dev);
  else
    k_next_node<0><<<blocks_for(count, 128), 128, 0, st>>>(w, algorithm, count, cur, dst, entity, stepk,
                                                           n_t, out_next, out_via, out_dev);
  return cudaGetLastError();
}

}  // namespace gmaco
