// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle harness, never the product).
//
// A thin extern "C" layer over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libmacosim_ref.so).  It converts the POD blocks of
// include/gmaco.h into the reference's C++ types, so the parity tests and the
// bench's reference arm can drive the reference through the same parameter
// vocabulary the product exposes.  Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline / --impl reference) load this library.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "gmaco.h"
#include "macosim/engine.hpp"
#include "macosim/net.hpp"
#include "macosim/parallel.hpp"
#include "macosim/pheromone.hpp"
#include "macosim/rng.hpp"
#include "macosim/routing.hpp"
#include "macosim/signals.hpp"

using namespace macosim;

namespace {

thread_local std::string g_err;

int fail_with(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define GUARD(body)                                         \
  try {                                                     \
    body                                                    \
  } catch (const ValidationError& e) {                      \
    return fail_with(e, 1);                                 \
  } catch (const std::exception& e) {                       \
    return fail_with(e, 2);                                 \
  }

RoadNetwork to_network(const gmaco_graph_desc* g) {
  std::vector<RoadNode> nodes(g->node_count);
  for (int i = 0; i < g->node_count; ++i) {
    nodes[i].id = i;
    nodes[i].signalized = g->signalized && g->signalized[i] != 0;
  }
  std::vector<RoadEdge> edges(g->edge_count);
  for (int i = 0; i < g->edge_count; ++i) {
    edges[i] = RoadEdge{i, g->edge_from[i], g->edge_to[i], g->edge_length_mm[i],
                        g->edge_lanes ? g->edge_lanes[i] : 1};
  }
  return RoadNetwork(std::move(nodes), std::move(edges));
}

SimConfig to_config(const gmaco_sim_config* c, const RoadNetwork* net) {
  SimConfig s;
  s.network = net;
  switch (c->algorithm) {
    case GMACO_DIJKSTRA: s.algorithm = Algorithm::Dijkstra; break;
    case GMACO_ACO: s.algorithm = Algorithm::Aco; break;
    case GMACO_MACO: s.algorithm = Algorithm::Maco; break;
    case GMACO_MACO_P: s.algorithm = Algorithm::MacoP; break;
    default: throw ValidationError("reference has no algorithm " + std::to_string(c->algorithm));
  }
  s.controller = static_cast<ControllerKind>(c->controller);
  s.vehicle_count = c->vehicle_count;
  s.dt_s = c->dt_s;
  s.max_steps = c->max_steps;
  s.seed = c->seed;
  s.decision_latency_s = c->decision_latency_s;
  s.spawn = c->spawn == GMACO_UNIFORM_WINDOW ? SpawnMode::UniformWindow : SpawnMode::AllAtStart;
  s.spawn_window_steps = c->spawn_window_steps;
  s.od.pattern = c->od_pattern == GMACO_OD_BLOCKS ? OdPattern::Blocks : OdPattern::UniformPairs;
  s.od.bias = c->od_bias;
  for (int i = 0; i < c->od_block_a_len; ++i) s.od.block_a.push_back(c->od_block_a[i]);
  for (int i = 0; i < c->od_block_b_len; ++i) s.od.block_b.push_back(c->od_block_b[i]);
  s.speed_min_mps = c->speed_min_mps;
  s.speed_max_mps = c->speed_max_mps;
  const gmaco_pheromone_params& p = c->pheromone;
  s.pheromone.tau_init_lo = p.tau_init_lo;
  s.pheromone.tau_init_hi = p.tau_init_hi;
  s.pheromone.delta_inc = p.delta_inc;
  s.pheromone.delta_dec = p.delta_dec;
  s.pheromone.rho = p.rho;
  s.pheromone.tau_min = p.tau_min;
  s.pheromone.tau_max = p.tau_max;
  s.pheromone.aco_deposit_q = p.aco_deposit_q;
  s.pheromone.decrement_siblings_only = p.decrement_siblings_only != 0;
  s.signal.th_max = c->signal.th_max;
  s.signal.t_max = c->signal.t_max;
  s.signal.green_duration_s = c->signal.green_duration_s;
  s.signal.saturation_flow = c->signal.saturation_flow;
  for (int i = 0; i < kPhaseCount; ++i) s.signal.fixed_cycle_order[i] = c->signal.fixed_cycle_order[i];
  s.routing.deviation_threshold = c->routing.deviation_threshold;
  s.routing.deviation_mode = c->routing.deviation_mode == GMACO_DEV_EDGE_OCCUPANCY
                                 ? DeviationMode::EdgeOccupancy
                                 : DeviationMode::Global;
  s.routing.progress_filter = c->routing.progress_filter != 0;
  s.routing.aco_alpha = c->routing.aco_alpha;
  s.routing.aco_beta = c->routing.aco_beta;
  return s;
}

PheromoneParams to_pheromone(const gmaco_pheromone_params* p) {
  PheromoneParams q;
  q.tau_init_lo = p->tau_init_lo;
  q.tau_init_hi = p->tau_init_hi;
  q.delta_inc = p->delta_inc;
  q.delta_dec = p->delta_dec;
  q.rho = p->rho;
  q.tau_min = p->tau_min;
  q.tau_max = p->tau_max;
  q.aco_deposit_q = p->aco_deposit_q;
  q.decrement_siblings_only = p->decrement_siblings_only != 0;
  return q;
}

SignalParams to_signal(const gmaco_signal_params* p) {
  SignalParams q;
  q.th_max = p->th_max;
  q.t_max = p->t_max;
  q.green_duration_s = p->green_duration_s;
  q.saturation_flow = p->saturation_flow;
  for (int i = 0; i < kPhaseCount; ++i) q.fixed_cycle_order[i] = p->fixed_cycle_order[i];
  return q;
}

void fill_result(const RunResult& r, gmaco_run_result* out, double* travel, int32_t* rvid,
                 int32_t* rnode, int32_t cap) {
  out->mean_travel_s = r.mean_travel_s;
  out->mean_wait_s = r.mean_wait_s;
  out->mean_queue_len = r.mean_queue_len;
  out->max_edge_occupancy = r.max_edge_occupancy;
  out->completed_count = r.completed_count;
  out->retired_count = r.retired_count;
  out->steps_executed = r.steps_executed;
  out->wall_clock_ms = r.wall_clock_ms;
  if (travel) std::copy(r.travel_times_s.begin(), r.travel_times_s.end(), travel);
  // diagnostics: "vehicle V retired unroutable at node N"
  int k = 0;
  for (const std::string& d : r.diagnostics) {
    if (k >= cap) break;
    int v = -1, n = -1;
    std::sscanf(d.c_str(), "vehicle %d retired unroutable at node %d", &v, &n);
    if (rvid) rvid[k] = v;
    if (rnode) rnode[k] = n;
    ++k;
  }
}

struct RefWorld {
  std::unique_ptr<RoadNetwork> net;
  std::unique_ptr<DistanceTable> dist;
  World w;
};

void copy_vehicles(const std::vector<Vehicle>& vs, const gmaco_vehicle_view* v) {
  for (std::size_t i = 0; i < vs.size(); ++i) {
    const Vehicle& x = vs[i];
    if (v->origin) v->origin[i] = x.origin;
    if (v->dest) v->dest[i] = x.dest;
    if (v->speed_mps) v->speed_mps[i] = x.speed_mps;
    if (v->advance_mm) v->advance_mm[i] = x.advance_mm;
    if (v->state) v->state[i] = static_cast<uint8_t>(x.state);
    if (v->at_node) v->at_node[i] = x.at_node;
    if (v->on_edge) v->on_edge[i] = x.on_edge;
    if (v->progress_mm) v->progress_mm[i] = x.progress_mm;
    if (v->overshoot_mm) v->overshoot_mm[i] = x.overshoot_mm;
    if (v->queued_phase) v->queued_phase[i] = x.queued_phase;
    if (v->queue_joined_step) v->queue_joined_step[i] = x.queue_joined_step;
    if (v->depart_step) v->depart_step[i] = x.depart_step;
    if (v->arrive_step) v->arrive_step[i] = x.arrive_step;
    if (v->latency_debt_us) v->latency_debt_us[i] = x.latency_debt_us;
    if (v->driving_steps) v->driving_steps[i] = x.driving_steps;
    if (v->queued_steps) v->queued_steps[i] = x.queued_steps;
    if (v->latency_steps) v->latency_steps[i] = x.latency_steps;
    if (v->decisions) v->decisions[i] = x.decisions;
    if (v->deviations) v->deviations[i] = x.deviations;
    if (v->path_length_mm) v->path_length_mm[i] = x.path_length_mm;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- rng.hpp -------------------------------------------------------------
uint64_t ref_mix64(uint64_t x) { return rng::mix64(x); }
uint64_t ref_draw(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return rng::draw(seed, a, b, c);
}
double ref_to_unit(uint64_t bits) { return rng::to_unit(bits); }
double ref_uniform(uint64_t bits, double lo, double hi) { return rng::uniform(bits, lo, hi); }
uint64_t ref_below(uint64_t bits, uint64_t n) { return rng::below(bits, n); }

// ---- net.cpp ---------------------------------------------------------------
// Sizes: node_count = rows*cols, edge_count = 2*(rows*(cols-1)+cols*(rows-1)).
int ref_generate_grid(int rows, int cols, double len_m, int lanes, int sig_interior,
                      uint8_t* signalized, int32_t* from, int32_t* to, int64_t* len_mm,
                      int32_t* lanes_out) {
  GUARD({
    RoadNetwork net = generate_grid(rows, cols, len_m, lanes, sig_interior != 0, 0);
    for (const RoadNode& n : net.nodes()) signalized[n.id] = n.signalized;
    for (const RoadEdge& e : net.edges()) {
      from[e.id] = e.from;
      to[e.id] = e.to;
      len_mm[e.id] = e.length_mm;
      lanes_out[e.id] = e.lanes;
    }
    return 0;
  })
}

// edge_count = 2*links.
int ref_generate_city(int nodes, int links, int lanes, uint64_t seed, uint8_t* signalized,
                      int32_t* from, int32_t* to, int64_t* len_mm, int32_t* lanes_out) {
  GUARD({
    RoadNetwork net = generate_city(nodes, links, lanes, seed);
    for (const RoadNode& n : net.nodes()) signalized[n.id] = n.signalized;
    for (const RoadEdge& e : net.edges()) {
      from[e.id] = e.from;
      to[e.id] = e.to;
      len_mm[e.id] = e.length_mm;
      lanes_out[e.id] = e.lanes;
    }
    return 0;
  })
}

// serialize_network (net.cpp:179-200) of a generated city (which carries
// node positions): *len = text length, written when cap >= *len.
int ref_serialize_city(int nodes, int links, int lanes, uint64_t seed, char* buf, size_t cap, size_t* len) {
  GUARD({
    const std::string s = serialize_network(generate_city(nodes, links, lanes, seed));
    *len = s.size();
    if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
    return 0;
  })
}

// serialize_network of a descriptor network (no positions).
int ref_serialize_desc(const gmaco_graph_desc* g, char* buf, size_t cap, size_t* len) {
  GUARD({
    const std::string s = serialize_network(to_network(g));
    *len = s.size();
    if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
    return 0;
  })
}

// load_network (net.cpp:112-168): sizes, then (arrays non-null) the SoA.
int ref_load_network(const char* text, size_t len, int32_t* n_out, int32_t* m_out, uint8_t* signalized,
                     int32_t* from, int32_t* to, int64_t* len_mm, int32_t* lanes_out, double* x, double* y,
                     uint8_t* has_pos) {
  GUARD({
    RoadNetwork net = load_network(std::string(text, len));
    *n_out = net.node_count();
    *m_out = net.edge_count();
    if (signalized)
      for (const RoadNode& nd : net.nodes()) {
        signalized[nd.id] = nd.signalized;
        if (x) x[nd.id] = nd.x_m;
        if (y) y[nd.id] = nd.y_m;
        if (has_pos) has_pos[nd.id] = nd.has_position;
      }
    if (from)
      for (const RoadEdge& e : net.edges()) {
        from[e.id] = e.from;
        to[e.id] = e.to;
        len_mm[e.id] = e.length_mm;
        lanes_out[e.id] = e.lanes;
      }
    return 0;
  })
}

// Validates through the RoadNetwork constructor (net.cpp:38-98).
int ref_validate_graph(const gmaco_graph_desc* g) {
  GUARD({
    (void)to_network(g);
    return 0;
  })
}

int ref_apsp(const gmaco_graph_desc* g, int64_t* dist, int32_t* next) {
  GUARD({
    RoadNetwork net = to_network(g);
    DistanceTable t = all_pairs_distances(net);
    const int n = net.node_count();
    for (int u = 0; u < n; ++u)
      for (int v = 0; v < n; ++v) {
        if (dist) dist[static_cast<std::size_t>(u) * n + v] = t.dist_mm(u, v);
        if (next) next[static_cast<std::size_t>(u) * n + v] = t.next_hop(u, v);
      }
    return 0;
  })
}

// ---- pheromone.cpp / parallel.cpp fold ------------------------------------
int64_t ref_evaporate_one(int64_t tau, const gmaco_pheromone_params* p) {
  return evaporate_one(tau, to_pheromone(p));
}
int64_t ref_deposit_amount(int64_t len_mm, const gmaco_pheromone_params* p) {
  try {
    return deposit_amount(len_mm, to_pheromone(p));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
int64_t ref_fold_maco_edge(int64_t tau, const int32_t* positions, int32_t n, int64_t total,
                           const gmaco_pheromone_params* p) {
  return fold_maco_edge(tau, std::span<const std::int32_t>(positions, n), total, to_pheromone(p));
}
// Stage F+G edge kernel of the reference's parallel executor
// (commit_pheromone, parallel.cpp:195-231): per edge,
// evaporate_one(fold_maco_edge(tau, positions of its decisions, D)), edges
// split over `threads` std::threads in contiguous ranges (partition_entities,
// parallel.cpp:8-21).  dec_edge[D] lists the step's decisions in vid order.
// Runs `iters` passes over tau (in place) and returns the seconds they took
// (edge-updates/s = m * iters / seconds).
double ref_fold_bench(int64_t* tau, int32_t m, const int32_t* dec_edge, int32_t D, int32_t iters,
                      int32_t threads, const gmaco_pheromone_params* p) {
  const PheromoneParams pp = to_pheromone(p);
  std::vector<int32_t> start(m + 1, 0), pos(D);
  for (int32_t i = 0; i < D; ++i) start[dec_edge[i] + 1]++;
  for (int32_t e = 0; e < m; ++e) start[e + 1] += start[e];
  std::vector<int32_t> fill(start.begin(), start.end() - 1);
  for (int32_t i = 0; i < D; ++i) pos[fill[dec_edge[i]]++] = i;  // ascending position per edge
  if (threads < 1) threads = 1;
  auto ranges = partition_entities(m, threads);
  const auto t0 = std::chrono::steady_clock::now();
  for (int32_t it = 0; it < iters; ++it) {
    auto work = [&](int t) {
      for (int32_t e = ranges[t].begin; e < ranges[t].end; ++e)
        tau[e] = evaporate_one(fold_maco_edge(tau[e], std::span<const std::int32_t>(pos.data() + start[e],
                                                                                     start[e + 1] - start[e]),
                                              D, pp),
                               pp);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int ref_apply_maco_update(int64_t* tau, int32_t m, int32_t chosen, const gmaco_pheromone_params* p) {
  GUARD({
    std::vector<TauMicros> t(tau, tau + m);
    apply_maco_update(t, chosen, to_pheromone(p));
    std::copy(t.begin(), t.end(), tau);
    return 0;
  })
}
int ref_init_random(const gmaco_graph_desc* g, const gmaco_pheromone_params* p, uint64_t seed,
                    int64_t* tau) {
  GUARD({
    RoadNetwork net = to_network(g);
    PheromoneField f = init_random(net, to_pheromone(p), seed);
    for (int e = 0; e < f.size(); ++e) tau[e] = f.level(e);
    return 0;
  })
}

// ---- signals.cpp -------------------------------------------------------------
// kind: 0 fixed, 1 adaptive, 2 preemptive.
int ref_select_phase(int kind, const int32_t* qlen, const double* head_wait, int cursor,
                     const gmaco_signal_params* sp) {
  SignalParams p = to_signal(sp);
  SignalState s;
  s.node = 0;
  for (int i = 0; i < kPhaseCount; ++i) {
    for (int k = 0; k < qlen[i]; ++k) s.phases[i].queue.push_back(QueueEntry{k, 0});
    s.phases[i].head_wait_s = head_wait[i];
  }
  s.cycle_cursor = cursor;
  s.green = cursor;
  switch (kind) {
    case 0: return select_phase_fixed(s, p);
    case 1: return select_phase_adaptive(s, p);
    default: return select_phase_preemptive(s, p);
  }
}

// One discharge call on a single green queue of `qlen` vehicles (ids 0..),
// returning the released count and the updated remainder.
int ref_discharge(int32_t qlen, double* remainder, double dt, int lanes,
                  const gmaco_signal_params* sp) {
  SignalParams p = to_signal(sp);
  SignalState s;
  s.green = 0;
  for (int k = 0; k < qlen; ++k) s.phases[0].queue.push_back(QueueEntry{k, 0});
  s.phases[0].service_remainder = *remainder;
  auto rel = discharge(s, dt, lanes, p);
  *remainder = s.phases[0].service_remainder;
  return static_cast<int>(rel.size());
}

// ---- engine.cpp / parallel.cpp ------------------------------------------------
// workers <= 0: run(cfg, dist); workers >= 1: parallel_run(cfg, dist, workers).
int ref_run(const gmaco_graph_desc* g, const gmaco_sim_config* c, int32_t workers,
            gmaco_run_result* out, double* travel, int32_t* rvid, int32_t* rnode, int32_t cap) {
  GUARD({
    RoadNetwork net = to_network(g);
    SimConfig cfg = to_config(c, &net);
    cfg.validate();
    DistanceTable dist = all_pairs_distances(net);
    RunResult r = workers <= 0 ? run(cfg, dist) : parallel_run(cfg, dist, workers);
    fill_result(r, out, travel, rvid, rnode, cap);
    return 0;
  })
}

int ref_spawn(const gmaco_graph_desc* g, const gmaco_sim_config* c, int32_t* origin,
              int32_t* dest, double* speed, int64_t* advance, int64_t* depart) {
  GUARD({
    RoadNetwork net = to_network(g);
    SimConfig cfg = to_config(c, &net);
    cfg.validate();
    DistanceTable dist = all_pairs_distances(net);
    auto fleet = spawn_vehicles(cfg, net, dist);
    for (std::size_t i = 0; i < fleet.size(); ++i) {
      origin[i] = fleet[i].origin;
      dest[i] = fleet[i].dest;
      speed[i] = fleet[i].speed_mps;
      advance[i] = fleet[i].advance_mm;
      depart[i] = fleet[i].depart_step;
    }
    return 0;
  })
}

void* ref_world_create(const gmaco_graph_desc* g, const gmaco_sim_config* c) {
  try {
    auto rw = std::make_unique<RefWorld>();
    rw->net = std::make_unique<RoadNetwork>(to_network(g));
    SimConfig cfg = to_config(c, rw->net.get());
    cfg.validate();
    rw->dist = std::make_unique<DistanceTable>(all_pairs_distances(*rw->net));
    rw->w = init_world(cfg, *rw->dist);
    return rw.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_world_destroy(void* h) { delete static_cast<RefWorld*>(h); }

int64_t ref_world_step(void* h, int64_t n) {
  auto* rw = static_cast<RefWorld*>(h);
  int64_t k = 0;
  for (; k < n && !finished(rw->w); ++k) sequential_step(rw->w);
  return k;
}

int ref_world_finished(void* h) { return finished(static_cast<RefWorld*>(h)->w) ? 1 : 0; }
int64_t ref_world_current_step(void* h) { return static_cast<RefWorld*>(h)->w.step; }

int ref_world_vehicles(void* h, const gmaco_vehicle_view* v) {
  copy_vehicles(static_cast<RefWorld*>(h)->w.vehicles, v);
  return 0;
}

int ref_world_path(void* h, int32_t vid, int32_t* out, int32_t cap, int32_t* len) {
  const auto& p = static_cast<RefWorld*>(h)->w.vehicles.at(vid).path_edges;
  *len = static_cast<int32_t>(p.size());
  for (int i = 0; i < std::min<int>(cap, p.size()); ++i) out[i] = p[i];
  return 0;
}

int ref_world_pheromone(void* h, int64_t* tau) {
  const auto& f = static_cast<RefWorld*>(h)->w.field;
  for (int e = 0; e < f.size(); ++e) tau[e] = f.level(e);
  return 0;
}

int ref_world_occupancy(void* h, int32_t* occ) {
  const auto& o = static_cast<RefWorld*>(h)->w.edge_occupancy;
  std::copy(o.begin(), o.end(), occ);
  return 0;
}

int32_t ref_world_signal_count(void* h) {
  return static_cast<int32_t>(static_cast<RefWorld*>(h)->w.signals.size());
}

int ref_world_signals(void* h, const gmaco_signal_view* v, int64_t cap) {
  const auto& sigs = static_cast<RefWorld*>(h)->w.signals;
  int64_t q = 0;
  for (std::size_t s = 0; s < sigs.size(); ++s) {
    const SignalState& st = sigs[s];
    if (v->node) v->node[s] = st.node;
    if (v->green) v->green[s] = st.green;
    if (v->cycle_cursor) v->cycle_cursor[s] = st.cycle_cursor;
    if (v->discharge_lanes) v->discharge_lanes[s] = st.discharge_lanes;
    if (v->green_elapsed_steps) v->green_elapsed_steps[s] = st.green_elapsed_steps;
    if (v->green_elapsed_s) v->green_elapsed_s[s] = st.green_elapsed_s;
    for (int p = 0; p < kPhaseCount; ++p) {
      const SignalPhase& ph = st.phases[p];
      const std::size_t k = s * kPhaseCount + p;
      if (v->queue_len) v->queue_len[k] = static_cast<int32_t>(ph.queue.size());
      if (v->head_wait_s) v->head_wait_s[k] = ph.head_wait_s;
      if (v->service_remainder) v->service_remainder[k] = ph.service_remainder;
      for (const QueueEntry& qe : ph.queue) {
        if (q < cap) {
          if (v->queue_vid) v->queue_vid[q] = qe.vehicle;
          if (v->queue_enqueue_step) v->queue_enqueue_step[q] = qe.enqueue_step;
        }
        ++q;
      }
    }
  }
  return q > cap ? 1 : 0;
}

int ref_world_collect(void* h, gmaco_run_result* out, double* travel, int32_t* rvid,
                      int32_t* rnode, int32_t cap) {
  RunResult r = collect_result(static_cast<RefWorld*>(h)->w);
  fill_result(r, out, travel, rvid, rnode, cap);
  return 0;
}

// Batched routing.hpp next_node_* over the world's current field / occupancy.
int ref_world_next_node(void* h, int algorithm, int32_t count, const int32_t* current,
                        const int32_t* dest, const uint64_t* entity, const uint64_t* step,
                        int64_t n_t, int32_t* out_next, int32_t* out_via, uint8_t* out_dev) {
  auto* rw = static_cast<RefWorld*>(h);
  const World& w = rw->w;
  for (int32_t i = 0; i < count; ++i) {
    std::optional<RouteDecision> rd;
    switch (algorithm) {
      case GMACO_DIJKSTRA:
        rd = next_node_dijkstra(current[i], dest[i], *w.net, *w.dist);
        break;
      case GMACO_ACO:
        rd = next_node_aco(current[i], dest[i], *w.net, w.field, *w.dist, w.cfg.routing,
                           RngKey{w.cfg.seed, entity[i], step[i]});
        break;
      default:
        rd = next_node_maco(current[i], dest[i], *w.net, w.field, *w.dist, w.cfg.routing, n_t,
                            w.edge_occupancy);
        break;
    }
    out_next[i] = rd ? rd->next : -1;
    out_via[i] = rd ? rd->via : -1;
    out_dev[i] = rd ? rd->deviated : 0;
  }
  return 0;
}

// ---- reference-arm workload (bench.py --impl reference) ----------------------
// Colony tour construction with the reference's own routing rule: for every
// active vehicle, `ants` full tours from its current position to its
// destination, each hop one next_node_aco call (routing.cpp:77-115), spread
// over `threads` std::threads by contiguous vehicle ranges (the
// partition_entities scheme, parallel.cpp:8-21); best tour by (length, ant);
// then one reference sequential_step (engine.cpp:352-400) advances the world.
// Returns ant-steps executed; *routes receives the tours completed.
int64_t ref_world_colony_iteration(void* h, int32_t ants, int32_t threads, int64_t* routes) {
  auto* rw = static_cast<RefWorld*>(h);
  World& w = rw->w;
  const int32_t V = static_cast<int32_t>(w.vehicles.size());
  if (threads < 1) threads = 1;
  auto ranges = partition_entities(V, threads);
  std::vector<int64_t> steps(threads, 0), done(threads, 0);
  auto work = [&](int t) {
    int64_t s = 0, r = 0;
    for (int32_t vid = ranges[t].begin; vid < ranges[t].end; ++vid) {
      const Vehicle& v = w.vehicles[vid];
      NodeId start;
      switch (v.state) {
        case VehicleState::AtNode:
        case VehicleState::Queued: start = v.at_node; break;
        case VehicleState::OnEdge: start = w.net->edge(v.on_edge).to; break;
        case VehicleState::Pending:
          if (v.depart_step != w.step) continue;
          start = v.origin;
          break;
        default: continue;
      }
      if (start == v.dest) continue;
      LengthMm best = kUnreachableMm;
      for (int32_t a = 0; a < ants; ++a) {
        NodeId x = start;
        LengthMm cost = 0;
        std::uint64_t hop = 0;
        while (x != v.dest) {
          auto rd = next_node_aco(x, v.dest, *w.net, w.field, *w.dist, w.cfg.routing,
                                  RngKey{w.cfg.seed,
                                         static_cast<std::uint64_t>(vid) |
                                             (static_cast<std::uint64_t>(a) << 32),
                                         static_cast<std::uint64_t>(w.step) | (hop << 40)});
          ++s;
          if (!rd) {
            cost = kUnreachableMm;
            break;
          }
          cost += w.net->edge(rd->via).length_mm;
          x = rd->next;
          ++hop;
        }
        best = std::min(best, cost);
      }
      ++r;
    }
    steps[t] = s;
    done[t] = r;
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  int64_t total = 0, rt = 0;
  for (int t = 0; t < threads; ++t) {
    total += steps[t];
    rt += done[t];
  }
  if (!finished(w)) sequential_step(w);
  if (routes) *routes = rt;
  return total;
}

}  // extern "C"
