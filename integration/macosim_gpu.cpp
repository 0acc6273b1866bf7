// macosim_gpu.cpp — implementation of gpu_run over the C ABI (include/gmaco.h).
// Converts the reference's types (RoadNetwork net.hpp:52-80, DistanceTable
// net.hpp:84-102, SimConfig engine.hpp:29-50) into the ABI's POD blocks and
// rebuilds RunResult (engine.hpp:92-107), diagnostics included
// (engine.cpp:416-421).
#include "macosim_gpu.hpp"

#include <chrono>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "gmaco.h"

namespace macosim {

namespace {

gmaco_sim_config to_abi(const SimConfig& c) {
  gmaco_sim_config o{};
  switch (c.algorithm) {
    case Algorithm::Dijkstra: o.algorithm = GMACO_DIJKSTRA; break;
    case Algorithm::Aco: o.algorithm = GMACO_ACO; break;
    case Algorithm::Maco: o.algorithm = GMACO_MACO; break;
    case Algorithm::MacoP: o.algorithm = GMACO_MACO_P; break;
  }
  o.controller = static_cast<int32_t>(c.controller);
  o.vehicle_count = c.vehicle_count;
  o.spawn = c.spawn == SpawnMode::UniformWindow ? GMACO_UNIFORM_WINDOW : GMACO_ALL_AT_START;
  o.spawn_window_steps = c.spawn_window_steps;
  o.od_pattern = c.od.pattern == OdPattern::Blocks ? GMACO_OD_BLOCKS : GMACO_OD_UNIFORM;
  o.dt_s = c.dt_s;
  o.max_steps = c.max_steps;
  o.seed = c.seed;
  o.decision_latency_s = c.decision_latency_s;
  o.od_bias = c.od.bias;
  o.od_block_a = c.od.block_a.data();
  o.od_block_b = c.od.block_b.data();
  o.od_block_a_len = static_cast<int32_t>(c.od.block_a.size());
  o.od_block_b_len = static_cast<int32_t>(c.od.block_b.size());
  o.speed_min_mps = c.speed_min_mps;
  o.speed_max_mps = c.speed_max_mps;
  const PheromoneParams& p = c.pheromone;
  o.pheromone = {p.tau_init_lo, p.tau_init_hi, p.delta_inc, p.delta_dec, p.rho, p.tau_min, p.tau_max,
                 p.aco_deposit_q, p.decrement_siblings_only ? 1 : 0, 0};
  o.signal.th_max = c.signal.th_max;
  for (int i = 0; i < GMACO_PHASES; ++i) o.signal.fixed_cycle_order[i] = c.signal.fixed_cycle_order[i];
  o.signal.t_max = c.signal.t_max;
  o.signal.green_duration_s = c.signal.green_duration_s;
  o.signal.saturation_flow = c.signal.saturation_flow;
  o.routing.deviation_threshold = c.routing.deviation_threshold;
  o.routing.deviation_mode =
      c.routing.deviation_mode == DeviationMode::EdgeOccupancy ? GMACO_DEV_EDGE_OCCUPANCY : GMACO_DEV_GLOBAL;
  o.routing.progress_filter = c.routing.progress_filter ? 1 : 0;
  o.routing.aco_alpha = c.routing.aco_alpha;
  o.routing.aco_beta = c.routing.aco_beta;
  o.colony = {1, 1, 0, GMACO_RNG_REFERENCE, 0, GMACO_DEPOSIT_COMPLETION, 0, 0};
  return o;
}

[[noreturn]] void raise(int rc, const char* msg) {
  if (rc == GMACO_EVALIDATION) throw ValidationError(msg);
  throw std::runtime_error(std::string("gmaco: ") + msg);
}

// Builds the graph descriptor, runs the engine to completion and rebuilds
// RunResult.  `dd` selects the distance service the engine uses.
RunResult run_on_device(const SimConfig& cfg, gmaco_distance_desc dd, int device,
                        std::chrono::steady_clock::time_point t0) {
  const RoadNetwork& net = *cfg.network;
  const int n = net.node_count(), m = net.edge_count();
  std::vector<uint8_t> sig(n);
  for (const RoadNode& nd : net.nodes()) sig[nd.id] = nd.signalized ? 1 : 0;
  std::vector<int32_t> from(m), to(m), lanes(m);
  std::vector<int64_t> len(m);
  for (const RoadEdge& e : net.edges()) {
    from[e.id] = e.from;
    to[e.id] = e.to;
    len[e.id] = e.length_mm;
    lanes[e.id] = e.lanes;
  }
  gmaco_graph_desc g{n, m, sig.data(), from.data(), to.data(), len.data(), lanes.data()};
  const gmaco_sim_config c = to_abi(cfg);

  gmaco_engine* h = nullptr;
  if (int rc = gmaco_create(&g, &dd, &c, device, &h)) raise(rc, gmaco_last_error(nullptr));
  std::unique_ptr<gmaco_engine, void (*)(gmaco_engine*)> guard(h, gmaco_destroy);
  gmaco_run_result r{};
  if (int rc = gmaco_run(h, &r, nullptr)) raise(rc, gmaco_last_error(h));
  RunResult out;
  out.travel_times_s.assign(cfg.vehicle_count, -1.0);
  std::vector<int32_t> rvid(cfg.vehicle_count), rnode(cfg.vehicle_count);
  if (int rc = gmaco_collect(h, &r, out.travel_times_s.data(), rvid.data(), rnode.data(), cfg.vehicle_count))
    raise(rc, gmaco_last_error(h));
  out.mean_travel_s = r.mean_travel_s;
  out.mean_wait_s = r.mean_wait_s;
  out.mean_queue_len = r.mean_queue_len;
  out.max_edge_occupancy = r.max_edge_occupancy;
  out.completed_count = r.completed_count;
  out.retired_count = r.retired_count;
  out.steps_executed = r.steps_executed;
  for (int i = 0; i < r.retired_count; ++i)  // engine.cpp:416-421
    out.diagnostics.push_back("vehicle " + std::to_string(rvid[i]) + " retired unroutable at node " +
                              std::to_string(rnode[i]));
  out.wall_clock_ms =
      std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

}  // namespace

// The caller already holds the reference's dense table (run_matrix builds
// one per network, harness.cpp:332): it is handed to the engine as is.
// DistanceTable keeps its storage private, so the table is read through its
// inline accessor row by row (one strided copy, no call per entry).
RunResult gpu_run(const SimConfig& cfg, const DistanceTable& dist, int device) {
  const auto t0 = std::chrono::steady_clock::now();
  cfg.validate();
  const int n = cfg.network->node_count();
  if (dist.size() != n) throw ValidationError("gpu_run: distance table size does not match the network");
  std::vector<int64_t> d(static_cast<size_t>(n) * n);
  for (int u = 0; u < n; ++u) {
    int64_t* row = d.data() + static_cast<size_t>(u) * n;
    for (int v = 0; v < n; ++v) row[v] = dist.dist_mm(u, v);
  }
  return run_on_device(cfg, gmaco_distance_desc{GMACO_DIST_DENSE, 0, 0, d.data(), nullptr, 0, 0}, device, t0);
}

// No table: the engine computes the exact distance table itself with its
// device SSSP (DIST_DENSE with a null table), so the host never runs the
// O(n^2)-memory all_pairs_distances (net.cpp:419-437).
RunResult gpu_run(const SimConfig& cfg, int device) {
  const auto t0 = std::chrono::steady_clock::now();
  cfg.validate();
  return run_on_device(cfg, gmaco_distance_desc{GMACO_DIST_DENSE, 0, 0, nullptr, nullptr, 0, 0}, device, t0);
}

}  // namespace macosim
