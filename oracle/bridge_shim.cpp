// bridge_shim.cpp — TEST INFRASTRUCTURE ONLY: runs the reference run() and
// the integration executor gpu_run() (integration/macosim_gpu.cpp) on the
// same SimConfig and reports RunResult::identical_to (engine.cpp:34-40).
#include <string>

#include "gmaco.h"
#include "macosim/engine.hpp"
#include "macosim_gpu.hpp"

namespace macosim {
// provided by ref_shim.cpp
}

extern "C" {
// 1 identical, 0 different, -1 error (message via bridge_last_error)
static thread_local std::string g_bridge_err;
const char* bridge_last_error(void) { return g_bridge_err.c_str(); }

int bridge_identical(const gmaco_graph_desc* gd, int algorithm, int vehicles, uint64_t seed, int device) {
  using namespace macosim;
  try {
    std::vector<RoadNode> nodes(gd->node_count);
    for (int i = 0; i < gd->node_count; ++i) nodes[i] = RoadNode{i, gd->signalized[i] != 0, false, 0, 0};
    std::vector<RoadEdge> edges(gd->edge_count);
    for (int i = 0; i < gd->edge_count; ++i)
      edges[i] = RoadEdge{i, gd->edge_from[i], gd->edge_to[i], gd->edge_length_mm[i], gd->edge_lanes[i]};
    RoadNetwork net(std::move(nodes), std::move(edges));
    SimConfig cfg;
    cfg.network = &net;
    cfg.algorithm = static_cast<Algorithm>(algorithm);
    cfg.controller = cfg.algorithm == Algorithm::MacoP ? ControllerKind::Preemptive : ControllerKind::Fixed;
    cfg.vehicle_count = vehicles;
    cfg.seed = seed;
    DistanceTable dist = all_pairs_distances(net);
    RunResult a = run(cfg, dist);
    RunResult b = gpu_run(cfg, dist, device);
    return a.identical_to(b) ? 1 : 0;
  } catch (const std::exception& e) {
    g_bridge_err = e.what();
    return -1;
  }
}
}
