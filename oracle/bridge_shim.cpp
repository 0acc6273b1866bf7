// bridge_shim.cpp — TEST INFRASTRUCTURE ONLY: runs the reference run() and
// the integration executor gpu_run() (integration/macosim_gpu.cpp) on the
// same SimConfig and reports RunResult::identical_to (engine.cpp:34-40); and
// drives the reference harness patched with the "gpu" executor
// (harness_gpu.patch): load_scenario -> run_matrix -> write_results_csv.
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <fstream>
#include <sstream>
#include <string>

#include "gmaco.h"
#include "macosim/engine.hpp"
#include "macosim/harness.hpp"
#include "macosim_gpu.hpp"

namespace {
// a crash inside the bridged code prints its native stack (the test log is
// the only trace the GPU box returns)
void bridge_segv(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  const char msg[] = "bridge: fatal signal, native stack:\n";
  (void)!write(2, msg, sizeof msg - 1);
  backtrace_symbols_fd(frames, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
struct SegvHook {
  SegvHook() { signal(SIGSEGV, bridge_segv); }
} segv_hook;
}  // namespace

extern "C" {
// 1 identical, 0 different, -1 error (message via bridge_last_error)
static thread_local std::string g_bridge_err;
const char* bridge_last_error(void) { return g_bridge_err.c_str(); }

// with_table = 1: gpu_run(cfg, dist, device) with the reference's dense
// table; 0: gpu_run(cfg, device), the engine builds the table on the device.
int bridge_identical(const gmaco_graph_desc* gd, int algorithm, int vehicles, uint64_t seed, int device,
                     int with_table) {
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
    RunResult b = with_table ? gpu_run(cfg, dist, device) : gpu_run(cfg, device);
    return a.identical_to(b) ? 1 : 0;
  } catch (const std::exception& e) {
    g_bridge_err = e.what();
    return -1;
  }
}

// The reference harness end to end: scenario JSON text -> load_scenario ->
// load_scenario_network -> run_matrix (executors as the scenario lists them)
// -> write_results_csv_file(csv_path) -> read_results_csv_file round trip ->
// emit_report into report_path.  Returns the row count (the round trip must
// reproduce it) or -1 with the message in bridge_last_error; failed cells are
// reported as an error too.
int bridge_run_matrix(const char* scenario_json, const char* csv_path, const char* report_path, int workers) {
  using namespace macosim;
  try {
    Scenario sc = load_scenario(scenario_json);
    RoadNetwork net = load_scenario_network(sc);
    ResultTable t = run_matrix(sc, net, workers, nullptr);
    if (!t.failures().empty()) {
      g_bridge_err = "run_matrix failures: " + t.failures().front();
      return -1;
    }
    write_results_csv_file(t, csv_path);
    ResultTable back = read_results_csv_file(csv_path);
    if (back.rows().size() != t.rows().size()) {
      g_bridge_err = "results csv round trip changed the row count";
      return -1;
    }
    std::ofstream rep(report_path);
    std::ostringstream data;
    emit_report(back, rep, data);
    rep << "\n" << data.str();
    return static_cast<int>(t.rows().size());
  } catch (const std::exception& e) {
    g_bridge_err = e.what();
    return -1;
  }
}

// load_scenario's validation alone (status 1 + message on a bad scenario).
int bridge_load_scenario(const char* scenario_json) {
  try {
    macosim::load_scenario(scenario_json);
    return 0;
  } catch (const std::exception& e) {
    g_bridge_err = e.what();
    return 1;
  }
}
}
