/*
 * gmaco.h — C ABI of the B200-native GMACO-P engine.
 *
 * This is the drop-in boundary for the reference simulator's hot path
 * (reference = /root/reference/proj, "macosim", C++20, CPU-only).  Every entry
 * point below names the reference interface it replaces.  The ABI is plain C:
 * opaque handle, POD parameter blocks, raw pointers + sizes, int status codes,
 * no exceptions, no torch types.
 *
 *   status 0 = ok, 1 = validation error (reference ValidationError,
 *   net.hpp:24-27), 2 = runtime / CUDA error.  These mirror the CLI exit codes
 *   of the reference (tools/main.cpp:149-158).  gmaco_last_error() returns the
 *   message of the last failing call on a handle (or the last failing create).
 *
 * Units are the reference's: lengths int64 millimetres (net.hpp:17), pheromone
 * int64 micro-units (pheromone.hpp:13-21), time in whole steps of dt seconds.
 */
#ifndef GMACO_H_
#define GMACO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GMACO_ABI_VERSION 2

enum gmaco_status { GMACO_OK = 0, GMACO_EVALIDATION = 1, GMACO_ERUNTIME = 2 };

/* Algorithm (engine.hpp:17) plus the colony extension of the north star. */
enum gmaco_algorithm {
  GMACO_DIJKSTRA = 0,
  GMACO_ACO = 1,
  GMACO_MACO = 2,
  GMACO_MACO_P = 3,
  GMACO_COLONY = 4 /* K-ant ACO colonies per vehicle, best-tour argmin */
};
enum gmaco_controller { GMACO_FIXED = 0, GMACO_ADAPTIVE = 1, GMACO_PREEMPTIVE = 2 }; /* engine.hpp:18 */
enum gmaco_spawn { GMACO_ALL_AT_START = 0, GMACO_UNIFORM_WINDOW = 1 };               /* engine.hpp:19 */
enum gmaco_od { GMACO_OD_UNIFORM = 0, GMACO_OD_BLOCKS = 1 };                          /* engine.hpp:20 */
enum gmaco_deviation { GMACO_DEV_GLOBAL = 0, GMACO_DEV_EDGE_OCCUPANCY = 1 };          /* routing.hpp:12 */
enum gmaco_rng { GMACO_RNG_PHILOX = 0, GMACO_RNG_REFERENCE = 1 };
enum gmaco_deposit { GMACO_DEPOSIT_COMPLETION = 0, GMACO_DEPOSIT_BEST_TOUR = 1, GMACO_DEPOSIT_NONE = 2 };
enum gmaco_vehicle_state {                                                           /* engine.hpp:52-59 */
  GMACO_PENDING = 0, GMACO_AT_NODE = 1, GMACO_ON_EDGE = 2,
  GMACO_QUEUED = 3, GMACO_ARRIVED = 4, GMACO_RETIRED = 5
};
enum gmaco_distance_kind {
  GMACO_DIST_DENSE = 0, /* reference DistanceTable layout, row u, column v (net.hpp:84-102) */
  GMACO_DIST_GRID = 1,  /* closed-form Manhattan distance of a generate_grid network (net.cpp:208-244) */
  GMACO_DIST_TARGETS = 2 /* exact distances to a bounded destination set, computed by the engine */
};

#define GMACO_PHASES 8 /* kPhaseCount, signals.hpp:12 */

/* PheromoneParams, pheromone.hpp:23-42. */
typedef struct {
  double tau_init_lo, tau_init_hi;
  double delta_inc, delta_dec;
  double rho;
  double tau_min, tau_max;
  double aco_deposit_q;
  int32_t decrement_siblings_only;
  int32_t _pad;
} gmaco_pheromone_params;

/* SignalParams, signals.hpp:14-22. */
typedef struct {
  int32_t th_max;
  int32_t fixed_cycle_order[GMACO_PHASES];
  int32_t _pad;
  double t_max;
  double green_duration_s;
  double saturation_flow;
} gmaco_signal_params;

/* RoutingParams, routing.hpp:14-23. */
typedef struct {
  int64_t deviation_threshold;
  int32_t deviation_mode; /* gmaco_deviation */
  int32_t progress_filter;
  double aco_alpha, aco_beta;
} gmaco_routing_params;

/* Colony extension (north star; not in the reference).
 * With ants=1, hop_limit=1, rng=GMACO_RNG_REFERENCE, congestion=0,
 * deposit=GMACO_DEPOSIT_COMPLETION, congestion_evaporation=0 the colony run is
 * bit-identical to the reference Algorithm::Aco run (routing.cpp:77-115). */
typedef struct {
  int32_t ants;                   /* K ants per vehicle per iteration, >= 1 */
  int32_t hop_limit;              /* 0 = walk to the destination, h > 0 = stop after h hops */
  int32_t max_hops;               /* tour cap (0 = node_count - 1); longer tours fail */
  int32_t rng;                    /* gmaco_rng */
  int32_t congestion;             /* 1: roulette weight x 1/(1+load), tour cost len x (1+load) */
  int32_t deposit;                /* gmaco_deposit */
  int32_t congestion_evaporation; /* 1: tau <- max(tau_min, evap(tau) - dec * occupancy) */
  int32_t replan_all;             /* 1: every active vehicle's colony runs every iteration */
} gmaco_colony_params;

/* Engine implementation switches.  None changes the simulation: every
 * setting gives bit-identical results (the parity tests pin each path).
 * Zero-initialised = the production configuration.  They exist for A/B
 * measurements and for tests that exercise each alternative kernel path. */
enum gmaco_option_bits {
  GMACO_OPT_NO_QUEUE = 1u << 0,       /* general graphs: CTA-per-vehicles walker instead of the ant queue */
  GMACO_OPT_NO_SCRATCH = 1u << 1,     /* replay the winner's tour instead of keeping every ant's tour */
  GMACO_OPT_NO_TT = 1u << 2,          /* no per-target candidate rows (shared slot records + filter bitmaps) */
  GMACO_OPT_NO_ORDER = 1u << 3,       /* no walk-length / destination-major walk order */
  GMACO_OPT_NO_PREFETCH = 1u << 4,    /* no bulk L2 prefetch CTA */
  GMACO_OPT_NO_PDL = 1u << 5,         /* tail not launched as a programmatic dependent of the walk */
  GMACO_OPT_NO_SMEM = 1u << 6,        /* lattice walker reads its tables from global memory */
  GMACO_OPT_NO_BITS = 1u << 7,        /* lattice tours kept as slots instead of per-hop move bits */
  GMACO_OPT_NO_E1_WALK = 1u << 8,     /* signal stages C, D, E1 in the tail instead of beside the walk */
  GMACO_OPT_NATURAL_ROWS = 1u << 9,   /* aligned-CSR rows in node order instead of BFS order */
  GMACO_OPT_PROFILE_CREATE = 1u << 10, /* print gmaco_create phase times to stderr */
  GMACO_OPT_REDZONES = 1u << 11        /* guard bytes around every device array (gmaco_debug_check_redzones) */
};
typedef struct {
  uint32_t flags;    /* gmaco_option_bits */
  int32_t _pad;
  double sssp_delta; /* device SSSP near/far step, in mean edge lengths (0 = default 32) */
} gmaco_engine_options;

/* SimConfig, engine.hpp:29-50 (network / distance passed separately). */
typedef struct {
  int32_t algorithm;  /* gmaco_algorithm */
  int32_t controller; /* gmaco_controller */
  int32_t vehicle_count;
  int32_t spawn; /* gmaco_spawn */
  int32_t spawn_window_steps;
  int32_t od_pattern; /* gmaco_od */
  double dt_s;
  int64_t max_steps;
  uint64_t seed;
  double decision_latency_s;
  double od_bias;
  const int32_t* od_block_a;
  const int32_t* od_block_b;
  int32_t od_block_a_len, od_block_b_len;
  double speed_min_mps, speed_max_mps;
  gmaco_pheromone_params pheromone;
  gmaco_signal_params signal;
  gmaco_routing_params routing;
  gmaco_colony_params colony;
  gmaco_engine_options options; /* not in SimConfig: implementation switches, zero = production */
} gmaco_sim_config;

/* Road network as SoA: RoadNode / RoadEdge (net.hpp:29-43).  Edge i has id i;
 * node i has id i (the reference requires dense ids, net.cpp:44-63). */
typedef struct {
  int32_t node_count;
  int32_t edge_count;
  const uint8_t* signalized;      /* [node_count] */
  const int32_t* edge_from;       /* [edge_count] */
  const int32_t* edge_to;         /* [edge_count] */
  const int64_t* edge_length_mm;  /* [edge_count] */
  const int32_t* edge_lanes;      /* [edge_count] */
} gmaco_graph_desc;

/* Distance service: what the candidate filter reads (routing.cpp:16-30). */
typedef struct {
  int32_t kind;            /* gmaco_distance_kind */
  int32_t grid_rows, grid_cols;
  const int64_t* dist_mm;  /* DENSE: [n*n], dist(u,v) at u*n+v, INT64_MAX = unreachable */
  const int32_t* targets;  /* TARGETS: destination node ids (vehicles must end there) */
  int32_t target_count;
  int32_t _pad;
} gmaco_distance_desc;

/* RunResult, engine.hpp:92-107 (diagnostic strings are rebuilt by the host
 * wrapper from retired_vid / retired_node, engine.cpp:416-421). */
typedef struct {
  double mean_travel_s, mean_wait_s, mean_queue_len;
  int32_t max_edge_occupancy;
  int32_t completed_count;
  int32_t retired_count;
  int32_t _pad;
  int64_t steps_executed;
  int64_t wall_clock_ms;
} gmaco_run_result;

/* Vehicle snapshot (Vehicle, engine.hpp:61-90); any pointer may be NULL. */
typedef struct {
  int32_t *origin, *dest;
  double* speed_mps;
  int64_t* advance_mm;
  uint8_t* state;
  int32_t *at_node, *on_edge;
  int64_t *progress_mm, *overshoot_mm;
  int32_t* queued_phase;
  int64_t *queue_joined_step, *depart_step, *arrive_step, *latency_debt_us;
  int64_t *driving_steps, *queued_steps, *latency_steps;
  int32_t *decisions, *deviations;
  int64_t* path_length_mm;
} gmaco_vehicle_view;

/* Signal snapshot (SignalState, signals.hpp:39-52); any pointer may be NULL.
 * Per-phase arrays are [signal_count * 8]; queue_vid lists every queue FIFO
 * head-to-tail, signal-major then phase, sized by the sum of queue_len. */
typedef struct {
  int32_t* node;
  int32_t *green, *cycle_cursor, *discharge_lanes;
  int64_t* green_elapsed_steps;
  double* green_elapsed_s;
  int32_t* queue_len;
  double *head_wait_s, *service_remainder;
  int32_t* queue_vid;
  int64_t* queue_enqueue_step;
} gmaco_signal_view;

/* Device work counters (the bench metric's units). */
typedef struct {
  int64_t ant_steps;       /* next-hop selections (routing.cpp:16-115 equivalents) */
  int64_t vehicle_routes;  /* complete best-of-K tours constructed */
  int64_t decisions;       /* engine routing decisions (StepDecision count) */
  int64_t candidates;      /* filtered candidates visited (sum of c) */
  int64_t degree_sum;      /* out-edges scanned (sum of d) */
  int64_t kernels_per_step; /* engine kernels launched per step (this configuration) */
  int64_t walk_bytes;      /* algorithmic bytes read by the stage-B walks so far */
} gmaco_counters;

typedef struct gmaco_engine gmaco_engine;

/* Library version / ABI check. */
int32_t gmaco_abi_version(void);

/* Builds the device world: CSR road graph, distance service, pheromone field,
 * signal states, fleet.  Replaces init_world (engine.cpp:116-144) +
 * spawn_vehicles (engine.cpp:71-114) + RoadNetwork validation (net.cpp:38-98).
 * `device` is the CUDA ordinal. */
int gmaco_create(const gmaco_graph_desc* graph, const gmaco_distance_desc* dist,
                 const gmaco_sim_config* cfg, int32_t device, gmaco_engine** out);

/* Multi-GPU: shard the fleet across `world` ranks (partition_entities,
 * parallel.cpp:8-21) and exchange the per-step vectors over NCCL.  `nccl_id`
 * is the 128-byte ncclUniqueId of rank 0.  Call before the first step.
 * Engines of one process attaching with the same (device, rank, world, id)
 * share one communicator: the first attach creates it (ncclCommInitRank),
 * later ones reuse it; communicators live until process exit. */
int gmaco_attach_comm(gmaco_engine* h, int32_t rank, int32_t world, const void* nccl_id);
int gmaco_nccl_unique_id(void* out128);

/* Host-mediated sharding (tests, or a caller with its own transport): this
 * engine plans vehicles [lo, hi) only (every algorithm: colonies, and the
 * reference's dijkstra / aco / maco / maco-p, whose MACO fold is replicated
 * from the exchanged decisions, parallel.cpp:195-258).  Per step:
 * gmaco_step_split(h, 1) (stage B over the shard); gmaco_exchange_export (the
 * shard's decision records [hi-lo] — edge id taken, with GMACO_REC_DEVIATED
 * set for a MACO deviation, -1 none, -2 retired — and its best-tour
 * deposits per edge id [edge_count]); combine across shards (concatenate
 * the records in vehicle order, sum the deposits); gmaco_exchange_import
 * ([vehicle_count] records, [edge_count] deposit sums); then
 * gmaco_step_split(h, 2) (apply the remote decisions, stages C..G). */
#define GMACO_REC_DEVIATED (1 << 30) /* decision record flag: a MACO deviation (RouteDecision::deviated) */
int gmaco_set_shard(gmaco_engine* h, int32_t lo, int32_t hi);
/* By-target shards (worlds with per-target candidate rows: TARGETS
 * distances, ant-queue walker): this engine plans the vehicles bound for the
 * destination targets dealt to `rank` (targets by vehicle count, largest
 * first, each to the least-loaded rank; identical on every rank), refreshes
 * only those targets' tables and keeps its walk destination-major.
 * gmaco_attach_comm picks this form by itself for such worlds.  With it,
 * gmaco_exchange_export returns the shard's records in the order
 * gmaco_shard_vehicles lists its vehicles (*n = shard size; vids written
 * when cap >= *n). */
int gmaco_shard_by_target(gmaco_engine* h, int32_t rank, int32_t world);
int gmaco_shard_vehicles(gmaco_engine* h, int32_t* vids, int32_t cap, int32_t* n);
int gmaco_step_split(gmaco_engine* h, int32_t part);
int gmaco_exchange_export(gmaco_engine* h, int32_t* decisions, int64_t* deposits);
int gmaco_exchange_import(gmaco_engine* h, const int32_t* decisions, const int64_t* deposits);

/* Executes up to `steps` engine steps (sequential_step, engine.cpp:352-400),
 * stopping early once finished() (engine.cpp:146-152) holds.  `executed`
 * (may be NULL) receives the number of steps run.  With executed == NULL the
 * call returns once the steps are enqueued on the engine's stream (steps past
 * finished() are no-ops); every later read (gmaco_get_*, gmaco_collect, ...)
 * is ordered after them. */
int gmaco_step(gmaco_engine* h, int64_t steps, int64_t* executed);
/* finished(w) (engine.cpp:146-152). */
int gmaco_finished(gmaco_engine* h, int32_t* out);
/* run(cfg, dist) (engine.cpp:435-444) / parallel_run(cfg, dist, workers)
 * (parallel.cpp:276-285): steps to completion and collects. */
int gmaco_run(gmaco_engine* h, gmaco_run_result* result, double* travel_times_s);
/* collect_result (engine.cpp:402-433).  travel_times_s is [vehicle_count] (or
 * NULL); retired_* receive up to retired_cap entries in vid order. */
int gmaco_collect(gmaco_engine* h, gmaco_run_result* result, double* travel_times_s,
                  int32_t* retired_vid, int32_t* retired_node, int32_t retired_cap);

/* State snapshots for stage-level parity. */
int gmaco_get_pheromone(gmaco_engine* h, int64_t* tau_micros /* [edge_count], edge-id order */);
int gmaco_set_pheromone(gmaco_engine* h, const int64_t* tau_micros);
int gmaco_get_occupancy(gmaco_engine* h, int32_t* occupancy /* [edge_count] */);
int gmaco_get_vehicles(gmaco_engine* h, const gmaco_vehicle_view* view);
int gmaco_get_signals(gmaco_engine* h, const gmaco_signal_view* view, int64_t queue_cap);
/* Double-buffered vehicle readback: gmaco_vehicles_enqueue snapshots the
 * fields a view requests (non-NULL pointers; their values are not read) of
 * the state after every step enqueued so far into internal pinned slot 0 or
 * 1, without waiting; gmaco_vehicles_wait blocks for that snapshot only and
 * copies it into `view` (same field set).  A caller reads every step's result
 * while the next step already runs (gmaco_step with executed == NULL). */
int gmaco_vehicles_enqueue(gmaco_engine* h, const gmaco_vehicle_view* fields, int32_t slot);

/* gmaco_step(h, 1, NULL) followed by gmaco_vehicles_enqueue(h, fields, slot),
 * enqueued as ONE graph launch (the step and the snapshot gather captured
 * together per slot); read the snapshot with gmaco_vehicles_wait. */
int gmaco_step_snapshot(gmaco_engine* h, const gmaco_vehicle_view* fields, int32_t slot);
int gmaco_vehicles_wait(gmaco_engine* h, int32_t slot, const gmaco_vehicle_view* view);
int gmaco_signal_count(gmaco_engine* h, int32_t* out);
int gmaco_get_counters(gmaco_engine* h, gmaco_counters* out);
int gmaco_current_step(gmaco_engine* h, int64_t* out);

/* Per-vehicle route query: the vehicle's realized path (path_edges,
 * engine.hpp:88) when planned == 0, or its current best-of-K planned tour from
 * the last colony iteration when planned == 1 (colony algorithm only). */
int gmaco_route_query(gmaco_engine* h, int32_t vid, int32_t planned, int32_t* out_edges,
                      int32_t cap, int32_t* out_len);

/* Batched next-hop selection over the engine's current pheromone field and
 * occupancy: next_node_dijkstra / next_node_aco / next_node_maco
 * (routing.hpp:52-73).  For ACO, rng_entity[i] / rng_step[i] form the RngKey
 * (routing.hpp:33-37).  Unroutable entries return next = via = -1. */
int gmaco_next_node(gmaco_engine* h, int32_t algorithm, int32_t count, const int32_t* current,
                    const int32_t* dest, const uint64_t* rng_entity, const uint64_t* rng_step,
                    int64_t n_t, int32_t* out_next, int32_t* out_via, uint8_t* out_deviated);

/* Device event timing of the last gmaco_step call's kernels (ms): walk
 * kernel total and whole-step total.  Recorded only while timing is enabled
 * (gmaco_set_timing), since every event serializes the stream (~2-3 us). */
int gmaco_last_timing(gmaco_engine* h, double* walk_ms, double* step_ms, int64_t* walk_launches);
int gmaco_set_timing(gmaco_engine* h, int32_t enabled);
/* Profiling hook: runs `steps` steps and returns the last one's stage
 * timestamps (ns, %globaltimer, 16 slots; see DevCtl::trace in
 * paper_2010_14244_b200/csrc/device.cuh). */
int gmaco_debug_trace(gmaco_engine* h, int32_t steps, uint64_t* out16);
/* Memory check of a world created with GMACO_OPT_REDZONES: settles the
 * stream and verifies every guard band around the engine's device arrays.
 * *corrupted receives the number of overwritten guards (0 = no out-of-bounds
 * write reached one); gmaco_last_error describes the first. */
int gmaco_debug_check_redzones(gmaco_engine* h, int64_t* corrupted);
/* Test hook of the lattice walker's roulette (LatRec in
 * paper_2010_14244_b200/csrc/device.cuh): for each pair of candidate weights
 * (wa first, wb second) the integer threshold thr such that the sequential
 * roulette of routing.cpp:100-113 over {wa, wb} with u = k * 2^-53 picks the
 * first candidate iff k < thr. */
int gmaco_debug_roulette_threshold(gmaco_engine* h, int32_t count, const double* wa, const double* wb,
                                   uint64_t* out);
/* Benchmark entry point: enqueues `steps` engine steps without host
 * synchronization (one CUDA graph per step), with an L2-flushing memset of
 * flush_bytes before each step outside the timed span; returns per-step
 * device times.  Pass step_ms only (events: begin, end of step), walk_ms only
 * (begin, end of the stage-B walk; the rest of the step runs untimed), or
 * both (three events; each event node costs ~2-3 us of serialization). */
int gmaco_bench_steps(gmaco_engine* h, int32_t steps, int64_t flush_bytes, double* walk_ms, double* step_ms);

/* ---- reference-schema network files --------------------
 * load_network / load_network_file (R/src/net.cpp:112-175): parse
 * {"nodes": [{"id","signalized","x"?,"y"?}], "edges": [{"id","from","to",
 * "length_m","lanes"}]} with the reference's checks and messages (status 1),
 * ids dense and sorted as the RoadNetwork ctor (net.cpp:38-98) leaves them;
 * length_mm = llround(length_m * 1000) (net.cpp:34).  The opaque handle owns
 * the parsed SoA arrays; gmaco_network_export copies them into caller buffers
 * sized by gmaco_network_info (any pointer may be NULL). */
typedef struct gmaco_network gmaco_network;
int gmaco_network_parse(const char* text, size_t len, gmaco_network** out);
int gmaco_network_load_file(const char* path, gmaco_network** out);
int gmaco_network_info(const gmaco_network* net, int32_t* node_count, int32_t* edge_count);
int gmaco_network_export(const gmaco_network* net, uint8_t* signalized, int32_t* edge_from, int32_t* edge_to,
                         int64_t* edge_length_mm, int32_t* edge_lanes, double* x_m, double* y_m,
                         uint8_t* has_position);
void gmaco_network_free(gmaco_network* net);
/* serialize_network / write_network_file (net.cpp:179-209): the same text as
 * nlohmann::json::dump(2) of the reference document.  serialize: *len gets the
 * text length; the text is written only when cap >= *len.  Positions are
 * optional (NULL x/y: none; has_position NULL: all present). */
int gmaco_network_serialize(const gmaco_graph_desc* g, const double* x_m, const double* y_m,
                            const uint8_t* has_position, char* buf, size_t cap, size_t* len);
int gmaco_network_write_file(const gmaco_graph_desc* g, const double* x_m, const double* y_m,
                             const uint8_t* has_position, const char* path);
const char* gmaco_network_last_error(void);

const char* gmaco_last_error(const gmaco_engine* h);
void gmaco_destroy(gmaco_engine* h);

#ifdef __cplusplus
}
#endif

#endif /* GMACO_H_ */
