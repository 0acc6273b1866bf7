// device.cuh — device-side world layout of the GMACO-P engine (sm_100a).
//
// Everything edge-indexed on the device is stored in CSR SLOT order: the
// out-edges of node x occupy slots [row[x].x, row[x].x + row[x].y), sorted
// by neighbour id exactly like RoadNetwork::out_edges (net.hpp:64-66,
// net.cpp:85-93).  A node's candidate row is therefore one contiguous run of
// columns / weights / lengths, and edge ids (the reference's numbering)
// appear only at the boundary through slot_edge / edge_slot.
#pragma once

#include <cstdint>

namespace gmaco {

constexpr int kPhases = 8;
constexpr int kMaxDegree = 32;  // out-degree bound of the walk kernels (validated at create)
constexpr int kTabu = 16;       // colony tabu tenure (progress filter off only)
constexpr int64_t kInf = INT64_MAX;

enum VState : uint8_t { kPending = 0, kAtNode = 1, kOnEdge = 2, kQueued = 3, kArrived = 4, kRetired = 5,
                        // released by this step's E1 while stage B runs (DevParams::e1_in_walk): Queued for
                        // B, AtNode for everything after it; the tail turns it into kAtNode
                        kReleased = 6 };

struct DevGraph {
  int32_t n, m;
  int32_t ell;              // ELL row width (4 or 8; slot = x*ell + i) or 0 for plain CSR
  int32_t M;                // slot-space size (n*ell for ELL, m for CSR); padding slots have slot_edge = -1
  const int2* row;          // [n] {first slot, row span} (span = ELL width, or out-degree for CSR)
  const int32_t* deg;       // [n] out-degree
  const int32_t* key;       // [M] colony fast path: packed grid (row<<16|col) of the neighbour, or
                            //     the neighbour id for table distances; -1 on padding
  const int32_t* col;       // [m] neighbour (edge.to) per slot
  const int64_t* len;       // [m] length_mm per slot
  const int32_t* bind;      // [m] signal*8+phase of the queue the edge feeds, -1 if none
  const int32_t* slot_edge; // [m] reference edge id per slot
  const int32_t* slot_from; // [m] edge.from per slot
  const double* eta_beta;   // [m] pow(1/(len/1000), beta), host std::pow (routing.cpp:92-94)
  const int2* nrow;         // [M] general-graph walker: {first, span | deg << 8} of col[slot]'s row
};

// Distance service read by the candidate filter (routing.cpp:16-30).
struct DevDist {
  int32_t kind;        // 0 dense / 2 targets: table; 1 grid closed form
  int32_t rows, cols;  // grid
  int64_t grid_len;    // grid edge length
  int32_t n;
  const int64_t* table;    // [slot * n + x] = dist(x, dest of slot), kInf unreachable
  const int32_t* slot_of;  // node -> table row (targets), nullptr = identity (dense)
  // Progress-filter bitmaps (general-graph walker): per table row t and slot
  // word, the closer bit of slot s = dist_t(col[s]) < dist_t(from[s]) with
  // dist_t(col[s]) != inf (routing.cpp:16-30 evaluated ahead of time, exact
  // int64 comparisons); fbw words per row incl. one padding word.  No reach
  // bits: with every edge length > 0 (net.cpp:74-75) a node x != dest with a
  // finite distance always has a strictly closer out-neighbour (the next node
  // of a shortest path), and from an infinite-distance node no neighbour is
  // reachable either, so candidate_neighbors' fallback (routing.cpp:24-29)
  // never changes the candidate set of a walk.
  const uint32_t* fbits;
  int64_t fbw;
};

struct DevParams {
  int32_t algorithm, controller, deviation_mode, progress_filter;
  int32_t V, S;
  int64_t deviation_threshold;
  double alpha;
  double dt_s;
  int64_t dt_us, latency_us;
  int64_t max_steps;
  uint64_t seed;
  // pheromone (micro-units)
  int64_t tau_lo, tau_hi, inc, dec;
  double one_minus_rho;  // (1.0 - rho), same expression as pheromone.cpp:64
  double deposit_q;
  int32_t siblings_only;
  // signals
  int32_t th_max;
  double t_max, green_duration_s, saturation_flow;
  int32_t order[kPhases];
  // colony
  int32_t ants, hop_limit, max_hops, rng, congestion, deposit, cong_evap, replan_all;
  int32_t plan_cap, path_cap;
  int32_t scratch_mode;     // 1: every ant's tour kept in scratch, the plan is the winner's row
  int32_t need_positions;  // MACO network-wide fold
  int32_t prefetch;        // bulk-prefetch the step's state into L2 at the start of stage B
  uint32_t rk[20];         // Philox4x32-10 round keys of `seed` (host key schedule)
  // vehicle sharding (multi-GPU): this rank plans vehicles [shard_lo, shard_hi);
  // the others' decisions arrive through the exchange (k_apply_remote)
  int32_t shard_lo, shard_hi, sharded;
  int32_t rank;          // this rank (by-target sharding: DevVehicles::owner)
  int32_t no_smem;          // A/B switch: read the walk tables from global memory
  int32_t grid_bits;        // lattice walker keeps tours as per-hop move bits (SMEM words)
  int32_t bit_words;        // 64-hop move-bit words per ant (ceil(plan_cap / 64))
  int32_t max_degree;       // largest out-degree (general-graph walker bound)
  int32_t csr_walker;       // colony runs on k_colony_csr (bitmaps + nrow built)
  int32_t ant_queue;        // csr walker in scratch mode: prologue / ant-queue walk / epilogue kernels
  int32_t pdl;              // cooperative tail launched as a programmatic dependent of the walk
  int32_t record_paths;
  // lattice colony walks: stages C, D, E1 run in extra CTAs of the walk kernel,
  // concurrently with B (they read only the previous step's signal state, and
  // a vehicle E1 releases stays Queued for B: kReleased); the tail does E3, F+G
  int32_t e1_in_walk;
};

// Control block.  The read-mostly step state shares one cache line; every
// counter that blocks update atomically lives on its own 128-byte line, so
// the per-block counter flushes of one stage neither serialize against each
// other in one L2 slice nor stall the next kernel's read of `done`/`step`.
struct DevCtl {
  int64_t step;        // w.step
  int64_t stop_at;     // host-set step limit for the current launch chunk
  int64_t n_t;         // count_active for the current step (engine.cpp:156-173)
  int64_t qsamples;
  int32_t done;
  int32_t max_occ;
  int32_t error;       // device-side overflow flag (path buffer)
  int32_t trace_on;
  alignas(128) int64_t n_next;      // accumulated for the next step
  alignas(128) int64_t unfinished;  // vehicles not Arrived/Retired after motion
  alignas(128) int64_t dcount;      // decisions this step
  alignas(128) int64_t qtotal;
  alignas(128) int64_t ant_steps;
  alignas(128) int64_t vehicle_routes;
  alignas(128) int64_t decisions;
  alignas(128) int64_t candidates;
  alignas(128) int64_t degree_sum;
  alignas(128) uint32_t blocks_done;
  alignas(128) int32_t nrel;          // vehicles released by a concurrent E1 this step (DevVehicles::rel)
  alignas(128) unsigned long long q_walkers;  // ant queue: walking vehicles this step
  unsigned long long q_next;                  // ant queue: next (vehicle, ant) item
  alignas(128) int32_t max_occ_acc;  // atomicMax target of stage F+G
  // stage trace of the current step (%globaltimer ns; written when trace_on
  // is set): [0] walk start (min), [1] walk staging done (max), [2] walk end
  // (max), [3] tail start (min), [4]/[7]-[15] probes, [5] signals done,
  // [6] F+G done
  alignas(128) unsigned long long trace[16];
};

struct DevVehicles {
  int32_t *origin, *dest;
  int64_t* advance;
  uint8_t* state;
  int32_t *at_node, *on_edge;  // on_edge is a SLOT
  int64_t *progress, *overshoot;
  int32_t* queued_phase;
  int64_t *joined, *depart, *arrive, *latency_debt;
  int64_t *driving, *queued, *lat_steps, *path_len_mm;
  int32_t *decisions, *deviations;
  int32_t* qnext;     // FIFO link inside a signal queue
  int32_t* arr_next;  // this step's arrival stack link
  int32_t* dec_next;  // this step's decision stack link (MACO fold)
  int32_t* dflag;     // decided this step (MACO positions)
  int32_t* pos;       // exclusive prefix of dflag = decision position
  int32_t* bsum;      // [cooperative tail blocks] decisions per tail block's vehicle chunk (pos scan)
  int32_t *path, *path_n;       // realized path (slots), [V * path_cap]
  int32_t *plan, *plan_n;       // best planned tour (slots), [V * plan_cap] (replay mode)
  int32_t* scratch;             // [V * ants * plan_cap] every ant's tour (scratch mode)
  int32_t* plan_ant;            // winning ant per vehicle (scratch mode)
  const int32_t* walk_order;    // walk slot -> vehicle (walk-length balanced / destination-major; a shard's
                                //     own vehicles at slots [shard_lo, shard_hi)), or nullptr
  const int16_t* owner;         // by-target sharding: [V] rank planning each vehicle (nullptr: the
                                //     contiguous range [shard_lo, shard_hi) is this rank's)
  // ant-queue walker (general graphs, scratch mode): per-vehicle walk start
  // (-1 = not walking), deciding flag, packed (cost, ant) argmin key, the
  // walking-vehicle list the queue indexes, and per-ant hop counts
  int32_t* walk_start;
  uint8_t* walk_dec;
  unsigned long long* best_key;
  int32_t* walkers;
  int32_t* ant_hops;            // [V * ants] hops, -1 when the first hop had no candidate
  int32_t* dec_rec;             // [V_pad] this step's decision per vehicle: slot, -1 none, -2 retired
  int32_t* rel;                 // [V] vehicles released by a concurrent E1 this step (e1_in_walk)
  int64_t* plan_step;
  uint8_t* plan_done;
};

struct DevSignals {
  int32_t* node;
  int32_t *green, *cursor, *lanes;
  int64_t* el_steps;
  double* el_s;
  // per queue [S*8]
  int32_t *qlen, *qhead, *qtail, *arr_head;
  double *head_wait, *rem;
  // e1_in_walk: queue lengths after this step's E1 [S*8] and this step's
  // arrivals per queue [2][S*8] (step-parity double buffer), so stage F+G's
  // congestion load qlen-after-E3 = qlen_e1 + arrivals needs no E3 result
  int32_t *qlen_e1, *arr_cnt;
};

// Per-target candidate rows (ant-queue walker with a bounded destination set,
// GMACO_DIST_TARGETS).  For target t and node x, x's row holds only the
// candidate_neighbors of x toward t (routing.cpp:16-30: out-slots whose head is
// strictly closer, kept in slot = ascending-neighbour order), one 16-B record
// per candidate {weight f64, int32 edge cost, head row meta}, padded to pairs
// (one LDG.256 covers a row of <= 2 candidates).  Row meta = off << 8 | c << 4 |
// deg with off the row's pair offset inside t's table, c the candidate count,
// deg the out-degree (counters).  Every row, including a candidate-free one,
// owns at least one pair, so a meta identifies its node.  Records 0-1 are a
// zero row (meta 0).  Weight and cost halves are refreshed from the shared slot
// records at the start of each step.
struct DevTT {
  int4* rec;             // [nrec] records
  const int2* sm;        // [nrec] {slot (-1 padding), head row meta}
  const int2* sl;        // [nrec] {slot, len_mm} for the epilogue (nullptr when a length >= 2^31)
  const uint32_t* meta;  // [T * n] row meta of node x in target t's table
  const int64_t* base;   // [T] first record of target t's table
  const int64_t* cstart; // [T * (nch + 1)] first record of each kTTChunk-row chunk (+ table end)
  int64_t nrec;
  int32_t T, nch;
  const int32_t* own_t;  // by-target sharding: the T_own tables this rank refreshes (nullptr: all T)
  int32_t T_own;
};
constexpr int kTTChunk = 1024;  // rows per refresh chunk

// Batched gather of device arrays into (mapped pinned) host memory.
struct PackField {
  const void* src;
  void* dst;  // device-visible pointer
  size_t bytes;
};
struct PackDesc {
  PackField f[24];
  int n = 0;
};

// Lattice walker record of one (node, walk quadrant): everything a hop needs
// in one 16-B load.  On a uniform lattice a walk toward its destination has
// at most two candidates (one vertical, one horizontal move) whose order and
// slots are fixed by the quadrant q = 2*(rows grow) + (cols grow).  The
// sequential roulette (routing.cpp:100-113) picks the first candidate iff
// fl(u * (w_a + w_b)) < w_a with u = k * 2^-53 (k = the draw's top 53 bits);
// that predicate is monotone in k, so it is exactly "k < thr" for an integer
// threshold tabulated once per step by stage F+G (lattice_threshold).  The
// non-finite / non-positive total case (uniform pick, "second iff u >= 1/2")
// is thr = 2^52.  lv / lh are the congestion loads of the vertical and
// horizontal slot: their edge costs are len * (1 + load) (slot_fg), so a
// walk's tour cost is len * (hops + the sum of its loads).
struct __align__(16) LatRec {
  unsigned long long thr;
  int32_t lv, lh;
};

struct DevWorld {
  DevGraph g;
  DevTT tt;
  DevDist d;
  DevParams p;
  DevVehicles v;
  DevSignals s;
  DevCtl* ctl;
  int64_t* tau;       // [m] pheromone micro-units (slot order)
  double* weight;     // [m] roulette weight for the coming step
  int4* rec;          // [M] ant-queue walker slot records {weight, head node, head row}; weight half
                      //     rewritten with `weight` (nullptr unless p.ant_queue)
  int64_t* ecost;     // [m] colony tour cost per edge for the coming step
  int32_t* ecost32;   // [M] int32 copy for the lattice walker's SMEM staging when
                      //     max len * (1 + V) < 2^31 (nullptr otherwise)
  LatRec* lrec;       // lattice walker records (nullptr unless the lattice walker runs):
                      //   lrec_stride == 0 (staged in SMEM): [4 n], index 4 * node + quadrant;
                      //   else four quadrant tables of lrec_stride records in diagonal-major
                      //   order (lrec_index), so the ants of one colony, which stand on one
                      //   diagonal at every hop, read neighbouring records
  int32_t* occ_cur;   // [m] edge occupancy of the previous step (engine.hpp:166)
  int32_t* occ_new;   // [m] being accumulated this step
  int64_t* dep;       // [m] ACO / best-tour deposit accumulator (exact int64 sums)
  int32_t* dec_head;  // [m] decision stack per slot (network-wide MACO) or per node (scoped)
  const int64_t* dep_amount;  // lattice: deposit_amount(h * edge length) for h = 0..plan_cap (host-computed)
  // tau^alpha for alpha not in {0, 1}: [tau_hi - tau_lo + 1] entries
  // pow(t / 1e6, alpha) for every reachable pheromone value t (the field is
  // clamped to [tau_lo, tau_hi] by every update), computed once by the host's
  // glibc pow, the function routing.cpp:93 calls, so the device weights are
  // bit-identical to the reference's; nullptr otherwise
  const double* taupow;
  // gmaco_step_snapshot of small worlds: the step's finalizing block gathers
  // these fields after the step (device copy of the slot's descriptor), in
  // place of a separate k_pack launch; nullptr for plain steps
  const PackDesc* snap;
  // (appended last: the hot kernels' parameter layout stays as it was)
  int32_t lrec_stride;  // see lrec
  int32_t pad_;
  uint64_t cols_magic;  // grid: ceil(2^64 / cols); x / cols = umul64hi(x, cols_magic) for 0 <= x < 2^31
};

// LatRec position of (node x, quadrant q).  Diagonal-major tables: every
// hop of a walk in quadrant q moves to the next diagonal -- key r + c when
// rows and cols change in the same sense (q = 0, 3), r - c + cols - 1
// otherwise -- so within a table the index is key * rows + r and a hop adds
// dr * rows (horizontal) or dr * (rows + 1) (vertical).
__device__ __forceinline__ int32_t lrec_index(const DevWorld& w, int32_t x, int q) {
  if (!w.lrec_stride) return 4 * x + q;
  const int32_t cols = w.d.cols, rows = w.d.rows;
  const int32_t r = (int32_t)__umul64hi((unsigned long long)x, w.cols_magic), c = x - r * cols;
  const int32_t key = (q == 0 || q == 3) ? r + c : r - c + cols - 1;
  return q * w.lrec_stride + key * rows + r;
}

// pow(tau_to_double(t), alpha) (routing.cpp:91-93; tau_to_double pheromone.hpp:19)
__device__ __forceinline__ double tau_alpha(const DevWorld& w, int64_t t) {
  const double a = w.p.alpha;
  if (a == 1.0) return __ddiv_rn((double)t, 1e6);
  if (a == 0.0) return 1.0;
  if (w.taupow) return w.taupow[t - w.p.tau_lo];
  return pow(__ddiv_rn((double)t, 1e6), a);  // table too large: device pow, <= 1 ulp
}

}  // namespace gmaco
