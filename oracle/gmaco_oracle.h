/* gmaco_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference hot path (see gmaco_oracle.c for
 * the per-function reference citations).  It is the checker the parity tests
 * compare the CUDA engine against; nothing in the product links it. */
#ifndef GMACO_ORACLE_H_
#define GMACO_ORACLE_H_

#include <stdint.h>

#include "gmaco.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct og_world og_world;

/* rng.hpp:21-56 */
uint64_t og_mix64(uint64_t x);
uint64_t og_draw(uint64_t seed, uint64_t a, uint64_t b, uint64_t c);
double og_to_unit(uint64_t bits);
double og_uniform(uint64_t bits, double lo, double hi);
uint64_t og_below(uint64_t bits, uint64_t n);
/* Philox4x32-10 (Salmon et al., SC'11): counter (c0..c3), key (k0,k1). */
void og_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* The ant uniform: GMACO_RNG_PHILOX or GMACO_RNG_REFERENCE keying. */
double og_ant_uniform(int rng, uint64_t seed, int64_t step, int32_t vid, int32_t ant, int32_t hop);

/* pheromone.cpp / parallel.cpp */
int64_t og_tau_from_double(double v);
int64_t og_evaporate_one(int64_t tau, const gmaco_pheromone_params* p);
int64_t og_deposit_amount(int64_t len_mm, const gmaco_pheromone_params* p);
int64_t og_fold_maco_edge(int64_t tau, const int32_t* pos, int32_t n, int64_t total,
                          const gmaco_pheromone_params* p);

/* signals.cpp: kind 0 fixed, 1 adaptive, 2 preemptive */
int og_select_phase(int kind, const int32_t* qlen, const double* head_wait, int cursor,
                    const gmaco_signal_params* p);
/* one discharge on a green queue of qlen vehicles; returns released count */
int og_discharge(int32_t qlen, double* remainder, double dt, int lanes, const gmaco_signal_params* p);

/* net.cpp */
int og_validate_graph(const gmaco_graph_desc* g, char* err, int32_t errcap);
int og_generate_grid(int rows, int cols, double len_m, int lanes, int sig_interior, int sig_all,
                     uint8_t* signalized, int32_t* from, int32_t* to, int64_t* len_mm, int32_t* lanes_out);
int og_apsp(const gmaco_graph_desc* g, int64_t* dist, int32_t* next);
int og_dijkstra_to(const gmaco_graph_desc* g, int32_t dst, int64_t* dist_to);

/* world: init_world + sequential_step + collect_result (engine.cpp) */
og_world* og_world_create(const gmaco_graph_desc* g, const gmaco_distance_desc* d,
                          const gmaco_sim_config* c, char* err, int32_t errcap);
void og_world_destroy(og_world* w);
int64_t og_world_step(og_world* w, int64_t n);
int og_world_finished(og_world* w);
int64_t og_world_current_step(og_world* w);
int og_world_vehicles(og_world* w, const gmaco_vehicle_view* v);
int32_t og_world_signal_count(og_world* w);
int og_world_signals(og_world* w, const gmaco_signal_view* v, int64_t cap);
int og_world_pheromone(og_world* w, int64_t* tau);
int og_world_set_pheromone(og_world* w, const int64_t* tau);
int og_world_occupancy(og_world* w, int32_t* occ);
int og_world_collect(og_world* w, gmaco_run_result* r, double* travel, int32_t* rvid,
                     int32_t* rnode, int32_t cap);
int og_world_route(og_world* w, int32_t vid, int32_t planned, int32_t* out, int32_t cap, int32_t* len);
int og_world_counters(og_world* w, gmaco_counters* c);
int og_world_next_node(og_world* w, int algorithm, int32_t count, const int32_t* current,
                       const int32_t* dest, const uint64_t* entity, const uint64_t* step, int64_t n_t,
                       int32_t* out_next, int32_t* out_via, uint8_t* out_dev);
/* Sharded protocol (the multi-GPU exchange, host-mediated): plan only
 * vehicles [lo, hi); per step part 1 (stage B over the shard), export the
 * shard's decision records (edge, -1, -2) and deposits, import everyone's,
 * part 2 (apply remote decisions, stages C..G). */
int og_world_set_vehicle_range(og_world* w, int32_t lo, int32_t hi);
int og_world_step_part(og_world* w, int32_t part);
int og_world_exchange_export(og_world* w, int32_t* decisions, int64_t* deposits);
int og_world_exchange_import(og_world* w, const int32_t* decisions, const int64_t* deposits);

#ifdef __cplusplus
}
#endif
#endif
