/* gmaco_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference simulator's hot path
 * (/root/reference/proj, "R/" below) plus the colony extension the north star
 * adds.  Every function cites the reference lines it restates.  Compiled with
 * -ffp-contract=off so every double expression rounds exactly as the
 * reference's (g++ -O2, x86-64 baseline, no FMA).  It is pinned against the
 * compiled reference (oracle/_ref) and the reference's own KATs by
 * tests/test_oracle_*.py.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load it.
 */
#include "gmaco_oracle.h"

#include <alloca.h>
#include <pthread.h>
#include <unistd.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define INF64 INT64_MAX
#define TABU_TENURE 16

/* ------------------------------------------------------------------------ */
/* rng.hpp:21-56                                                              */
/* ------------------------------------------------------------------------ */
uint64_t og_mix64(uint64_t x) { /* rng.hpp:21-26 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t og_draw(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) { /* rng.hpp:28-35 */
  uint64_t h = og_mix64(seed);
  h = og_mix64(h ^ a);
  h = og_mix64(h ^ b);
  h = og_mix64(h ^ c);
  return h;
}
double og_to_unit(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; } /* rng.hpp:42-45 */
double og_uniform(uint64_t bits, double lo, double hi) {                      /* rng.hpp:47-49 */
  return lo + og_to_unit(bits) * (hi - lo);
}
uint64_t og_below(uint64_t bits, uint64_t n) { /* rng.hpp:51-56 */
  return (uint64_t)(((unsigned __int128)bits * n) >> 64);
}

enum { S_PHER_INIT = 1, S_SPAWN_PAIR = 2, S_SPAWN_SPEED = 3, S_SPAWN_DEPART = 4, S_ACO = 5 };

/* Philox4x32-10, the counter-based generator of Salmon et al. (SC'11). */
void og_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Ant uniform.  REFERENCE keying reduces to RngKey{seed, vid, step} of the
 * reference ACO decision (routing.cpp:97-98, engine.cpp:189-194) at ant 0,
 * hop 0.  PHILOX keying: counter (step, vid, ant, hop/2), key = seed. */
double og_ant_uniform(int rng, uint64_t seed, int64_t step, int32_t vid, int32_t ant, int32_t hop) {
  if (rng == GMACO_RNG_REFERENCE) {
    uint64_t a = (uint64_t)(uint32_t)vid | ((uint64_t)(uint32_t)ant << 32);
    uint64_t b = (uint64_t)step | ((uint64_t)(uint32_t)hop << 40);
    return og_to_unit(og_draw(seed, S_ACO, a, b));
  }
  /* one 128-bit Philox block serves two hops: counter (step, vid, ant, hop/2),
   * hop&1 selects the 64-bit half */
  uint32_t ctr[4] = {(uint32_t)step, (uint32_t)vid, (uint32_t)ant, (uint32_t)hop >> 1};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  og_philox4x32_10(ctr, key, o);
  return og_to_unit((hop & 1) ? (((uint64_t)o[2] << 32) | o[3]) : (((uint64_t)o[0] << 32) | o[1]));
}

/* ------------------------------------------------------------------------ */
/* pheromone.hpp:16-21, pheromone.cpp, parallel.cpp:77-92                     */
/* ------------------------------------------------------------------------ */
int64_t og_tau_from_double(double v) { return llround(v * 1e6); } /* pheromone.hpp:18 */
static double tau_to_double(int64_t v) { return (double)v / 1e6; } /* pheromone.hpp:19 */
static int64_t min_u(const gmaco_pheromone_params* p) { return og_tau_from_double(p->tau_min); }
static int64_t max_u(const gmaco_pheromone_params* p) { return og_tau_from_double(p->tau_max); }
static int64_t inc_u(const gmaco_pheromone_params* p) { return og_tau_from_double(p->delta_inc); }
static int64_t dec_u(const gmaco_pheromone_params* p) { return og_tau_from_double(p->delta_dec); }
static int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }

int64_t og_evaporate_one(int64_t tau, const gmaco_pheromone_params* p) { /* pheromone.cpp:61-67 */
  int64_t scaled = (int64_t)floor((1.0 - p->rho) * (double)tau);
  return i64max(min_u(p), scaled);
}

int64_t og_deposit_amount(int64_t len_mm, const gmaco_pheromone_params* p) { /* pheromone.cpp:73-78 */
  if (len_mm <= 0) return -1;
  const double length_km = (double)len_mm / 1e6;
  return og_tau_from_double(p->aco_deposit_q / length_km);
}

int64_t og_fold_maco_edge(int64_t t, const int32_t* pos, int32_t n, int64_t total,
                          const gmaco_pheromone_params* p) { /* parallel.cpp:77-92 */
  const int64_t lo = min_u(p), hi = max_u(p), inc = inc_u(p), dec = dec_u(p);
  int64_t done = 0;
  for (int32_t i = 0; i < n; ++i) {
    const int64_t gap = pos[i] - done;
    if (gap > 0) t = i64max(lo, t - gap * dec);
    t = i64min(hi, t + inc);
    done = (int64_t)pos[i] + 1;
  }
  const int64_t gap = total - done;
  if (gap > 0) t = i64max(lo, t - gap * dec);
  return t;
}

/* ------------------------------------------------------------------------ */
/* signals.cpp                                                                */
/* ------------------------------------------------------------------------ */
static int order_position(const gmaco_signal_params* p, int phase) { /* signals.cpp:50-54 */
  for (int i = 0; i < GMACO_PHASES; ++i)
    if (p->fixed_cycle_order[i] == phase) return i;
  return 0;
}
static int next_in_order(const gmaco_signal_params* p, int cursor) { /* signals.cpp:56-58 */
  return p->fixed_cycle_order[(order_position(p, cursor) + 1) % GMACO_PHASES];
}

int og_select_phase(int kind, const int32_t* q, const double* hw, int cursor,
                    const gmaco_signal_params* p) {
  if (kind == GMACO_FIXED) return next_in_order(p, cursor); /* signals.cpp:92-94 */
  if (kind == GMACO_ADAPTIVE) {                             /* signals.cpp:96-103 */
    int pos = order_position(p, cursor);
    for (int i = 0; i < GMACO_PHASES; ++i) {
      int ph = p->fixed_cycle_order[(pos + i) % GMACO_PHASES];
      if (q[ph] > 0) return ph;
    }
    return next_in_order(p, cursor);
  }
  /* preemptive, signals.cpp:62-90 */
  int best = -1;
  for (int ph = 0; ph < GMACO_PHASES; ++ph)
    if (q[ph] > p->th_max && (best == -1 || q[ph] > q[best])) best = ph;
  if (best != -1) return best;
  for (int ph = 0; ph < GMACO_PHASES; ++ph)
    if (hw[ph] > p->t_max && (best == -1 || hw[ph] > hw[best])) best = ph;
  if (best != -1) return best;
  for (int ph = 0; ph < GMACO_PHASES; ++ph)
    if (q[ph] > 0 && (best == -1 || q[ph] > q[best])) best = ph;
  if (best != -1) return best;
  return next_in_order(p, cursor);
}

static int discharge_budget(double* rem, double dt, int lanes, const gmaco_signal_params* p) {
  /* signals.cpp:121-124 */
  *rem += p->saturation_flow * lanes * dt;
  int budget = (int)floor(*rem);
  *rem -= budget;
  return budget;
}

int og_discharge(int32_t qlen, double* rem, double dt, int lanes, const gmaco_signal_params* p) {
  int budget = discharge_budget(rem, dt, lanes, p);
  return budget < qlen ? budget : qlen;
}

/* ------------------------------------------------------------------------ */
/* Errors                                                                     */
/* ------------------------------------------------------------------------ */
static void set_err(char* err, int32_t cap, const char* fmt, ...) {
  if (!err || cap <= 0) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, (size_t)cap, fmt, ap);
  va_end(ap);
}

/* ------------------------------------------------------------------------ */
/* net.cpp: RoadNetwork validation + adjacency (net.cpp:38-98)               */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t n, m;
  const int32_t *from, *to, *lanes;
  const int64_t* len;
  int32_t *out_ptr, *out_nbr, *out_edge; /* out-edges sorted by neighbor id */
  int32_t *in_ptr, *in_edge;             /* in-edges ascending */
} og_net;

static void net_free(og_net* g) {
  free(g->out_ptr); free(g->out_nbr); free(g->out_edge);
  free(g->in_ptr); free(g->in_edge);
  memset(g, 0, sizeof(*g));
}

static int net_build(const gmaco_graph_desc* d, og_net* g, char* err, int32_t cap) {
  memset(g, 0, sizeof(*g));
  const int32_t n = d->node_count, m = d->edge_count;
  if (n <= 0) { set_err(err, cap, "network has no nodes"); return 1; }
  if (m < 0) { set_err(err, cap, "network edge count must be >= 0"); return 1; }
  for (int32_t e = 0; e < m; ++e) { /* net.cpp:58-79, input order */
    if (d->edge_from[e] < 0 || d->edge_from[e] >= n) {
      set_err(err, cap, "edge %d references missing node %d", e, d->edge_from[e]); return 1;
    }
    if (d->edge_to[e] < 0 || d->edge_to[e] >= n) {
      set_err(err, cap, "edge %d references missing node %d", e, d->edge_to[e]); return 1;
    }
    if (d->edge_from[e] == d->edge_to[e]) {
      set_err(err, cap, "edge %d is a self-loop at node %d", e, d->edge_from[e]); return 1;
    }
    if (d->edge_length_mm[e] <= 0) { set_err(err, cap, "edge %d has nonpositive length", e); return 1; }
    if (d->edge_lanes && d->edge_lanes[e] < 1) { set_err(err, cap, "edge %d has lanes < 1", e); return 1; }
  }
  g->n = n; g->m = m;
  g->from = d->edge_from; g->to = d->edge_to; g->len = d->edge_length_mm; g->lanes = d->edge_lanes;
  g->out_ptr = calloc((size_t)n + 1, sizeof(int32_t));
  g->in_ptr = calloc((size_t)n + 1, sizeof(int32_t));
  g->out_nbr = malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  g->out_edge = malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  g->in_edge = malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  for (int32_t e = 0; e < m; ++e) { g->out_ptr[d->edge_from[e] + 1]++; g->in_ptr[d->edge_to[e] + 1]++; }
  for (int32_t u = 0; u < n; ++u) { g->out_ptr[u + 1] += g->out_ptr[u]; g->in_ptr[u + 1] += g->in_ptr[u]; }
  int32_t* oc = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* ic = malloc(sizeof(int32_t) * (size_t)n);
  memcpy(oc, g->out_ptr, sizeof(int32_t) * (size_t)n);
  memcpy(ic, g->in_ptr, sizeof(int32_t) * (size_t)n);
  for (int32_t e = 0; e < m; ++e) { /* ascending edge id; in-lists stay ascending */
    int32_t u = d->edge_from[e], v = d->edge_to[e];
    g->out_nbr[oc[u]] = v; g->out_edge[oc[u]] = e; oc[u]++;
    g->in_edge[ic[v]++] = e;
  }
  free(oc); free(ic);
  for (int32_t u = 0; u < n; ++u) { /* sort out-list by neighbor (insertion; degrees are small) */
    for (int32_t i = g->out_ptr[u] + 1; i < g->out_ptr[u + 1]; ++i) {
      int32_t nb = g->out_nbr[i], ed = g->out_edge[i], j = i - 1;
      while (j >= g->out_ptr[u] && g->out_nbr[j] > nb) {
        g->out_nbr[j + 1] = g->out_nbr[j]; g->out_edge[j + 1] = g->out_edge[j]; --j;
      }
      g->out_nbr[j + 1] = nb; g->out_edge[j + 1] = ed;
    }
    for (int32_t i = g->out_ptr[u] + 1; i < g->out_ptr[u + 1]; ++i) /* net.cpp:89-93 */
      if (g->out_nbr[i] == g->out_nbr[i - 1]) {
        set_err(err, cap, "duplicate edge between nodes %d and %d", u, g->out_nbr[i]);
        net_free(g);
        return 1;
      }
  }
  return 0;
}

int og_validate_graph(const gmaco_graph_desc* d, char* err, int32_t cap) {
  og_net g;
  int rc = net_build(d, &g, err, cap);
  if (rc == 0) net_free(&g);
  return rc;
}

/* generate_grid (net.cpp:208-244); sig_all additionally signalizes every
 * node (the C2 "signals at every intersection" config). */
int og_generate_grid(int rows, int cols, double len_m, int lanes, int sig_interior, int sig_all,
                     uint8_t* signalized, int32_t* from, int32_t* to, int64_t* len_mm, int32_t* lanes_out) {
  if (rows < 2 || cols < 2 || len_m <= 0 || lanes < 1) return 1;
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      int interior = r > 0 && r < rows - 1 && c > 0 && c < cols - 1;
      signalized[r * cols + c] = (uint8_t)(sig_all || (sig_interior && interior));
    }
  const int64_t len = llround(len_m * 1000.0);
  int32_t id = 0;
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      int32_t here = r * cols + c;
      int32_t nb[2]; int k = 0;
      if (c + 1 < cols) nb[k++] = here + 1;
      if (r + 1 < rows) nb[k++] = here + cols;
      for (int i = 0; i < k; ++i) {
        from[id] = here; to[id] = nb[i]; len_mm[id] = len; lanes_out[id] = lanes; ++id;
        from[id] = nb[i]; to[id] = here; len_mm[id] = len; lanes_out[id] = lanes; ++id;
      }
    }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Shortest paths: dijkstra_to / greedy_hop / all_pairs_distances            */
/* (net.cpp:359-437), binary heap keyed (dist, node) like the reference's    */
/* std::priority_queue<pair> with std::greater.                              */
/* ------------------------------------------------------------------------ */
typedef struct { int64_t d; int32_t u; } hitem;
static int hless(hitem a, hitem b) { return a.d < b.d || (a.d == b.d && a.u < b.u); }

static void dijkstra_rev(const og_net* g, const int32_t* rptr, const int32_t* rsrc, const int32_t* redge,
                         int32_t dst, int64_t* dist) {
  const int32_t n = g->n;
  for (int32_t i = 0; i < n; ++i) dist[i] = INF64;
  hitem* h = malloc(sizeof(hitem) * ((size_t)g->m + 2));
  size_t hs = 0;
  dist[dst] = 0;
  h[hs++] = (hitem){0, dst};
  while (hs) {
    hitem top = h[0];
    h[0] = h[--hs];
    for (size_t i = 0;;) { /* sift down */
      size_t l = 2 * i + 1, r = l + 1, s = i;
      if (l < hs && hless(h[l], h[s])) s = l;
      if (r < hs && hless(h[r], h[s])) s = r;
      if (s == i) break;
      hitem t = h[i]; h[i] = h[s]; h[s] = t; i = s;
    }
    if (top.d != dist[top.u]) continue;
    for (int32_t k = rptr[top.u]; k < rptr[top.u + 1]; ++k) {
      int32_t x = rsrc[k];
      int64_t nd = top.d + g->len[redge[k]];
      if (nd < dist[x]) {
        dist[x] = nd;
        size_t i = hs++;
        h[i] = (hitem){nd, x};
        while (i > 0) { /* sift up */
          size_t p = (i - 1) / 2;
          if (!hless(h[i], h[p])) break;
          hitem t = h[i]; h[i] = h[p]; h[p] = t; i = p;
        }
      }
    }
  }
  free(h);
}

static void build_reverse(const og_net* g, int32_t** rptr, int32_t** rsrc, int32_t** redge) {
  *rptr = calloc((size_t)g->n + 1, sizeof(int32_t));
  *rsrc = malloc(sizeof(int32_t) * (size_t)(g->m ? g->m : 1));
  *redge = malloc(sizeof(int32_t) * (size_t)(g->m ? g->m : 1));
  for (int32_t e = 0; e < g->m; ++e) (*rptr)[g->to[e] + 1]++;
  for (int32_t u = 0; u < g->n; ++u) (*rptr)[u + 1] += (*rptr)[u];
  int32_t* c = malloc(sizeof(int32_t) * (size_t)g->n);
  memcpy(c, *rptr, sizeof(int32_t) * (size_t)g->n);
  for (int32_t e = 0; e < g->m; ++e) { /* edge-id order, as net.cpp:363 */
    int32_t v = g->to[e];
    (*rsrc)[c[v]] = g->from[e]; (*redge)[c[v]] = e; c[v]++;
  }
  free(c);
}

/* One reverse Dijkstra per target (dijkstra_to, net.cpp:359-385), the
 * targets spread over host threads (each row is independent). */
typedef struct {
  const og_net* g;
  const int32_t *rp, *rs, *re, *targets;
  int64_t* out;
  int32_t ntargets, next;
  pthread_mutex_t mu;
} sssp_job;

static void* sssp_worker(void* arg) {
  sssp_job* j = (sssp_job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int32_t t = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (t >= j->ntargets) return NULL;
    dijkstra_rev(j->g, j->rp, j->rs, j->re, j->targets[t], j->out + (size_t)t * j->g->n);
  }
}

static void targets_sssp_run(const og_net* g, const int32_t* targets, int32_t T, int64_t* out) {
  int32_t *rp, *rs, *re;
  build_reverse(g, &rp, &rs, &re);
  sssp_job j = {g, rp, rs, re, targets, out, T, 0, PTHREAD_MUTEX_INITIALIZER};
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  if (nt < 1) nt = 1;
  if (nt > T) nt = T;
  if (nt > 64) nt = 64;
  pthread_t th[64];
  for (long i = 0; i < nt; ++i) pthread_create(&th[i], NULL, sssp_worker, &j);
  for (long i = 0; i < nt; ++i) pthread_join(th[i], NULL);
  free(rp); free(rs); free(re);
}

static int32_t greedy_hop(const og_net* g, const int64_t* dist_to, int32_t u) { /* net.cpp:387-395 */
  for (int32_t k = g->out_ptr[u]; k < g->out_ptr[u + 1]; ++k) {
    int32_t nb = g->out_nbr[k];
    if (dist_to[nb] == INF64) continue;
    if (g->len[g->out_edge[k]] + dist_to[nb] == dist_to[u]) return nb;
  }
  return -1;
}

int og_dijkstra_to(const gmaco_graph_desc* d, int32_t dst, int64_t* dist_to) {
  og_net g;
  if (net_build(d, &g, NULL, 0)) return 1;
  int32_t *rp, *rs, *re;
  build_reverse(&g, &rp, &rs, &re);
  dijkstra_rev(&g, rp, rs, re, dst, dist_to);
  free(rp); free(rs); free(re);
  net_free(&g);
  return 0;
}

int og_apsp(const gmaco_graph_desc* d, int64_t* dist, int32_t* next) { /* net.cpp:419-437 */
  og_net g;
  if (net_build(d, &g, NULL, 0)) return 1;
  const int32_t n = g.n;
  int32_t *rp, *rs, *re;
  build_reverse(&g, &rp, &rs, &re);
  int64_t* dt = malloc(sizeof(int64_t) * (size_t)n);
  for (int32_t dst = 0; dst < n; ++dst) {
    dijkstra_rev(&g, rp, rs, re, dst, dt);
    for (int32_t u = 0; u < n; ++u) {
      if (dist) dist[(size_t)u * n + dst] = dt[u];
      if (next) next[(size_t)u * n + dst] = u == dst ? u : (dt[u] != INF64 ? greedy_hop(&g, dt, u) : -1);
    }
  }
  free(dt); free(rp); free(rs); free(re);
  net_free(&g);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* World (engine.hpp:157-177)                                                 */
/* ------------------------------------------------------------------------ */
typedef struct { int32_t* vid; int64_t* enq; int64_t head, size, cap; } fifo;

static void fifo_push(fifo* q, int32_t vid, int64_t enq) {
  if (q->head + q->size == q->cap) {
    if (q->head > 0) {
      memmove(q->vid, q->vid + q->head, sizeof(int32_t) * (size_t)q->size);
      memmove(q->enq, q->enq + q->head, sizeof(int64_t) * (size_t)q->size);
      q->head = 0;
    }
    if (q->size == q->cap) {
      q->cap = q->cap ? 2 * q->cap : 8;
      q->vid = realloc(q->vid, sizeof(int32_t) * (size_t)q->cap);
      q->enq = realloc(q->enq, sizeof(int64_t) * (size_t)q->cap);
    }
  }
  q->vid[q->head + q->size] = vid;
  q->enq[q->head + q->size] = enq;
  q->size++;
}

typedef struct { int32_t* a; int32_t n, cap; } ivec;
static void ivec_push(ivec* v, int32_t x) {
  if (v->n == v->cap) { v->cap = v->cap ? 2 * v->cap : 8; v->a = realloc(v->a, sizeof(int32_t) * (size_t)v->cap); }
  v->a[v->n++] = x;
}

struct og_world {
  og_net g;
  uint8_t* sig;
  /* distance service */
  int32_t dkind, grows, gcols;
  int64_t* dense;     /* [n*n] */
  int32_t* slot_of;   /* TARGETS: node -> slot or -1 */
  int64_t* tdist;     /* TARGETS: [k*n] */
  int32_t ntargets;
  int32_t* targets;
  int64_t grid_len;
  gmaco_sim_config cfg;
  int32_t *block_a, *block_b;
  /* pheromone */
  int64_t* tau;
  double* eta_beta; /* pow(1/(len/1000), beta), routing.cpp:92-94 */
  double* weight;   /* per-edge roulette weight for the coming step */
  int64_t* ecost;   /* per-edge colony tour cost for the coming step */
  /* signals */
  int32_t S;
  int32_t *sig_node, *sig_of_node, *bind_sig, *bind_phase;
  int32_t *green, *cursor, *dlanes;
  int64_t* el_steps;
  double* el_s;
  fifo* q;
  double *head_wait, *rem;
  /* vehicles */
  int32_t V;
  int32_t *origin, *dest, *at_node, *on_edge, *queued_phase, *decisions, *deviations;
  double* speed;
  int64_t *advance, *progress, *overshoot, *joined, *depart, *arrive, *latency_debt;
  int64_t *driving, *queued, *lat_steps, *path_len_mm;
  uint8_t* state;
  ivec* path;
  ivec* plan;
  int64_t* plan_step;
  uint8_t* plan_done;
  int64_t* dep; /* per-edge deposit accumulator (best-tour mode) */
  int32_t* occ;
  int64_t step, active, dt_us, latency_us;
  int64_t qtotal, qsamples;
  int32_t max_occ;
  /* step scratch */
  ivec dec_vid, dec_edge, completions, enq_vid;
  gmaco_counters ctr;
  int32_t vlo, vhi; /* planning range (sharded protocol) */
  int32_t* dec_rec; /* this step's decision per vehicle: edge (| GMACO_REC_DEVIATED), -1 none, -2 retired */
};

static void targets_sssp(og_world* w) { targets_sssp_run(&w->g, w->targets, w->ntargets, w->tdist); }

/* ---- distance service (routing.cpp reads dist.reachable / dist.dist_mm) -- */
static int64_t dist_to_dest(const og_world* w, int32_t x, int32_t dest) {
  switch (w->dkind) {
    case GMACO_DIST_GRID: {
      int32_t rx = x / w->gcols, cx = x % w->gcols, rd = dest / w->gcols, cd = dest % w->gcols;
      int64_t h = (int64_t)(rx > rd ? rx - rd : rd - rx) + (cx > cd ? cx - cd : cd - cx);
      return h * w->grid_len;
    }
    case GMACO_DIST_TARGETS: {
      int32_t s = w->slot_of[dest];
      return s < 0 ? INF64 : w->tdist[(size_t)s * w->g.n + x];
    }
    default:
      return w->dense[(size_t)x * w->g.n + dest];
  }
}

/* candidate_neighbors (routing.cpp:16-30) into caller arrays; returns count.
 * tabu (colony, progress filter off only): nodes excluded from the set. */
static int32_t candidates(const og_world* w, int32_t cur, int32_t dest, int progress_filter,
                          const int32_t* tabu, int32_t ntabu, int32_t* cn, int32_t* ce,
                          int64_t* scanned) {
  const og_net* g = &w->g;
  const int64_t dcur = dist_to_dest(w, cur, dest);
  int32_t nr = 0, nc = 0;
  int32_t deg = g->out_ptr[cur + 1] - g->out_ptr[cur];
  int32_t* rn = (int32_t*)alloca(sizeof(int32_t) * (size_t)(deg + 1));
  int32_t* re = (int32_t*)alloca(sizeof(int32_t) * (size_t)(deg + 1));
  if (scanned) *scanned += deg;
  for (int32_t k = g->out_ptr[cur]; k < g->out_ptr[cur + 1]; ++k) {
    int32_t nb = g->out_nbr[k];
    int64_t dn = dist_to_dest(w, nb, dest);
    if (dn == INF64) continue;
    int is_tabu = 0;
    for (int32_t t = 0; t < ntabu; ++t) if (tabu[t] == nb) is_tabu = 1;
    if (is_tabu) continue;
    rn[nr] = nb; re[nr] = g->out_edge[k]; nr++;
    if (dn < dcur) { cn[nc] = nb; ce[nc] = g->out_edge[k]; nc++; }
  }
  if (progress_filter && nc > 0) return nc;
  memcpy(cn, rn, sizeof(int32_t) * (size_t)nr);
  memcpy(ce, re, sizeof(int32_t) * (size_t)nr);
  return nr;
}

/* ACO roulette over per-edge weights (routing.cpp:88-113). */
static int32_t roulette(const double* weight, const int32_t* ce, int32_t c, double u) {
  double total = 0.0;
  for (int32_t i = 0; i < c; ++i) total += weight[ce[i]];
  int32_t pick = c - 1;
  if (total <= 0.0 || !isfinite(total)) {
    pick = (int32_t)(u * (double)c);
    if (pick > c - 1) pick = c - 1;
  } else {
    double point = u * total, cum = 0.0;
    for (int32_t i = 0; i < c; ++i) {
      cum += weight[ce[i]];
      if (point < cum) { pick = i; break; }
    }
  }
  return pick;
}

static double base_weight(const og_world* w, int32_t e) { /* routing.cpp:90-94 */
  double tau = tau_to_double(w->tau[e]);
  double a = w->cfg.routing.aco_alpha;
  double ta = a == 1.0 ? tau : pow(tau, a);
  return ta * w->eta_beta[e];
}

/* next_node_maco (routing.cpp:32-75) over a candidate list. */
static int32_t maco_pick(const og_world* w, const int32_t* ce, int32_t c, int64_t n_t, int* deviated) {
  int32_t primary = 0;
  for (int32_t i = 1; i < c; ++i)
    if (w->tau[ce[i]] < w->tau[ce[primary]]) primary = i;
  int trigger = 0;
  if (c >= 2) {
    if (w->cfg.routing.deviation_mode == GMACO_DEV_GLOBAL)
      trigger = n_t > w->cfg.routing.deviation_threshold;
    else
      trigger = (int64_t)w->occ[ce[primary]] > w->cfg.routing.deviation_threshold;
  }
  *deviated = trigger;
  if (!trigger) return primary;
  int32_t second = primary == 0 ? 1 : 0;
  for (int32_t i = 0; i < c; ++i) {
    if (i == primary || i == second) continue;
    if (w->tau[ce[i]] < w->tau[ce[second]]) second = i;
  }
  return second;
}

/* One routing decision (next_node_{dijkstra,aco,maco}, routing.cpp:32-125).
 * Returns the chosen edge or -1 when unroutable. */
static int32_t route_one(og_world* w, int algorithm, int32_t cur, int32_t dest, uint64_t entity,
                         uint64_t step, int64_t n_t, int use_fresh_weights, int32_t* next, int* dev) {
  const og_net* g = &w->g;
  *dev = 0;
  if (algorithm == GMACO_DIJKSTRA) { /* routing.cpp:117-125 + greedy_hop net.cpp:387-395 */
    int64_t dc = dist_to_dest(w, cur, dest);
    if (dc == INF64) return -1;
    for (int32_t k = g->out_ptr[cur]; k < g->out_ptr[cur + 1]; ++k) {
      int32_t nb = g->out_nbr[k];
      int64_t dn = dist_to_dest(w, nb, dest);
      if (dn == INF64) continue;
      if (g->len[g->out_edge[k]] + dn == dc) { *next = nb; return g->out_edge[k]; }
    }
    return -1;
  }
  int32_t deg = g->out_ptr[cur + 1] - g->out_ptr[cur];
  int32_t* cn = (int32_t*)alloca(sizeof(int32_t) * (size_t)(deg + 1));
  int32_t* ce = (int32_t*)alloca(sizeof(int32_t) * (size_t)(deg + 1));
  int32_t c = candidates(w, cur, dest, w->cfg.routing.progress_filter, NULL, 0, cn, ce, &w->ctr.degree_sum);
  if (c == 0) return -1;
  w->ctr.candidates += c;
  int32_t pick;
  if (algorithm == GMACO_ACO) {
    double u = og_to_unit(og_draw(w->cfg.seed, S_ACO, entity, step));
    if (use_fresh_weights) {
      double* wt = (double*)alloca(sizeof(double) * (size_t)c);
      for (int32_t i = 0; i < c; ++i) wt[i] = base_weight(w, ce[i]);
      double total = 0.0;
      for (int32_t i = 0; i < c; ++i) total += wt[i];
      pick = c - 1;
      if (total <= 0.0 || !isfinite(total)) {
        pick = (int32_t)(u * (double)c);
        if (pick > c - 1) pick = c - 1;
      } else {
        double point = u * total, cum = 0.0;
        for (int32_t i = 0; i < c; ++i) { cum += wt[i]; if (point < cum) { pick = i; break; } }
      }
    } else {
      pick = roulette(w->weight, ce, c, u);
    }
  } else {
    pick = maco_pick(w, ce, c, n_t, dev);
  }
  *next = cn[pick];
  return ce[pick];
}

/* ---- colony (north-star extension) -------- */
/* Walks one ant from `start`; writes its edges to tour (if non-NULL) and
 * returns the hop count; *cost is INF64 for a failed ant.  *first_ok is set
 * when hop 0 had a candidate. */
/* Work counters of one planning thread (summed into w->ctr in vid order). */
typedef struct { int64_t ant_steps, candidates, degree_sum, vehicle_routes; } og_ctr_local;

static int32_t ant_walk(const og_world* w, int32_t vid, int32_t ant, int32_t start, int32_t dest,
                        int64_t* cost, int32_t* tour, int* first_ok, og_ctr_local* count) {
  const gmaco_colony_params* cp = &w->cfg.colony;
  const int pf = w->cfg.routing.progress_filter;
  const int32_t max_hops = cp->max_hops > 0 ? cp->max_hops : w->g.n - 1;
  int32_t tabu[TABU_TENURE];
  int32_t ntabu = 0, tpos = 0;
  int32_t x = start, hops = 0;
  int64_t c = 0;
  *first_ok = 0;
  int32_t cn[64], ce[64];
  if (!pf) { tabu[0] = start; ntabu = 1; tpos = 1 % TABU_TENURE; }
  while (x != dest && (cp->hop_limit == 0 || hops < cp->hop_limit)) {
    if (hops >= max_hops) { *cost = INF64; return hops; }
    int32_t deg = w->g.out_ptr[x + 1] - w->g.out_ptr[x];
    int32_t *pcn = cn, *pce = ce;
    if (deg > 63) {
      pcn = (int32_t*)malloc(sizeof(int32_t) * (size_t)(deg + 1));
      pce = (int32_t*)malloc(sizeof(int32_t) * (size_t)(deg + 1));
    }
    int64_t scanned = 0;
    int32_t nc = candidates(w, x, dest, pf, pf ? NULL : tabu, pf ? 0 : ntabu, pcn, pce, &scanned);
    if (nc == 0) {
      if (pcn != cn) { free(pcn); free(pce); }
      *cost = INF64;
      return hops;
    }
    if (hops == 0) *first_ok = 1;
    double u = og_ant_uniform(cp->rng, w->cfg.seed, w->step, vid, ant, hops);
    int32_t pick = roulette(w->weight, pce, nc, u);
    int32_t e = pce[pick];
    x = pcn[pick];
    if (pcn != cn) { free(pcn); free(pce); }
    if (count) { count->ant_steps++; count->candidates += nc; count->degree_sum += scanned; }
    c += w->ecost[e];
    if (tour) tour[hops] = e;
    hops++;
    if (!pf) {
      tabu[tpos] = x;
      tpos = (tpos + 1) % TABU_TENURE;
      if (ntabu < TABU_TENURE) ntabu++;
    }
  }
  *cost = c;
  return hops;
}

/* ------------------------------------------------------------------------ */
/* Config validation (engine.cpp:12-32, pheromone.cpp:9-19, signals.cpp:8-21,*/
/* routing.cpp:9-14)                                                          */
/* ------------------------------------------------------------------------ */
static int validate_config(const gmaco_sim_config* c, char* err, int32_t cap) {
  if (c->vehicle_count < 1) { set_err(err, cap, "config: vehicle_count must be >= 1"); return 1; }
  if (!(c->dt_s > 0)) { set_err(err, cap, "config: dt must be positive"); return 1; }
  if (c->max_steps < 0) { set_err(err, cap, "config: max_steps must be >= 0"); return 1; }
  if (c->decision_latency_s < 0) { set_err(err, cap, "config: decision_latency_s must be >= 0"); return 1; }
  if (c->spawn == GMACO_UNIFORM_WINDOW && c->spawn_window_steps < 1) {
    set_err(err, cap, "config: spawn_window_steps must be >= 1"); return 1;
  }
  if (c->speed_min_mps <= 0 || c->speed_max_mps < c->speed_min_mps) {
    set_err(err, cap, "config: speed range must satisfy 0 < min <= max"); return 1;
  }
  if (c->od_pattern == GMACO_OD_BLOCKS) {
    if (c->od_bias < 0 || c->od_bias > 1) { set_err(err, cap, "config: od bias must lie in [0, 1]"); return 1; }
    if (c->od_block_a_len <= 0 || c->od_block_b_len <= 0) {
      set_err(err, cap, "config: od blocks must be non-empty"); return 1;
    }
  }
  const gmaco_pheromone_params* p = &c->pheromone;
  if (!(p->tau_min <= p->tau_init_lo && p->tau_init_lo <= p->tau_init_hi && p->tau_init_hi <= p->tau_max)) {
    set_err(err, cap, "pheromone init range must satisfy tau_min <= lo <= hi <= tau_max"); return 1;
  }
  if (p->delta_inc <= 0 || p->delta_dec <= 0) {
    set_err(err, cap, "pheromone delta_inc and delta_dec must be positive"); return 1;
  }
  if (p->rho < 0 || p->rho >= 1) { set_err(err, cap, "pheromone rho must lie in [0, 1)"); return 1; }
  if (p->tau_min < 0) { set_err(err, cap, "pheromone tau_min must be >= 0"); return 1; }
  const gmaco_signal_params* s = &c->signal;
  if (s->th_max < 1) { set_err(err, cap, "signal th_max must be >= 1"); return 1; }
  if (s->t_max <= 0) { set_err(err, cap, "signal t_max must be positive"); return 1; }
  if (s->green_duration_s <= 0) { set_err(err, cap, "signal green_duration must be positive"); return 1; }
  if (s->saturation_flow <= 0) { set_err(err, cap, "signal saturation_flow must be positive"); return 1; }
  int seen[GMACO_PHASES] = {0};
  for (int i = 0; i < GMACO_PHASES; ++i) {
    int ph = s->fixed_cycle_order[i];
    if (ph < 0 || ph >= GMACO_PHASES || seen[ph]) {
      set_err(err, cap, "signal fixed_cycle_order must be a permutation of 0..7"); return 1;
    }
    seen[ph] = 1;
  }
  if (c->routing.deviation_threshold < 0) { set_err(err, cap, "routing deviation_threshold must be >= 0"); return 1; }
  if (c->routing.aco_alpha < 0 || c->routing.aco_beta < 0) {
    set_err(err, cap, "routing aco exponents must be >= 0"); return 1;
  }
  if (c->algorithm < GMACO_DIJKSTRA || c->algorithm > GMACO_COLONY) {
    set_err(err, cap, "config: unknown algorithm %d", c->algorithm); return 1;
  }
  if (c->controller < GMACO_FIXED || c->controller > GMACO_PREEMPTIVE) {
    set_err(err, cap, "config: unknown controller %d", c->controller); return 1;
  }
  if (c->algorithm == GMACO_COLONY) {
    const gmaco_colony_params* k = &c->colony;
    if (k->ants < 1) { set_err(err, cap, "colony: ants must be >= 1"); return 1; }
    if (k->hop_limit < 0 || k->max_hops < 0) { set_err(err, cap, "colony: hop limits must be >= 0"); return 1; }
    if (k->rng != GMACO_RNG_PHILOX && k->rng != GMACO_RNG_REFERENCE) { set_err(err, cap, "colony: unknown rng"); return 1; }
    if (k->deposit < GMACO_DEPOSIT_COMPLETION || k->deposit > GMACO_DEPOSIT_NONE) {
      set_err(err, cap, "colony: unknown deposit mode"); return 1;
    }
  }
  return 0;
}

/* ---- spawn_vehicles (engine.cpp:71-114) ---------------------------------- */
/* The uniform OD pool is the (u, v)-lexicographic list of ordered pairs with
 * u != v and v reachable from u (feasible_pairs, engine.cpp:50-57).  It is
 * indexed, not materialized: per-row counts + prefix sums select the row, a
 * row scan selects v.  For TARGETS distances the pool keeps v in the target
 * set (ascending). */
static int reachable(const og_world* w, int32_t u, int32_t v) { return dist_to_dest(w, u, v) != INF64; }

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : x > y;
}

typedef struct { int32_t* u; int32_t* v; int64_t n; } pairlist;

static void block_pairs(const og_world* w, const int32_t* from, int32_t nf, const int32_t* to,
                        int32_t nt, pairlist* out) { /* engine.cpp:59-66 */
  out->u = malloc(sizeof(int32_t) * (size_t)(nf * nt + 1));
  out->v = malloc(sizeof(int32_t) * (size_t)(nf * nt + 1));
  out->n = 0;
  for (int32_t i = 0; i < nf; ++i)
    for (int32_t j = 0; j < nt; ++j)
      if (from[i] != to[j] && reachable(w, from[i], to[j])) {
        out->u[out->n] = from[i]; out->v[out->n] = to[j]; out->n++;
      }
}

static int spawn(og_world* w, char* err, int32_t cap) {
  const gmaco_sim_config* c = &w->cfg;
  const int32_t n = w->g.n;
  int32_t* dests = NULL; /* candidate destination columns, ascending */
  int32_t nd = n;
  if (w->dkind == GMACO_DIST_TARGETS) {
    nd = w->ntargets;
    dests = malloc(sizeof(int32_t) * (size_t)nd);
    memcpy(dests, w->targets, sizeof(int32_t) * (size_t)nd);
    qsort(dests, (size_t)nd, sizeof(int32_t), cmp_i32);
  }
  int64_t* prefix = malloc(sizeof(int64_t) * ((size_t)n + 1));
  prefix[0] = 0;
  for (int32_t u = 0; u < n; ++u) {
    int64_t cnt = 0;
    if (w->dkind == GMACO_DIST_GRID) {
      cnt = n - 1;
    } else {
      for (int32_t j = 0; j < nd; ++j) {
        int32_t v = dests ? dests[j] : j;
        if (u != v && reachable(w, u, v)) cnt++;
      }
    }
    prefix[u + 1] = prefix[u] + cnt;
  }
  const int64_t pool = prefix[n];
  if (pool == 0) {
    set_err(err, cap, "spawn: network has no reachable origin/destination pair");
    free(prefix); free(dests);
    return 1;
  }
  pairlist ab = {0}, ba = {0};
  if (c->od_pattern == GMACO_OD_BLOCKS) {
    block_pairs(w, w->block_a, c->od_block_a_len, w->block_b, c->od_block_b_len, &ab);
    block_pairs(w, w->block_b, c->od_block_b_len, w->block_a, c->od_block_a_len, &ba);
  }
  for (int32_t vid = 0; vid < w->V; ++vid) {
    const pairlist* biased = NULL;
    if (c->od_pattern == GMACO_OD_BLOCKS) { /* engine.cpp:88-97 */
      double r = og_to_unit(og_draw(c->seed, S_SPAWN_PAIR, (uint64_t)vid, 0));
      if (r < c->od_bias) {
        int forward = og_to_unit(og_draw(c->seed, S_SPAWN_PAIR, (uint64_t)vid, 1)) < 0.5;
        const pairlist* b = forward ? &ab : &ba;
        if (b->n > 0) biased = b;
      }
    }
    uint64_t bits = og_draw(c->seed, S_SPAWN_PAIR, (uint64_t)vid, 2);
    if (biased) {
      uint64_t idx = og_below(bits, (uint64_t)biased->n);
      w->origin[vid] = biased->u[idx];
      w->dest[vid] = biased->v[idx];
    } else {
      int64_t idx = (int64_t)og_below(bits, (uint64_t)pool);
      int32_t lo = 0, hi = n; /* largest u with prefix[u] <= idx */
      while (hi - lo > 1) {
        int32_t mid = (lo + hi) / 2;
        if (prefix[mid] <= idx) lo = mid; else hi = mid;
      }
      int32_t u = lo;
      int64_t r = idx - prefix[u];
      int32_t v = -1;
      if (w->dkind == GMACO_DIST_GRID) {
        v = (int32_t)(r + (r >= u));
      } else {
        for (int32_t j = 0; j < nd; ++j) {
          int32_t cand = dests ? dests[j] : j;
          if (u != cand && reachable(w, u, cand)) {
            if (r == 0) { v = cand; break; }
            --r;
          }
        }
      }
      w->origin[vid] = u;
      w->dest[vid] = v;
    }
    w->speed[vid] = og_uniform(og_draw(c->seed, S_SPAWN_SPEED, (uint64_t)vid, 0), c->speed_min_mps,
                               c->speed_max_mps); /* engine.cpp:103-104 */
    w->advance[vid] = llround(w->speed[vid] * c->dt_s * 1000.0);
    w->depart[vid] = 0;
    if (c->spawn == GMACO_UNIFORM_WINDOW) /* engine.cpp:107-111 */
      w->depart[vid] = (int64_t)og_below(og_draw(c->seed, S_SPAWN_DEPART, (uint64_t)vid, 0),
                                         (uint64_t)c->spawn_window_steps);
  }
  free(ab.u); free(ab.v); free(ba.u); free(ba.v);
  free(prefix); free(dests);
  return 0;
}

/* ---- per-edge weights / costs for the coming step ------------------------ */
static int32_t edge_load(const og_world* w, int32_t e) {
  int32_t load = w->occ[e];
  if (w->bind_sig[e] >= 0) load += (int32_t)w->q[w->bind_sig[e] * GMACO_PHASES + w->bind_phase[e]].size;
  return load;
}

static void refresh_edge_terms(og_world* w) {
  const int congestion = w->cfg.algorithm == GMACO_COLONY && w->cfg.colony.congestion;
  for (int32_t e = 0; e < w->g.m; ++e) {
    double wt = base_weight(w, e);
    int64_t cost = w->g.len[e];
    if (congestion) {
      int32_t load = edge_load(w, e);
      wt = wt * (1.0 / (1.0 + (double)load));
      cost = cost + cost * (int64_t)load;
    }
    w->weight[e] = wt;
    w->ecost[e] = cost;
  }
}

/* ---- init_world (engine.cpp:116-144) ------------------------------------- */
void og_world_destroy(og_world* w) {
  if (!w) return;
  net_free(&w->g);
  free(w->sig); free(w->dense); free(w->slot_of); free(w->tdist); free(w->targets);
  free(w->block_a); free(w->block_b);
  free(w->tau); free(w->eta_beta); free(w->weight); free(w->ecost);
  free(w->sig_node); free(w->sig_of_node); free(w->bind_sig); free(w->bind_phase);
  free(w->green); free(w->cursor); free(w->dlanes); free(w->el_steps); free(w->el_s);
  if (w->q)
    for (int64_t i = 0; i < (int64_t)w->S * GMACO_PHASES; ++i) { free(w->q[i].vid); free(w->q[i].enq); }
  free(w->q); free(w->head_wait); free(w->rem);
  free(w->origin); free(w->dest); free(w->at_node); free(w->on_edge); free(w->queued_phase);
  free(w->decisions); free(w->deviations); free(w->speed); free(w->advance); free(w->progress);
  free(w->overshoot); free(w->joined); free(w->depart); free(w->arrive); free(w->latency_debt);
  free(w->driving); free(w->queued); free(w->lat_steps); free(w->path_len_mm); free(w->state);
  if (w->path) for (int32_t i = 0; i < w->V; ++i) free(w->path[i].a);
  if (w->plan) for (int32_t i = 0; i < w->V; ++i) free(w->plan[i].a);
  free(w->path); free(w->plan); free(w->plan_step); free(w->plan_done); free(w->dep); free(w->occ);
  free(w->dec_rec);
  free(w->dec_vid.a); free(w->dec_edge.a); free(w->completions.a); free(w->enq_vid.a);
  free(w);
}

static size_t nz(int64_t n) { return n > 0 ? (size_t)n : 1; }
#define ALLOC(p, n) ((p) = calloc(nz(n), sizeof(*(p))))

og_world* og_world_create(const gmaco_graph_desc* gd, const gmaco_distance_desc* dd,
                          const gmaco_sim_config* c, char* err, int32_t cap) {
  og_world* w = calloc(1, sizeof(og_world));
  if (net_build(gd, &w->g, err, cap)) { free(w); return NULL; }
  if (validate_config(c, err, cap)) { og_world_destroy(w); return NULL; }
  const int32_t n = w->g.n, m = w->g.m;
  w->cfg = *c;
  ALLOC(w->block_a, c->od_block_a_len);
  ALLOC(w->block_b, c->od_block_b_len);
  if (c->od_block_a_len > 0) memcpy(w->block_a, c->od_block_a, sizeof(int32_t) * (size_t)c->od_block_a_len);
  if (c->od_block_b_len > 0) memcpy(w->block_b, c->od_block_b, sizeof(int32_t) * (size_t)c->od_block_b_len);
  w->cfg.od_block_a = w->block_a;
  w->cfg.od_block_b = w->block_b;
  ALLOC(w->sig, n);
  for (int32_t i = 0; i < n; ++i) w->sig[i] = gd->signalized ? gd->signalized[i] : 0;

  /* distance service */
  w->dkind = dd->kind;
  if (dd->kind == GMACO_DIST_DENSE) {
    w->dense = malloc(sizeof(int64_t) * (size_t)n * (size_t)n);
    if (dd->dist_mm) memcpy(w->dense, dd->dist_mm, sizeof(int64_t) * (size_t)n * (size_t)n);
    else og_apsp(gd, w->dense, NULL);
  } else if (dd->kind == GMACO_DIST_GRID) {
    w->grows = dd->grid_rows; w->gcols = dd->grid_cols;
    if ((int64_t)w->grows * w->gcols != n || m == 0) { set_err(err, cap, "grid distance: shape mismatch"); og_world_destroy(w); return NULL; }
    w->grid_len = w->g.len[0];
  } else if (dd->kind == GMACO_DIST_TARGETS) {
    w->ntargets = dd->target_count;
    if (w->ntargets < 1) { set_err(err, cap, "targets distance: empty target set"); og_world_destroy(w); return NULL; }
    ALLOC(w->targets, w->ntargets);
    memcpy(w->targets, dd->targets, sizeof(int32_t) * (size_t)w->ntargets);
    w->slot_of = malloc(sizeof(int32_t) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) w->slot_of[i] = -1;
    w->tdist = malloc(sizeof(int64_t) * (size_t)w->ntargets * (size_t)n);
    for (int32_t t = 0; t < w->ntargets; ++t) {
      int32_t x = w->targets[t];
      if (x < 0 || x >= n || w->slot_of[x] >= 0) {
        set_err(err, cap, "targets distance: invalid or duplicate target %d", x);
        og_world_destroy(w); return NULL;
      }
      w->slot_of[x] = t;
    }
    targets_sssp(w);
  } else {
    set_err(err, cap, "unknown distance kind %d", dd->kind); og_world_destroy(w); return NULL;
  }

  w->dt_us = llround(c->dt_s * 1e6);
  w->latency_us = llround(c->decision_latency_s * 1e6);
  /* init_random (pheromone.cpp:21-32) */
  ALLOC(w->tau, m); ALLOC(w->eta_beta, m); ALLOC(w->weight, m); ALLOC(w->ecost, m);
  const gmaco_pheromone_params* p = &c->pheromone;
  for (int32_t e = 0; e < m; ++e) {
    double v = og_uniform(og_draw(c->seed, S_PHER_INIT, (uint64_t)e, 0), p->tau_init_lo, p->tau_init_hi);
    w->tau[e] = i64min(i64max(og_tau_from_double(v), min_u(p)), max_u(p));
    double vis = 1.0 / ((double)w->g.len[e] / 1000.0); /* routing.cpp:92 */
    w->eta_beta[e] = pow(vis, c->routing.aco_beta);
  }
  /* signals (engine.cpp:124-136, make_signal_state signals.cpp:29-46) */
  ALLOC(w->sig_of_node, n);
  ALLOC(w->bind_sig, m); ALLOC(w->bind_phase, m);
  for (int32_t e = 0; e < m; ++e) { w->bind_sig[e] = -1; w->bind_phase[e] = -1; }
  w->S = 0;
  for (int32_t i = 0; i < n; ++i) { w->sig_of_node[i] = w->sig[i] ? w->S : -1; if (w->sig[i]) w->S++; }
  const int32_t S = w->S;
  ALLOC(w->sig_node, S); ALLOC(w->green, S); ALLOC(w->cursor, S); ALLOC(w->dlanes, S);
  ALLOC(w->el_steps, S); ALLOC(w->el_s, S);
  ALLOC(w->q, (int64_t)S * GMACO_PHASES); ALLOC(w->head_wait, (int64_t)S * GMACO_PHASES);
  ALLOC(w->rem, (int64_t)S * GMACO_PHASES);
  for (int32_t i = 0; i < n; ++i) {
    int32_t s = w->sig_of_node[i];
    if (s < 0) continue;
    w->sig_node[s] = i;
    w->dlanes[s] = 1;
    int32_t slot = 0;
    for (int32_t k = w->g.in_ptr[i]; k < w->g.in_ptr[i + 1]; ++k, ++slot) {
      int32_t e = w->g.in_edge[k];
      w->bind_sig[e] = s;
      w->bind_phase[e] = slot % GMACO_PHASES;
      int32_t ln = gd->edge_lanes ? gd->edge_lanes[e] : 1;
      if (ln > w->dlanes[s]) w->dlanes[s] = ln;
    }
    w->cursor[s] = c->signal.fixed_cycle_order[GMACO_PHASES - 1];
    w->green[s] = w->cursor[s];
    w->el_s[s] = c->signal.green_duration_s;
    w->el_steps[s] = 0;
  }
  /* vehicles */
  const int32_t V = c->vehicle_count;
  w->V = V; w->vlo = 0; w->vhi = V;
  ALLOC(w->origin, V); ALLOC(w->dest, V); ALLOC(w->at_node, V); ALLOC(w->on_edge, V);
  ALLOC(w->queued_phase, V); ALLOC(w->decisions, V); ALLOC(w->deviations, V); ALLOC(w->speed, V);
  ALLOC(w->advance, V); ALLOC(w->progress, V); ALLOC(w->overshoot, V); ALLOC(w->joined, V);
  ALLOC(w->depart, V); ALLOC(w->arrive, V); ALLOC(w->latency_debt, V); ALLOC(w->driving, V);
  ALLOC(w->queued, V); ALLOC(w->lat_steps, V); ALLOC(w->path_len_mm, V); ALLOC(w->state, V);
  ALLOC(w->path, V); ALLOC(w->plan, V); ALLOC(w->plan_step, V); ALLOC(w->plan_done, V);
  ALLOC(w->dec_rec, V);
  for (int32_t i = 0; i < V; ++i) {
    w->at_node[i] = -1; w->on_edge[i] = -1; w->queued_phase[i] = -1; w->arrive[i] = -1;
    w->state[i] = GMACO_PENDING;
    w->plan_step[i] = -1;
  }
  if (spawn(w, err, cap)) { og_world_destroy(w); return NULL; }
  ALLOC(w->occ, m);
  ALLOC(w->dep, m);
  refresh_edge_terms(w);
  return w;
}

/* ---- stages (engine.cpp:154-324) ----------------------------------------- */
static int64_t count_active(const og_world* w) { /* engine.cpp:156-173 */
  int64_t n = 0;
  for (int32_t i = 0; i < w->V; ++i) {
    uint8_t s = w->state[i];
    if (s == GMACO_AT_NODE || s == GMACO_ON_EDGE || s == GMACO_QUEUED) ++n;
    else if (s == GMACO_PENDING && w->depart[i] == w->step) ++n;
  }
  return n;
}

static void take_edge(og_world* w, int32_t vid, int32_t e, int deviated) { /* engine.cpp:207-216 */
  w->state[vid] = GMACO_ON_EDGE;
  w->on_edge[vid] = e;
  w->progress[vid] = w->overshoot[vid];
  w->overshoot[vid] = 0;
  w->latency_debt[vid] += w->latency_us;
  w->decisions[vid]++;
  if (deviated) w->deviations[vid]++;
  ivec_push(&w->path[vid], e);
  w->path_len_mm[vid] += w->g.len[e];
  ivec_push(&w->dec_vid, vid);
  ivec_push(&w->dec_edge, e);
  w->ctr.decisions++;
}

static void activate(og_world* w, int32_t vid) { /* engine.cpp:177-180 */
  if (w->state[vid] == GMACO_PENDING && w->depart[vid] == w->step) {
    w->state[vid] = GMACO_AT_NODE;
    w->at_node[vid] = w->origin[vid];
  }
}

static void decide(og_world* w, int32_t vid) { /* engine.cpp:175-217 */
  activate(w, vid);
  if (vid < w->vlo || vid >= w->vhi) return; /* sharded: another shard decides (apply_remote) */
  w->dec_rec[vid] = -1;
  if (w->state[vid] != GMACO_AT_NODE) return;
  int32_t next = -1;
  int dev = 0;
  int32_t e = route_one(w, w->cfg.algorithm, w->at_node[vid], w->dest[vid], (uint64_t)vid,
                        (uint64_t)w->step, w->active, 0, &next, &dev);
  if (e < 0) { w->state[vid] = GMACO_RETIRED; w->dec_rec[vid] = -2; return; }
  w->ctr.ant_steps++;
  take_edge(w, vid, e, dev);
  w->dec_rec[vid] = e | (dev ? GMACO_REC_DEVIATED : 0);
}

/* Colony stage B (north-star extension): K ants per planning vehicle, best
 * tour by (cost, ant), winner replayed to materialize its tour; vehicles at
 * a node take the winner's first hop. */
/* Colony stage B for one vehicle: its K ants' walks, the winner's tour as
 * the vehicle's plan.  Touches only the vehicle's own state and plan, so the
 * vehicles of a step are planned on all host threads (colony_stage); the
 * shared effects -- counters, deposits, the decision's take_edge -- are
 * returned and applied in ascending vid by the caller. */
static void colony_plan_vehicle(og_world* w, int32_t vid, og_ctr_local* ctr, int64_t* dep_amount,
                                int32_t* decide_edge) {
  *dep_amount = 0;
  *decide_edge = -1;
  activate(w, vid);
  if (vid < w->vlo || vid >= w->vhi) return;
  w->dec_rec[vid] = -1;
  const gmaco_colony_params* cp = &w->cfg.colony;
  int32_t start = -1;
  const int deciding = w->state[vid] == GMACO_AT_NODE;
  if (deciding) start = w->at_node[vid];
  else if (cp->replan_all && w->state[vid] == GMACO_QUEUED) start = w->at_node[vid];
  else if (cp->replan_all && w->state[vid] == GMACO_ON_EDGE) start = w->g.to[w->on_edge[vid]];
  if (start < 0) return;
  if (start == w->dest[vid]) { w->plan[vid].n = 0; w->plan_step[vid] = w->step; w->plan_done[vid] = 0; return; }
  int64_t best = INF64;
  int32_t winner = 0;
  int first_ok = 0;
  for (int32_t a = 0; a < cp->ants; ++a) {
    int64_t cost;
    int ok;
    ant_walk(w, vid, a, start, w->dest[vid], &cost, NULL, &ok, ctr);
    if (a == 0) first_ok = ok;
    if (cost < best) { best = cost; winner = a; }
  }
  if (!first_ok) {
    w->plan[vid].n = 0;
    w->plan_step[vid] = w->step;
    w->plan_done[vid] = 0;
    if (deciding) {
      w->state[vid] = GMACO_RETIRED;
      w->dec_rec[vid] = -2;
    }
    return;
  }
  const int32_t max_hops = cp->max_hops > 0 ? cp->max_hops : w->g.n - 1;
  ivec* pl = &w->plan[vid];
  if (pl->cap < max_hops + 1) { pl->cap = max_hops + 1; pl->a = realloc(pl->a, sizeof(int32_t) * (size_t)pl->cap); }
  int64_t cost;
  int ok;
  pl->n = ant_walk(w, vid, winner, start, w->dest[vid], &cost, pl->a, &ok, NULL);
  w->plan_step[vid] = w->step;
  w->plan_done[vid] = pl->n > 0 && w->g.to[pl->a[pl->n - 1]] == w->dest[vid];
  ctr->vehicle_routes++;
  if (w->plan_done[vid] && w->cfg.colony.deposit == GMACO_DEPOSIT_BEST_TOUR) {
    /* best-tour deposit: deposit_amount(tour length) per tour edge, summed
     * exactly per edge; applied (sum-then-clamp) in stage F */
    int64_t len = 0;
    for (int32_t i = 0; i < pl->n; ++i) len += w->g.len[pl->a[i]];
    *dep_amount = og_deposit_amount(len, &w->cfg.pheromone);
  }
  if (deciding) *decide_edge = pl->a[0];
}

typedef struct {
  og_world* w;
  int64_t* dep_amount;
  int32_t* decide_edge;
  og_ctr_local ctr[64];
  int32_t slots, cursor; /* threads registered; next vehicle */
  pthread_mutex_t mu;
} colony_job;

static void* colony_worker(void* arg) {
  colony_job* j = (colony_job*)arg;
  pthread_mutex_lock(&j->mu);
  og_ctr_local* ctr = &j->ctr[j->slots++];
  pthread_mutex_unlock(&j->mu);
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int32_t lo = j->cursor;
    if (j->cursor < j->w->V) j->cursor += 16;
    pthread_mutex_unlock(&j->mu);
    if (lo >= j->w->V) return NULL;
    const int32_t hi = lo + 16 < j->w->V ? lo + 16 : j->w->V;
    for (int32_t vid = lo; vid < hi; ++vid) colony_plan_vehicle(j->w, vid, ctr, &j->dep_amount[vid], &j->decide_edge[vid]);
  }
}

/* Colony stage B for the whole fleet: per-vehicle planning on all host
 * threads, then the shared effects in ascending vid (deposits are exact
 * integer sums, so their order is immaterial; take_edge keeps vid order). */
static void colony_stage(og_world* w) {
  const int32_t V = w->V;
  colony_job j;
  memset(&j, 0, sizeof j);
  j.w = w;
  j.dep_amount = calloc((size_t)(V ? V : 1), sizeof(int64_t));
  j.decide_edge = malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
  pthread_mutex_init(&j.mu, NULL);
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  if ((int64_t)V * (w->cfg.colony.ants > 0 ? w->cfg.colony.ants : 1) < 4096) nt = 1; /* small worlds: no threads */
  if (nt == 1) {
    colony_worker(&j);
  } else {
    pthread_t th[64];
    for (long i = 0; i < nt; ++i) pthread_create(&th[i], NULL, colony_worker, &j);
    for (long i = 0; i < nt; ++i) pthread_join(th[i], NULL);
  }
  pthread_mutex_destroy(&j.mu);
  for (int i = 0; i < 64; ++i) {
    w->ctr.ant_steps += j.ctr[i].ant_steps;
    w->ctr.candidates += j.ctr[i].candidates;
    w->ctr.degree_sum += j.ctr[i].degree_sum;
    w->ctr.vehicle_routes += j.ctr[i].vehicle_routes;
  }
  for (int32_t vid = 0; vid < V; ++vid) {
    if (j.dep_amount[vid]) {
      const ivec* pl = &w->plan[vid];
      for (int32_t i = 0; i < pl->n; ++i) w->dep[pl->a[i]] += j.dep_amount[vid];
    }
    if (j.decide_edge[vid] >= 0) {
      take_edge(w, vid, j.decide_edge[vid], 0);
      w->dec_rec[vid] = j.decide_edge[vid];
    }
  }
  free(j.dep_amount);
  free(j.decide_edge);
}

static void assign(og_world* w, int32_t s) { /* engine.cpp:223-239 */
  if (w->el_s[s] < w->cfg.signal.green_duration_s) return;
  int32_t ql[GMACO_PHASES];
  for (int ph = 0; ph < GMACO_PHASES; ++ph) ql[ph] = (int32_t)w->q[s * GMACO_PHASES + ph].size;
  int ph = og_select_phase(w->cfg.controller, ql, w->head_wait + (size_t)s * GMACO_PHASES, w->cursor[s],
                           &w->cfg.signal);
  w->green[s] = ph; /* assign_green, signals.cpp:111-117 */
  w->cursor[s] = ph;
  w->el_s[s] = 0.0;
  w->el_steps[s] = 0;
  w->rem[s * GMACO_PHASES + ph] = 0.0;
}

static void discharge_signal(og_world* w, int32_t s) { /* engine.cpp:241-252, signals.cpp:119-135 */
  const int64_t k = (int64_t)s * GMACO_PHASES + w->green[s];
  fifo* q = &w->q[k];
  int budget = discharge_budget(&w->rem[k], w->cfg.dt_s, w->dlanes[s], &w->cfg.signal);
  while (budget > 0 && q->size > 0) {
    int32_t vid = q->vid[q->head];
    q->head++; q->size--;
    --budget;
    w->queued[vid] += w->step - w->joined[vid] + 1;
    w->state[vid] = GMACO_AT_NODE;
    w->at_node[vid] = w->sig_node[s];
    w->queued_phase[vid] = -1;
  }
  if (q->size == 0) { w->head_wait[k] = 0.0; q->head = 0; }
}

static void move(og_world* w, int32_t vid) { /* engine.cpp:254-295 */
  if (w->state[vid] != GMACO_ON_EDGE) return;
  if (w->latency_debt[vid] >= w->dt_us) {
    w->latency_debt[vid] -= w->dt_us;
    w->lat_steps[vid]++;
    return;
  }
  w->progress[vid] += w->advance[vid];
  w->driving[vid]++;
  const int32_t e = w->on_edge[vid];
  if (w->progress[vid] < w->g.len[e]) return;
  const int64_t overshoot = w->progress[vid] - w->g.len[e];
  const int32_t reached = w->g.to[e];
  if (reached == w->dest[vid]) {
    w->state[vid] = GMACO_ARRIVED;
    w->arrive[vid] = w->step + 1;
    ivec_push(&w->completions, vid);
    return;
  }
  if (w->bind_sig[e] >= 0) {
    w->state[vid] = GMACO_QUEUED;
    w->at_node[vid] = reached;
    w->queued_phase[vid] = w->bind_phase[e];
    w->joined[vid] = w->step + 1;
    w->progress[vid] = 0;
    ivec_push(&w->enq_vid, vid);
    return;
  }
  w->state[vid] = GMACO_AT_NODE;
  w->at_node[vid] = reached;
  w->overshoot[vid] = overshoot;
  w->progress[vid] = 0;
}

static void update_timers(og_world* w, int32_t s) { /* engine.cpp:303-314 */
  const int64_t now = w->step + 1;
  for (int ph = 0; ph < GMACO_PHASES; ++ph) {
    const int64_t k = (int64_t)s * GMACO_PHASES + ph;
    fifo* q = &w->q[k];
    w->head_wait[k] = q->size == 0 ? 0.0 : (double)(now - q->enq[q->head]) * w->cfg.dt_s;
  }
  w->el_steps[s]++;
  w->el_s[s] = (double)w->el_steps[s] * w->cfg.dt_s;
}

static void aco_deposit_path(og_world* w, const int32_t* path, int32_t n, int64_t len_mm) {
  /* apply_aco_deposit, pheromone.cpp:80-90 */
  if (n == 0) return;
  const int64_t amount = og_deposit_amount(len_mm, &w->cfg.pheromone);
  const int64_t hi = max_u(&w->cfg.pheromone);
  for (int32_t i = 0; i < n; ++i) w->tau[path[i]] = i64min(w->tau[path[i]] + amount, hi);
}

/* The step's decisions in ascending vid (commit_pheromone's order,
 * parallel.cpp:195-231).  A sharded world applied its own shard's decisions
 * in stage B and the others' in apply_remote, so its lists are re-sorted. */
static void decisions_in_vid_order(og_world* w) {
  if (w->vlo == 0 && w->vhi == w->V) return;
  int32_t* edge_of = malloc(sizeof(int32_t) * (size_t)(w->V ? w->V : 1));
  for (int32_t v = 0; v < w->V; ++v) edge_of[v] = -1;
  for (int32_t i = 0; i < w->dec_vid.n; ++i) edge_of[w->dec_vid.a[i]] = w->dec_edge.a[i];
  int32_t k = 0;
  for (int32_t v = 0; v < w->V; ++v)
    if (edge_of[v] >= 0) { w->dec_vid.a[k] = v; w->dec_edge.a[k] = edge_of[v]; k++; }
  free(edge_of);
}

static void pheromone_commit(og_world* w) { /* engine.cpp:326-350, parallel.cpp:195-258 */
  const gmaco_pheromone_params* p = &w->cfg.pheromone;
  const int alg = w->cfg.algorithm;
  if (alg == GMACO_MACO || alg == GMACO_MACO_P) {
    decisions_in_vid_order(w);
    if (p->decrement_siblings_only) { /* apply_maco_update_scoped, pheromone.cpp:48-59 */
      const int64_t lo = min_u(p), hi = max_u(p), inc = inc_u(p), dec = dec_u(p);
      for (int32_t i = 0; i < w->dec_vid.n; ++i) {
        int32_t chosen = w->dec_edge.a[i], u = w->g.from[chosen];
        w->tau[chosen] = i64min(w->tau[chosen] + inc, hi);
        for (int32_t k = w->g.out_ptr[u]; k < w->g.out_ptr[u + 1]; ++k) {
          int32_t e = w->g.out_edge[k];
          if (e == chosen) continue;
          w->tau[e] = i64max(w->tau[e] - dec, lo);
        }
      }
      return;
    }
    const int32_t D = w->dec_vid.n;
    if (D == 0) return;
    /* fold: positions per edge (parallel.cpp:213-230) */
    int32_t* cnt = calloc((size_t)w->g.m + 1, sizeof(int32_t));
    for (int32_t i = 0; i < D; ++i) cnt[w->dec_edge.a[i] + 1]++;
    for (int32_t e = 0; e < w->g.m; ++e) cnt[e + 1] += cnt[e];
    int32_t* pos = malloc(sizeof(int32_t) * (size_t)D);
    int32_t* cur = malloc(sizeof(int32_t) * ((size_t)w->g.m + 1));
    memcpy(cur, cnt, sizeof(int32_t) * ((size_t)w->g.m + 1));
    for (int32_t i = 0; i < D; ++i) pos[cur[w->dec_edge.a[i]]++] = i;
    for (int32_t e = 0; e < w->g.m; ++e)
      w->tau[e] = og_fold_maco_edge(w->tau[e], pos + cnt[e], cnt[e + 1] - cnt[e], D, p);
    free(cnt); free(pos); free(cur);
    return;
  }
  const int deposit_completion =
      alg == GMACO_ACO || (alg == GMACO_COLONY && w->cfg.colony.deposit == GMACO_DEPOSIT_COMPLETION);
  if (deposit_completion) {
    for (int32_t i = 0; i < w->completions.n; ++i) {
      int32_t vid = w->completions.a[i];
      aco_deposit_path(w, w->path[vid].a, w->path[vid].n, w->path_len_mm[vid]);
    }
  } else if (alg == GMACO_COLONY && w->cfg.colony.deposit == GMACO_DEPOSIT_BEST_TOUR) {
    /* best-tour deposit: every planned tour that reaches its destination adds
     * deposit_amount(tour length) to its edges; sum-then-clamp is exact. */
    const int64_t hi = max_u(p);
    for (int32_t e = 0; e < w->g.m; ++e) {
      if (w->dep[e]) w->tau[e] = i64min(w->tau[e] + w->dep[e], hi);
      w->dep[e] = 0;
    }
  }
}

/* ---- stage G + occupancy (pheromone.cpp:61-71, engine.cpp:316-322) ------- */
static void refresh_occupancy(og_world* w) {
  memset(w->occ, 0, sizeof(int32_t) * (size_t)w->g.m);
  for (int32_t i = 0; i < w->V; ++i)
    if (w->state[i] == GMACO_ON_EDGE) w->occ[w->on_edge[i]]++;
  for (int32_t e = 0; e < w->g.m; ++e)
    if (w->occ[e] > w->max_occ) w->max_occ = w->occ[e];
}

static void evaporate(og_world* w) {
  const gmaco_pheromone_params* p = &w->cfg.pheromone;
  const int cong = w->cfg.algorithm == GMACO_COLONY && w->cfg.colony.congestion_evaporation;
  const int64_t lo = min_u(p), dec = dec_u(p);
  for (int32_t e = 0; e < w->g.m; ++e) {
    int64_t t = og_evaporate_one(w->tau[e], p);
    /* colony congestion term: occupied edges lose dec per vehicle */
    if (cong && w->occ[e] > 0) t = i64max(lo, t - dec * (int64_t)w->occ[e]);
    w->tau[e] = t;
  }
}

/* sequential_step (engine.cpp:352-400).  Occupancy is refreshed before F/G
 * (the reference refreshes after G); neither F nor G reads it and the
 * refresh reads no pheromone, so the order is immaterial except that the
 * colony congestion term sees this step's occupancy. */
static void step_part1(og_world* w) {
  w->dec_vid.n = 0; w->dec_edge.n = 0; w->completions.n = 0; w->enq_vid.n = 0;
  w->active = count_active(w);
  /* B */
  if (w->cfg.algorithm == GMACO_COLONY)
    colony_stage(w);
  else
    for (int32_t vid = 0; vid < w->V; ++vid) decide(w, vid);
}

/* Sharded protocol: apply the other shards' decision records. */
static void apply_remote(og_world* w) {
  if (w->vlo == 0 && w->vhi == w->V) return;
  for (int32_t vid = 0; vid < w->V; ++vid) {
    if (vid >= w->vlo && vid < w->vhi) continue;
    const int32_t rec = w->dec_rec[vid];
    if (rec >= 0) take_edge(w, vid, rec & ~GMACO_REC_DEVIATED, (rec & GMACO_REC_DEVIATED) != 0);
    else if (rec == -2) w->state[vid] = GMACO_RETIRED;
  }
}

static void step_part2(og_world* w) {
  apply_remote(w);
  /* C */
  int64_t qt = 0;
  for (int64_t k = 0; k < (int64_t)w->S * GMACO_PHASES; ++k) qt += w->q[k].size;
  w->qtotal += qt;
  w->qsamples += w->S;
  /* D, E1 */
  for (int32_t s = 0; s < w->S; ++s) assign(w, s);
  for (int32_t s = 0; s < w->S; ++s) discharge_signal(w, s);
  /* E2 */
  for (int32_t vid = 0; vid < w->V; ++vid) move(w, vid);
  /* E3: enqueue commit in ascending vid, then timers */
  for (int32_t i = 0; i < w->enq_vid.n; ++i) {
    int32_t vid = w->enq_vid.a[i];
    int32_t e = w->on_edge[vid];
    fifo_push(&w->q[(int64_t)w->bind_sig[e] * GMACO_PHASES + w->bind_phase[e]], vid, w->joined[vid]);
  }
  for (int32_t s = 0; s < w->S; ++s) update_timers(w, s);
  refresh_occupancy(w);
  /* F, G */
  pheromone_commit(w);
  evaporate(w);
  refresh_edge_terms(w);
  w->step++;
}

static void step(og_world* w) {
  step_part1(w);
  step_part2(w);
}

int og_world_finished(og_world* w) { /* engine.cpp:146-152 */
  if (w->step >= w->cfg.max_steps) return 1;
  for (int32_t i = 0; i < w->V; ++i)
    if (w->state[i] != GMACO_ARRIVED && w->state[i] != GMACO_RETIRED) return 0;
  return 1;
}

int64_t og_world_step(og_world* w, int64_t n) {
  int64_t k = 0;
  for (; k < n && !og_world_finished(w); ++k) step(w);
  return k;
}

int64_t og_world_current_step(og_world* w) { return w->step; }

int og_world_collect(og_world* w, gmaco_run_result* r, double* travel, int32_t* rvid,
                     int32_t* rnode, int32_t cap) { /* collect_result, engine.cpp:402-433 */
  memset(r, 0, sizeof(*r));
  r->steps_executed = w->step;
  double ts = 0.0, ws = 0.0;
  int32_t k = 0;
  for (int32_t i = 0; i < w->V; ++i) {
    if (travel) travel[i] = -1.0;
    if (w->state[i] == GMACO_ARRIVED) {
      double t = (double)(w->arrive[i] - w->depart[i]) * w->cfg.dt_s;
      if (travel) travel[i] = t;
      ts += t;
      ws += (double)w->queued[i] * w->cfg.dt_s + (double)w->decisions[i] * w->cfg.decision_latency_s;
      r->completed_count++;
    } else if (w->state[i] == GMACO_RETIRED) {
      r->retired_count++;
      if (k < cap) {
        if (rvid) rvid[k] = i;
        if (rnode) rnode[k] = w->at_node[i];
      }
      ++k;
    }
  }
  if (r->completed_count > 0) {
    r->mean_travel_s = ts / r->completed_count;
    r->mean_wait_s = ws / r->completed_count;
  }
  if (w->qsamples > 0) r->mean_queue_len = (double)w->qtotal / (double)w->qsamples;
  r->max_edge_occupancy = w->max_occ;
  return 0;
}

/* ---- snapshots ----------------------------------------------------------- */
int og_world_vehicles(og_world* w, const gmaco_vehicle_view* v) {
  for (int32_t i = 0; i < w->V; ++i) {
    if (v->origin) v->origin[i] = w->origin[i];
    if (v->dest) v->dest[i] = w->dest[i];
    if (v->speed_mps) v->speed_mps[i] = w->speed[i];
    if (v->advance_mm) v->advance_mm[i] = w->advance[i];
    if (v->state) v->state[i] = w->state[i];
    if (v->at_node) v->at_node[i] = w->at_node[i];
    if (v->on_edge) v->on_edge[i] = w->on_edge[i];
    if (v->progress_mm) v->progress_mm[i] = w->progress[i];
    if (v->overshoot_mm) v->overshoot_mm[i] = w->overshoot[i];
    if (v->queued_phase) v->queued_phase[i] = w->queued_phase[i];
    if (v->queue_joined_step) v->queue_joined_step[i] = w->joined[i];
    if (v->depart_step) v->depart_step[i] = w->depart[i];
    if (v->arrive_step) v->arrive_step[i] = w->arrive[i];
    if (v->latency_debt_us) v->latency_debt_us[i] = w->latency_debt[i];
    if (v->driving_steps) v->driving_steps[i] = w->driving[i];
    if (v->queued_steps) v->queued_steps[i] = w->queued[i];
    if (v->latency_steps) v->latency_steps[i] = w->lat_steps[i];
    if (v->decisions) v->decisions[i] = w->decisions[i];
    if (v->deviations) v->deviations[i] = w->deviations[i];
    if (v->path_length_mm) v->path_length_mm[i] = w->path_len_mm[i];
  }
  return 0;
}

int32_t og_world_signal_count(og_world* w) { return w->S; }

int og_world_signals(og_world* w, const gmaco_signal_view* v, int64_t cap) {
  int64_t qi = 0;
  for (int32_t s = 0; s < w->S; ++s) {
    if (v->node) v->node[s] = w->sig_node[s];
    if (v->green) v->green[s] = w->green[s];
    if (v->cycle_cursor) v->cycle_cursor[s] = w->cursor[s];
    if (v->discharge_lanes) v->discharge_lanes[s] = w->dlanes[s];
    if (v->green_elapsed_steps) v->green_elapsed_steps[s] = w->el_steps[s];
    if (v->green_elapsed_s) v->green_elapsed_s[s] = w->el_s[s];
    for (int ph = 0; ph < GMACO_PHASES; ++ph) {
      const int64_t k = (int64_t)s * GMACO_PHASES + ph;
      const fifo* q = &w->q[k];
      if (v->queue_len) v->queue_len[k] = (int32_t)q->size;
      if (v->head_wait_s) v->head_wait_s[k] = w->head_wait[k];
      if (v->service_remainder) v->service_remainder[k] = w->rem[k];
      for (int64_t j = 0; j < q->size; ++j, ++qi)
        if (qi < cap) {
          if (v->queue_vid) v->queue_vid[qi] = q->vid[q->head + j];
          if (v->queue_enqueue_step) v->queue_enqueue_step[qi] = q->enq[q->head + j];
        }
    }
  }
  return qi > cap ? 1 : 0;
}

int og_world_pheromone(og_world* w, int64_t* tau) {
  memcpy(tau, w->tau, sizeof(int64_t) * (size_t)w->g.m);
  return 0;
}

int og_world_set_pheromone(og_world* w, const int64_t* tau) {
  memcpy(w->tau, tau, sizeof(int64_t) * (size_t)w->g.m);
  refresh_edge_terms(w);
  return 0;
}

int og_world_occupancy(og_world* w, int32_t* occ) {
  memcpy(occ, w->occ, sizeof(int32_t) * (size_t)w->g.m);
  return 0;
}

int og_world_route(og_world* w, int32_t vid, int32_t planned, int32_t* out, int32_t cap, int32_t* len) {
  if (vid < 0 || vid >= w->V) return 1;
  const ivec* p = planned ? &w->plan[vid] : &w->path[vid];
  *len = p->n;
  for (int32_t i = 0; i < p->n && i < cap; ++i) out[i] = p->a[i];
  return 0;
}

int og_world_counters(og_world* w, gmaco_counters* c) {
  *c = w->ctr;
  return 0;
}

int og_world_next_node(og_world* w, int algorithm, int32_t count, const int32_t* current,
                       const int32_t* dest, const uint64_t* entity, const uint64_t* stp, int64_t n_t,
                       int32_t* out_next, int32_t* out_via, uint8_t* out_dev) {
  for (int32_t i = 0; i < count; ++i) {
    int32_t next = -1;
    int dev = 0;
    int32_t e = route_one(w, algorithm, current[i], dest[i], entity ? entity[i] : 0, stp ? stp[i] : 0,
                          n_t, 1, &next, &dev);
    out_next[i] = e < 0 ? -1 : next;
    out_via[i] = e;
    out_dev[i] = (uint8_t)(e < 0 ? 0 : dev);
  }
  return 0;
}

int og_world_set_vehicle_range(og_world* w, int32_t lo, int32_t hi) {
  if (lo < 0 || hi > w->V || lo > hi) return 1;
  w->vlo = lo;
  w->vhi = hi;
  return 0;
}

/* ---- sharded protocol (multi-GPU exchange, host-mediated) ---------------- */
int og_world_step_part(og_world* w, int32_t part) {
  if (og_world_finished(w)) return 0;
  if (part == 1) step_part1(w);
  else step_part2(w);
  return 1;
}

int og_world_exchange_export(og_world* w, int32_t* decisions, int64_t* deposits) {
  if (decisions)
    for (int32_t vid = w->vlo; vid < w->vhi; ++vid) decisions[vid - w->vlo] = w->dec_rec[vid];
  if (deposits) memcpy(deposits, w->dep, sizeof(int64_t) * (size_t)w->g.m);
  return 0;
}

int og_world_exchange_import(og_world* w, const int32_t* decisions, const int64_t* deposits) {
  if (decisions) memcpy(w->dec_rec, decisions, sizeof(int32_t) * (size_t)w->V);
  if (deposits) memcpy(w->dep, deposits, sizeof(int64_t) * (size_t)w->g.m);
  return 0;
}
