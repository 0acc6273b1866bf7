// kernels.h — host-side entry points of kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "device.cuh"

namespace gmaco {

struct StepResources {
  void* scan_temp = nullptr;
  size_t scan_temp_bytes = 0;
  bool capturing = false;
  int part = 0;  // 0 whole step, 1 stage-B walk only, 2 stages C..G only
  int coop_blocks = 0;  // >0: stages C..G as one cooperative launch of this many blocks
  int queue_blocks = 0; // ant-queue walker: persistent grid (one full wave)
  // sharded runs: enqueues the decision / deposit exchange between stage B
  // and the rest of the step (NCCL); null for host-mediated exchange
  cudaError_t (*exchange)(void* ctx, cudaStream_t st) = nullptr;
  void* exchange_ctx = nullptr;
};

// Enqueues one engine step (stages B..G) on `st`.  Optional events bracket
// the stage-B walk kernel (recorded as external events while capturing).
cudaError_t gather_dist(const int64_t* table, int32_t n, const int32_t* row, const int32_t* x, int32_t count,
                        int64_t* out, cudaStream_t st);
// By-target sharding exchange buffers (gmaco_capi.cpp nccl_exchange).
cudaError_t rec_pack(const DevWorld& w, int32_t* send, int32_t pad, cudaStream_t st);
cudaError_t rec_unpack(const DevWorld& w, const int32_t* recv, const int32_t* gath, int32_t count, cudaStream_t st);
cudaError_t launch_step(const DevWorld& w, const StepResources& r, cudaStream_t st,
                        cudaEvent_t walk_begin, cudaEvent_t walk_end);
size_t scan_temp_bytes(int V);
// Lattice walker records (LatRec) from the current weights and tour costs.
cudaError_t launch_lattice_rec(const DevWorld& w, cudaStream_t st);
cudaError_t launch_threshold_batch(int32_t count, const double* wa, const double* wb, uint64_t* out,
                                   cudaStream_t st);
int kernels_per_step(const DevWorld& w, const StepResources& r);
// Reference algorithms (unsharded, cooperative launch available): up to
// nsteps whole steps in one persistent cooperative launch.
bool run_coop_ok(const DevWorld& w, const StepResources& r);
cudaError_t launch_run_coop(const DevWorld& w, const StepResources& r, int64_t nsteps, cudaStream_t st);
cudaError_t configure_kernels();
int coop_tail_blocks(const DevWorld& w, int device);
int queue_blocks(const DevWorld& w, int device);
// Lattice walker: bytes of tables staged in SMEM per CTA (0: not staged).
size_t grid_smem_bytes(const DevWorld& w);
cudaError_t configure_grid_carveout(const DevWorld& w);
// Device distance service (exact multi-target SSSP over the reversed graph).
struct SsspArgs {
  int32_t n;
  const int32_t* rptr;  // [n+1] reversed CSR: in-edges of u
  const int32_t* rsrc;  // [m] tail node of each in-edge
  const int64_t* rlen;  // [m] its length (mm)
  int64_t* D;           // [T][n] distances to each target
  uint32_t* inq;        // [T][n] in-next-frontier flags
};
cudaError_t sssp_fill_seed(int64_t* D, size_t total, const int32_t* dests, int32_t T, int32_t n, uint32_t* cur,
                           cudaStream_t st);
cudaError_t sssp_run_coop(const SsspArgs& a, uint32_t* const* q, uint32_t* cnt, uint32_t count, int64_t delta,
                          int device, cudaStream_t st);
cudaError_t build_fbits(const DevWorld& w, int32_t T, uint32_t* fb, cudaStream_t st);
// per-target candidate rows (DevTT): count pairs per (t, p), scan, build, refresh
cudaError_t tt_count(const DevWorld& w, int32_t T, const int32_t* place, int32_t* units, cudaStream_t st);
cudaError_t tt_scan(const int32_t* units, int64_t* offs, int64_t count, cudaStream_t st);
cudaError_t tt_build(const DevWorld& w, int32_t T, const int32_t* place, const int64_t* offs, uint32_t* meta,
                     int64_t* base, int64_t* cstart, int4* rec, int2* sm, int2* sl, cudaStream_t st);
cudaError_t tt_refresh(const DevWorld& w, cudaStream_t st);
cudaError_t build_reach_bits(const int64_t* D, int32_t T, int32_t n, int64_t words, uint64_t* out, cudaStream_t st);
cudaError_t launch_pack(const PackDesc& d, cudaStream_t st);
// Copies `weight` into the weight half of the slot records (ant-queue walker).
cudaError_t sync_rec_weights(const DevWorld& w, cudaStream_t st);
void colony_shape(int ants, int* threads, int* vpb);
cudaError_t launch_next_node(const DevWorld& w, int algorithm, int count, const int32_t* cur,
                             const int32_t* dst, const uint64_t* entity, const uint64_t* stepk, int64_t n_t,
                             int32_t* out_next, int32_t* out_via, uint8_t* out_dev, cudaStream_t st);

}  // namespace gmaco
