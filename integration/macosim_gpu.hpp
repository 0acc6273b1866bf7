// macosim_gpu.hpp — the reference-side executor a macosim maintainer adds
// next to run() / parallel_run() (R/include/macosim/engine.hpp:209-210,
// R/include/macosim/parallel.hpp:118-124).  Same contract as parallel_run:
// the returned RunResult is identical_to run(cfg, dist) (engine.cpp:34-40).
#pragma once

#include "macosim/engine.hpp"

namespace macosim {

// Runs cfg on CUDA device `device` through the C ABI of include/gmaco.h.
// Throws ValidationError on invalid input (status 1) and std::runtime_error
// on CUDA/runtime failures (status 2) — as run() would throw.
RunResult gpu_run(const SimConfig& cfg, const DistanceTable& dist, int device = 0);
RunResult gpu_run(const SimConfig& cfg, int device = 0);

}  // namespace macosim
