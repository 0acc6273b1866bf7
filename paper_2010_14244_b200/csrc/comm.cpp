// comm.cpp — multi-GPU plumbing (placeholder until the NCCL exchange lands).
#include "gmaco.h"

extern "C" {
int gmaco_nccl_unique_id(void*) { return GMACO_ERUNTIME; }
int gmaco_attach_comm(gmaco_engine*, int32_t, int32_t, const void*) { return GMACO_ERUNTIME; }
}
