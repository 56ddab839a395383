// comm.h -- the gradient-exchange transport of a row-sharded learner group.
#pragma once

#include <cuda_runtime.h>

#include <cstring>

#include "../../include/spz.h"

namespace spz {

struct Comm {
  void* handle = nullptr;  // ncclComm_t
  int world = 1, rank = 0;
};

spz_status nccl_available();
spz_status comm_init(Comm* c, const uint8_t* uid, int world, int rank);
// Sub-communicator of the ranks with the same color (ncclCommSplit), ordered by key.
spz_status comm_split(const Comm& world, int color, int key, Comm* out);
void comm_destroy(Comm* c);
// In-place broadcast of `count` fp32 from `root` (graph-capturable).
cudaError_t comm_broadcast_f32(const Comm& c, float* buf, size_t count, int root, cudaStream_t st);
// In-place SUM allreduce of `count` fp32 (or fp64) elements on `st` (graph-capturable).
cudaError_t comm_allreduce_sum(const Comm& c, void* buf, size_t count, bool f64, cudaStream_t st);

}  // namespace spz
