// internal.h -- host-side objects behind the opaque spz handles.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/spz.h"
#include "common.cuh"

namespace spz {

spz_status fail(spz_status st, const std::string& msg);
spz_status check_device(int device);

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace spz

#define SPZ_TRY(expr)            \
  do {                           \
    spz_status _s = (expr);      \
    if (_s != SPZ_OK) return _s; \
  } while (0)

struct spz_replay {
  int o = 0, m = 0, R = 0;
  int64_t C = 0;
  int64_t cursor = 0;
  int device = 0;
  float* rec = nullptr;       // [C x R] fp32, device
  float* staging = nullptr;   // pinned host staging for pushes
  size_t staging_bytes = 0;
  int64_t* d_fill = nullptr;  // fill = min(cursor, C) on the device, written in stream order by every push
  int64_t* h_fill = nullptr;  // pinned staging for it
  float* dstage = nullptr;    // device staging of the five field arrays (pinned-host pushes)
  size_t dstage_bytes = 0;
  cudaStream_t stream = nullptr;
  // ordering against in-flight updates (the update reads the pool while samplers write it):
  // every write to `rec` is enqueued after the readers' last recorded reads; learners wait on ev_pack
  cudaEvent_t ev_copy = nullptr;       // pinned push: the caller's buffers have been read (H2D done)
  cudaEvent_t ev_pack = nullptr;       // the last push's records are in `rec`
  std::vector<cudaEvent_t> readers;    // one per learner: its last enqueued update (registered at create)
  // experience transmission loss (spz_replay_track): one "sampled" bit per slot, set by every sample;
  // a push counts the unsampled records it overwrites (device) and the records that never land (host)
  uint32_t* tags = nullptr;
  unsigned long long* d_lost = nullptr;
  int64_t lost_host = 0, pushed0 = 0;
  int track_gen = 0;                   // bumped on every spz_replay_track call (learners rebuild their plan)
  std::mutex mu;
  int64_t fill() const { return cursor < C ? cursor : C; }
};
