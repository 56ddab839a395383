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

namespace spz {
// replay.cu: the deferred pack of the last pinned-host push, enqueued on `st` (caller holds r->mu and
// has ordered `st` after every reader of the records); records ev_pack and the stage's free event
cudaError_t ring_enqueue_pack(spz_replay* r, cudaStream_t st);
// replay.cu: run any deferred pack on the ring's own stream after every reader (caller holds r->mu)
cudaError_t ring_flush_pending(spz_replay* r);
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
  // pinned-host pushes: the five field arrays are DMA'd into one of two device staging buffers; the
  // record pack is deferred to the next update of the ring's only learner (enqueued on its stream
  // right before its graph: no cross-stream hand-off per update), or run on the ring stream by the
  // next ring operation that needs the records
  float* dstage[2] = {nullptr, nullptr};
  size_t dstage_bytes[2] = {0, 0};
  cudaEvent_t ev_stage_free[2] = {nullptr, nullptr};  // the pack that last read staging buffer s is done
  int next_stage = 0;
  struct PendingPack {
    bool active = false;
    int stage = 0;
    int64_t first = 0, start = 0, nn = 0, fill_after = 0;
  } pend;
  cudaStream_t stream = nullptr;
  // ordering against in-flight updates (the update reads the pool while samplers write it):
  // every write to `rec` is enqueued after the readers' last recorded reads; learners wait on ev_pack
  cudaEvent_t ev_copy = nullptr;       // pinned push: the caller's buffers have been read (H2D done)
  bool copy_pending = false;           // spz_replay_push_async: ev_copy not yet waited for
  cudaEvent_t ev_pack = nullptr;       // the last push's records are in `rec`
  uint64_t pack_gen = 0;               // packs enqueued on the ring's own stream and not synchronised by the push
                                       // (a learner waits on ev_pack only when this moved since its last wait)
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
