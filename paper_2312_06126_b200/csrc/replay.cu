// replay.cu -- device-resident replay ring: create / push / sample (a1-a2 of SURVEY.md §8(a)).
//
// PAPER.md §3.3.2: the experience pool the update process reads
// "without consuming the time of the network update process".  Here the pool
// lives in HBM as fp32 records [s | a | r | d | s2 | pad] (16-byte aligned rows),
// slot(i) = i mod C, fill = min(cursor, C).
#include <algorithm>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <vector>

#include "internal.h"

namespace spz {

// ------------------------------------------------------------------ pack (device source)
__global__ void pack_records_kernel(float* __restrict__ rec, int R, int o, int m, int64_t C, int64_t first, int64_t n,
                                    const float* __restrict__ obs, const float* __restrict__ act,
                                    const float* __restrict__ rew, const float* __restrict__ nobs,
                                    const float* __restrict__ done, int64_t* __restrict__ fill_out, int64_t fill) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *fill_out = fill;  // the ring's fill after this push
  // one thread per 16-byte unit of a record (R % 4 == 0, rows 16-byte aligned); 32-bit indexing within
  // the push (n <= C rows), one conditional wrap for the slot
  const int R4 = R >> 2;
  const int total = (int)n * R4;
  const int64_t slot0 = first % C;
  const int c_a = o, c_r = o + m, c_d = o + m + 1, c_s2 = o + m + 2, c_end = 2 * o + m + 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int t = e / R4;
    const int q = e - t * R4;
    int64_t slot = slot0 + t;
    if (slot >= C) slot -= C;
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // field of column c chosen by selects (one predicated load per element, no divergent per-field loads)
      const int c = 4 * q + k;
      const float* src = c < c_a ? obs + (int64_t)t * o + c
                         : c < c_r ? act + (int64_t)t * m + (c - c_a)
                         : c == c_r ? rew + t
                         : c == c_d ? done + t
                                    : nobs + (int64_t)t * o + (c - c_s2);
      v[k] = c < c_end ? __ldg(src) : 0.f;
    }
    reinterpret_cast<float4*>(rec + slot * R)[q] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// ------------------------------------------------------------------ transmission-loss accounting
// A push lands records on slots [slot0, slot0 + n) mod C.  Each landing slot that held a tracked record
// (slot < occupied; its record global index >= pushed0) whose sampled bit is clear counts one lost
// record; the bits of the landing slots are then cleared for the new records.  One thread per slot.
__global__ void loss_account_kernel(uint32_t* __restrict__ tags, int64_t C, int64_t slot0, int64_t n, int64_t occupied,
                                    int64_t first, int64_t pushed0, unsigned long long* __restrict__ lost) {
  __shared__ unsigned cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned mine = 0;
  if (t < n) {
    const int64_t s = (slot0 + t) % C;
    if (s < occupied) {
      const int64_t old = (first - 1) - ((first - 1 - s) % C);  // the record being overwritten
      const bool sampled = (tags[s >> 5] >> (s & 31)) & 1u;
      if (old >= pushed0 && !sampled) mine = 1;
    }
  }
  if (mine) atomicAdd(&cnt, 1u);
  __syncthreads();
  if (threadIdx.x == 0 && cnt) atomicAdd(lost, (unsigned long long)cnt);
  // clear after every thread of the block has read its bit (a word may span blocks: clear bit-wise)
  if (t < n) {
    const int64_t s = (slot0 + t) % C;
    atomicAnd(&tags[s >> 5], ~(1u << (s & 31)));
  }
}

// ------------------------------------------------------------------ sample (API form)
// One warp per row group: indices from Philox, 128-bit record loads, scatter to the
// caller's separate arrays.
constexpr int SAMPLE_ROWS = 32;

__global__ void __launch_bounds__(256) sample_kernel(const float* __restrict__ rec, int R, int o, int m, int64_t fill,
                                                     uint64_t seed, uint64_t step, int64_t B, int32_t* idx_out,
                                                     float* obs, float* act, float* rew, float* nobs, float* done,
                                                     uint32_t* tags) {
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  __shared__ int64_t sidx[SAMPLE_ROWS];
  const int64_t r0 = (int64_t)blockIdx.x * SAMPLE_ROWS;
  const int nrows = (int)(B - r0 < SAMPLE_ROWS ? B - r0 : SAMPLE_ROWS);
  if (threadIdx.x < nrows) {
    const int64_t i = sample_index(seed, step, (uint64_t)(r0 + threadIdx.x), (uint64_t)fill);
    sidx[threadIdx.x] = i;
    if (idx_out) idx_out[r0 + threadIdx.x] = (int32_t)i;
    if (tags) atomicOr(&tags[i >> 5], 1u << (i & 31));  // sampled at least once
  }
  __syncthreads();
  const int R4 = R >> 2;
  for (int e = threadIdx.x; e < nrows * R4; e += blockDim.x) {
    const int r = e / R4, q = e - r * R4;
    sm4[e] = __ldg(reinterpret_cast<const float4*>(rec + sidx[r] * R) + q);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nrows * o; e += blockDim.x) {
    const int r = e / o, c = e - r * o;
    if (obs) obs[(r0 + r) * o + c] = sm[r * R + c];
    if (nobs) nobs[(r0 + r) * o + c] = sm[r * R + o + m + 2 + c];
  }
  for (int e = threadIdx.x; e < nrows * m; e += blockDim.x) {
    const int r = e / m, c = e - r * m;
    if (act) act[(r0 + r) * m + c] = sm[r * R + o + c];
  }
  if (threadIdx.x < nrows) {
    if (rew) rew[r0 + threadIdx.x] = sm[threadIdx.x * R + o + m];
    if (done) done[r0 + threadIdx.x] = sm[threadIdx.x * R + o + m + 1];
  }
}

// true if every pointer is page-locked host memory (cudaHostAlloc / cudaHostRegister / torch pin_memory)
static bool all_pinned(std::initializer_list<const float*> ps) {
  for (const float* p : ps) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (at.type != cudaMemoryTypeHost) return false;
  }
  return true;
}

static cudaError_t wait_readers(spz_replay* r) {
  for (cudaEvent_t e : r->readers) {
    cudaError_t err = cudaStreamWaitEvent(r->stream, e, 0);
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

cudaError_t ring_enqueue_pack(spz_replay* r, cudaStream_t st) {
  spz_replay::PendingPack& p = r->pend;
  if (!p.active) return cudaSuccess;
  const int o = r->o, m = r->m, R = r->R;
  const int64_t nn = p.nn;
  float* d_obs = r->dstage[p.stage];
  float* d_act = d_obs + nn * o;
  float* d_nobs = d_act + nn * m;
  float* d_rew = d_nobs + nn * o;
  float* d_done = d_rew + nn;
  if (st != r->stream) {  // on a learner stream: after the push's H2D copies (spz_replay_push_async returns before them)
    const cudaError_t we = cudaStreamWaitEvent(st, r->ev_copy, 0);
    if (we != cudaSuccess) return we;
  }
  if (r->tags && nn > 0) {
    const int64_t occupied = p.first < r->C ? p.first : r->C;
    loss_account_kernel<<<(unsigned)cdiv(nn, 256), 256, 0, st>>>(r->tags, r->C, p.start % r->C, nn, occupied, p.first,
                                                                r->pushed0, r->d_lost);
  }
  const int64_t total = nn * (R / 4);
  const int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 16);
  pack_records_kernel<<<blocks, 256, 0, st>>>(r->rec, R, o, m, r->C, p.start, nn, d_obs, d_act, d_rew, d_nobs, d_done,
                                              r->d_fill, p.fill_after);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaEventRecord(r->ev_pack, st);
  if (st == r->stream) ++r->pack_gen;
  if (e == cudaSuccess) e = cudaEventRecord(r->ev_stage_free[p.stage], st);
  p.active = false;
  return e;
}

cudaError_t ring_flush_pending(spz_replay* r) {
  if (!r->pend.active) return cudaSuccess;
  cudaError_t e = wait_readers(r);
  return e == cudaSuccess ? ring_enqueue_pack(r, r->stream) : e;
}

}  // namespace spz

using namespace spz;

extern "C" {

spz_status spz_replay_create(const spz_replay_desc* desc, spz_replay** out) {
  if (!desc || !out) return fail(SPZ_EINVAL, "spz_replay_create: NULL argument");
  *out = nullptr;
  if (desc->obs_dim < 1 || desc->act_dim < 1) return fail(SPZ_EINVAL, "spz_replay_create: obs_dim and act_dim must be >= 1");
  if (desc->capacity < 1) return fail(SPZ_EINVAL, "spz_replay_create: capacity must be >= 1 (S:193)");
  // the gather / sample kernels stage 32 records per block in shared memory (opt-in up to 227 KB)
  if ((int64_t)32 * round_up(2 * (int64_t)desc->obs_dim + desc->act_dim + 2, 4) * 4 > 227 * 1024)
    return fail(SPZ_EUNSUPPORTED, "spz_replay_create: record of 2 obs_dim + act_dim + 2 floats exceeds the 1816-float gather staging limit");
  spz_status st = check_device(desc->device);
  if (st != SPZ_OK) return st;
  auto* r = new spz_replay();
  r->o = desc->obs_dim;
  r->m = desc->act_dim;
  r->C = desc->capacity;
  r->R = (int)round_up(2 * r->o + r->m + 2, 4);
  r->device = desc->device;
  DeviceGuard dg(r->device);
  const size_t bytes = (size_t)r->C * r->R * sizeof(float);
  if (cudaMalloc(&r->rec, bytes) != cudaSuccess) {
    cudaGetLastError();
    delete r;
    return fail(SPZ_ENOMEM, "spz_replay_create: cannot allocate " + std::to_string(bytes) + " bytes for the ring");
  }
  if (cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&r->ev_copy, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&r->d_fill, sizeof(int64_t)) != cudaSuccess || cudaMallocHost(&r->h_fill, sizeof(int64_t)) != cudaSuccess ||
      cudaMemsetAsync(r->d_fill, 0, sizeof(int64_t), r->stream) != cudaSuccess ||
      cudaEventCreateWithFlags(&r->ev_pack, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&r->ev_stage_free[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&r->ev_stage_free[1], cudaEventDisableTiming) != cudaSuccess ||
      cudaMemsetAsync(r->rec, 0, bytes, r->stream) != cudaSuccess || cudaStreamSynchronize(r->stream) != cudaSuccess) {
    cudaFree(r->rec);
    delete r;
    return fail(SPZ_ECUDA, "spz_replay_create: CUDA setup failed");
  }
  *out = r;
  return SPZ_OK;
}

static spz_status push_impl(spz_replay* r, int64_t n, const float* obs, const float* act, const float* rew,
                            const float* next_obs, const float* done, int32_t src_on_device, int64_t* first, bool async) {
  if (!r) return fail(SPZ_EINVAL, "spz_replay_push: NULL ring");
  if (n < 0) return fail(SPZ_EINVAL, "spz_replay_push: n < 0");
  if (n > 0 && (!obs || !act || !rew || !next_obs || !done)) return fail(SPZ_EINVAL, "spz_replay_push: NULL field array");
  DeviceGuard dg(r->device);
  std::lock_guard<std::mutex> lk(r->mu);
  if (r->copy_pending) {  // the previous asynchronous push's buffers are read before this push returns
    SPZ_CUDA_TRY(cudaEventSynchronize(r->ev_copy));
    r->copy_pending = false;
  }
  const int64_t first_idx = r->cursor;
  if (first) *first = first_idx;
  if (n == 0) return SPZ_OK;
  // only the last C records of a push can survive
  const int64_t skip = n > r->C ? n - r->C : 0;
  const int64_t nn = n - skip;
  const int64_t start = first_idx + skip;
  const int o = r->o, m = r->m, R = r->R;
  // an earlier push's deferred pack lands first (it precedes this push); writes to the records wait for
  // every learner's last enqueued read of them
  SPZ_CUDA_TRY(ring_flush_pending(r));
  // transmission loss: records that never land, and the unsampled records the landing ones overwrite
  const auto account = [&]() -> cudaError_t {
    if (!r->tags || nn == 0) return cudaSuccess;
    r->lost_host += skip;
    const int64_t occupied = first_idx < r->C ? first_idx : r->C;
    loss_account_kernel<<<(unsigned)cdiv(nn, 256), 256, 0, r->stream>>>(r->tags, r->C, start % r->C, nn, occupied,
                                                                        first_idx, r->pushed0, r->d_lost);
    return cudaGetLastError();
  };
  if (src_on_device) {
    SPZ_CUDA_TRY(wait_readers(r));
    SPZ_CUDA_TRY(account());
    const int64_t total = nn * (R / 4);
    const int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 16);
    pack_records_kernel<<<blocks, 256, 0, r->stream>>>(r->rec, R, o, m, r->C, start, nn, obs + skip * o, act + skip * m,
                                                        rew + skip, next_obs + skip * o, done + skip, r->d_fill,
                                                        std::min(first_idx + n, r->C));
    SPZ_CUDA_TRY(cudaGetLastError());
  } else if (all_pinned({obs, act, rew, next_obs, done})) {
    // page-locked host fields: DMA them as they are into a device staging buffer (no host-side record
    // assembly); the pack is deferred (ring_enqueue_pack).  The copies read the caller's buffers, so
    // the call still waits for them.
    const int sg = r->next_stage;
    r->next_stage ^= 1;
    const size_t F = (size_t)(2 * o + m + 2);
    const size_t bytes = (size_t)nn * F * sizeof(float);
    if (r->dstage_bytes[sg] < bytes) {
      SPZ_CUDA_TRY(cudaEventSynchronize(r->ev_stage_free[sg]));
      if (r->dstage[sg]) cudaFree(r->dstage[sg]);
      r->dstage[sg] = nullptr;
      r->dstage_bytes[sg] = 0;
      SPZ_CUDA_TRY(cudaMalloc(&r->dstage[sg], bytes));
      r->dstage_bytes[sg] = bytes;
    }
    SPZ_CUDA_TRY(cudaStreamWaitEvent(r->stream, r->ev_stage_free[sg], 0));  // its previous pack has read it
    float* d_obs = r->dstage[sg];
    float* d_act = d_obs + nn * o;
    float* d_nobs = d_act + nn * m;
    float* d_rew = d_nobs + nn * o;
    float* d_done = d_rew + nn;
    const auto h2d = [&](float* dst, const float* src, int w) {
      return cudaMemcpyAsync(dst, src + skip * w, (size_t)nn * w * sizeof(float), cudaMemcpyHostToDevice, r->stream);
    };
    SPZ_CUDA_TRY(h2d(d_obs, obs, o));
    SPZ_CUDA_TRY(h2d(d_act, act, m));
    SPZ_CUDA_TRY(h2d(d_nobs, next_obs, o));
    SPZ_CUDA_TRY(h2d(d_rew, rew, 1));
    SPZ_CUDA_TRY(h2d(d_done, done, 1));
    SPZ_CUDA_TRY(cudaEventRecord(r->ev_copy, r->stream));
    if (r->tags) r->lost_host += skip;
    r->pend.active = true;
    r->pend.stage = sg;
    r->pend.first = first_idx;
    r->pend.start = start;
    r->pend.nn = nn;
    r->pend.fill_after = std::min(first_idx + n, r->C);
    // the pack waits for the staged data: on the ring stream it follows the copies; a learner stream
    // that takes it waits for ev_copy (ring_enqueue_pack callers)
    if (async) r->copy_pending = true;  // read by the time the next push (or spz_replay_sync) returns
    else SPZ_CUDA_TRY(cudaEventSynchronize(r->ev_copy));  // return once the caller's buffers are read
    r->cursor += n;
    return SPZ_OK;
  } else {
    const size_t bytes = (size_t)nn * R * sizeof(float);
    if (r->staging_bytes < bytes) {
      SPZ_CUDA_TRY(cudaStreamSynchronize(r->stream));
      if (r->staging) cudaFreeHost(r->staging);
      r->staging = nullptr;
      r->staging_bytes = 0;
      SPZ_CUDA_TRY(cudaMallocHost(&r->staging, bytes));
      r->staging_bytes = bytes;
    } else {
      SPZ_CUDA_TRY(cudaStreamSynchronize(r->stream));  // previous copy out of the staging buffer done
    }
    float* s = r->staging;
    for (int64_t t = 0; t < nn; ++t) {
      const int64_t src = t + skip;
      float* d = s + t * R;
      std::memcpy(d, obs + src * o, sizeof(float) * o);
      std::memcpy(d + o, act + src * m, sizeof(float) * m);
      d[o + m] = rew[src];
      d[o + m + 1] = done[src];
      std::memcpy(d + o + m + 2, next_obs + src * o, sizeof(float) * o);
      for (int c = 2 * o + m + 2; c < R; ++c) d[c] = 0.f;
    }
    // at most two pieces, split at the wrap point
    SPZ_CUDA_TRY(wait_readers(r));
    SPZ_CUDA_TRY(account());
    const int64_t slot = start % r->C;
    const int64_t n1 = std::min(nn, r->C - slot);
    SPZ_CUDA_TRY(cudaMemcpyAsync(r->rec + slot * R, s, (size_t)n1 * R * sizeof(float), cudaMemcpyHostToDevice, r->stream));
    *r->h_fill = std::min(first_idx + n, r->C);  // stable: this path synchronises before returning
    SPZ_CUDA_TRY(cudaMemcpyAsync(r->d_fill, r->h_fill, sizeof(int64_t), cudaMemcpyHostToDevice, r->stream));
    if (nn > n1)
      SPZ_CUDA_TRY(cudaMemcpyAsync(r->rec, s + n1 * R, (size_t)(nn - n1) * R * sizeof(float), cudaMemcpyHostToDevice, r->stream));
  }
  SPZ_CUDA_TRY(cudaEventRecord(r->ev_pack, r->stream));
  SPZ_CUDA_TRY(cudaStreamSynchronize(r->stream));
  r->cursor += n;
  return SPZ_OK;
}

spz_status spz_replay_push(spz_replay* r, int64_t n, const float* obs, const float* act, const float* rew,
                           const float* next_obs, const float* done, int32_t src_on_device, int64_t* first) {
  return push_impl(r, n, obs, act, rew, next_obs, done, src_on_device, first, false);
}

spz_status spz_replay_push_async(spz_replay* r, int64_t n, const float* obs, const float* act, const float* rew,
                                 const float* next_obs, const float* done, int32_t src_on_device, int64_t* first) {
  return push_impl(r, n, obs, act, rew, next_obs, done, src_on_device, first, true);
}

spz_status spz_replay_sync(spz_replay* r) {
  if (!r) return fail(SPZ_EINVAL, "spz_replay_sync: NULL ring");
  DeviceGuard dg(r->device);
  std::lock_guard<std::mutex> lk(r->mu);
  if (r->copy_pending) {
    SPZ_CUDA_TRY(cudaEventSynchronize(r->ev_copy));
    r->copy_pending = false;
  }
  return SPZ_OK;
}

spz_status spz_replay_sample(spz_replay* r, int64_t batch, uint64_t seed, uint64_t step, int32_t* idx, float* obs,
                             float* act, float* rew, float* next_obs, float* done) {
  if (!r) return fail(SPZ_EINVAL, "spz_replay_sample: NULL ring");
  if (batch < 0) return fail(SPZ_EINVAL, "spz_replay_sample: batch < 0");
  DeviceGuard dg(r->device);
  const int64_t F = r->fill();
  if (F < batch || F < 1) return fail(SPZ_ENODATA, "spz_replay_sample: fill " + std::to_string(F) + " < batch " + std::to_string(batch));
  if (batch == 0) return SPZ_OK;
  {
    std::lock_guard<std::mutex> lk(r->mu);
    SPZ_CUDA_TRY(ring_flush_pending(r));  // the last pinned push's records land first
    SPZ_CUDA_TRY(cudaStreamWaitEvent(r->stream, r->ev_pack, 0));  // (or were packed on a learner's stream)
  }
  const unsigned blocks = (unsigned)cdiv(batch, SAMPLE_ROWS);
  const size_t smem = (size_t)SAMPLE_ROWS * r->R * sizeof(float);
  if (smem > 48 * 1024)
    SPZ_CUDA_TRY(cudaFuncSetAttribute(sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  sample_kernel<<<blocks, 256, smem, r->stream>>>(r->rec, r->R, r->o, r->m, F, seed, step, batch, idx, obs, act, rew,
                                                  next_obs, done, r->tags);
  SPZ_CUDA_TRY(cudaGetLastError());
  SPZ_CUDA_TRY(cudaStreamSynchronize(r->stream));
  return SPZ_OK;
}

spz_status spz_replay_info(const spz_replay* r, int64_t* cursor, int64_t* fill, int64_t* capacity) {
  if (!r) return fail(SPZ_EINVAL, "spz_replay_info: NULL ring");
  if (cursor) *cursor = r->cursor;
  if (fill) *fill = r->fill();
  if (capacity) *capacity = r->C;
  return SPZ_OK;
}

spz_status spz_replay_records(const spz_replay* r, const float** records, int32_t* record_floats) {
  if (!r) return fail(SPZ_EINVAL, "spz_replay_records: NULL ring");
  if (records) *records = r->rec;
  if (record_floats) *record_floats = r->R;
  return SPZ_OK;
}

spz_status spz_replay_track(spz_replay* r, int32_t on) {
  if (!r) return fail(SPZ_EINVAL, "spz_replay_track: NULL ring");
  DeviceGuard dg(r->device);
  std::lock_guard<std::mutex> lk(r->mu);
  SPZ_CUDA_TRY(ring_flush_pending(r));  // pushes before the switch are accounted under the old setting
  SPZ_CUDA_TRY(cudaStreamSynchronize(r->stream));
  for (cudaEvent_t e : r->readers) SPZ_CUDA_TRY(cudaEventSynchronize(e));  // no update still marks the old bitmap
  if (r->tags) cudaFree(r->tags);
  if (r->d_lost) cudaFree(r->d_lost);
  r->tags = nullptr;
  r->d_lost = nullptr;
  if (on) {
    const size_t words = (size_t)cdiv(r->C, 32);
    if (cudaMalloc(&r->tags, words * 4) != cudaSuccess || cudaMalloc(&r->d_lost, 8) != cudaSuccess) {
      cudaGetLastError();
      return fail(SPZ_ENOMEM, "spz_replay_track: cannot allocate the tag bitmap");
    }
    SPZ_CUDA_TRY(cudaMemsetAsync(r->tags, 0, words * 4, r->stream));
    SPZ_CUDA_TRY(cudaMemsetAsync(r->d_lost, 0, 8, r->stream));
    SPZ_CUDA_TRY(cudaStreamSynchronize(r->stream));
  }
  r->lost_host = 0;
  r->pushed0 = r->cursor;
  ++r->track_gen;
  return SPZ_OK;
}

spz_status spz_replay_loss(spz_replay* r, int64_t* pushed, int64_t* lost, int64_t* resident_unsampled) {
  if (!r) return fail(SPZ_EINVAL, "spz_replay_loss: NULL ring");
  if (!r->tags) return fail(SPZ_ESTATE, "spz_replay_loss: tracking is off (spz_replay_track)");
  DeviceGuard dg(r->device);
  std::lock_guard<std::mutex> lk(r->mu);
  SPZ_CUDA_TRY(ring_flush_pending(r));
  for (cudaEvent_t e : r->readers) SPZ_CUDA_TRY(cudaEventSynchronize(e));
  SPZ_CUDA_TRY(cudaStreamSynchronize(r->stream));
  unsigned long long dl = 0;
  std::vector<uint32_t> bits((size_t)cdiv(r->C, 32));
  SPZ_CUDA_TRY(cudaMemcpy(&dl, r->d_lost, 8, cudaMemcpyDeviceToHost));
  SPZ_CUDA_TRY(cudaMemcpy(bits.data(), r->tags, bits.size() * 4, cudaMemcpyDeviceToHost));
  int64_t res = 0;
  const int64_t c = r->cursor, F = r->fill();
  for (int64_t s = 0; s < F; ++s) {
    const int64_t g = (c - 1) - ((c - 1 - s) % r->C);  // global index of the resident record
    if (g >= r->pushed0 && !((bits[s >> 5] >> (s & 31)) & 1u)) ++res;
  }
  if (pushed) *pushed = c - r->pushed0;
  if (lost) *lost = (int64_t)dl + r->lost_host;
  if (resident_unsampled) *resident_unsampled = res;
  return SPZ_OK;
}

void spz_replay_destroy(spz_replay* r) {
  if (!r) return;
  {
    DeviceGuard dg(r->device);
    cudaStreamSynchronize(r->stream);
    cudaFree(r->rec);
    if (r->staging) cudaFreeHost(r->staging);
    for (int sg = 0; sg < 2; ++sg) {
      if (r->dstage[sg]) cudaFree(r->dstage[sg]);
      if (r->ev_stage_free[sg]) cudaEventDestroy(r->ev_stage_free[sg]);
    }
    if (r->d_fill) cudaFree(r->d_fill);
    if (r->h_fill) cudaFreeHost(r->h_fill);
    if (r->tags) cudaFree(r->tags);
    if (r->d_lost) cudaFree(r->d_lost);
    cudaEventDestroy(r->ev_copy);
    cudaEventDestroy(r->ev_pack);
    cudaStreamDestroy(r->stream);
  }
  delete r;
}

}  // extern "C"
