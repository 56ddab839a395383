// policy.cu -- batched actor inference for the samplers, the consumer of the
// spz_sync_actor payload.
//
// PAPER.md §3.2.1: the sampling processes' actions are "generate[d] ... by forward propagation"
// of the policy; §3.2.2: the test process acts deterministically.  One call maps n
// observations to n actions with the same dense layers as the update (tcgen05 bf16 GEMMs, or 3xTF32 in
// FP32 precision) and one elementwise head kernel:
//   SAC  deterministic  a = tanh(mu)            stochastic  a = tanh(mu + exp(clamp(l, lo, hi)) n)
//   TD3  deterministic  a = tanh(z)             stochastic  a = clip(tanh(z) + sigma_x n, -1, 1)
// n[j, i] = Box-Muller normal i of call row j from Philox(seed, (j, i / 4, step, S_ACT = 7)), the same
// counter layout as the update's noise streams (readings #13, #21).
#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "internal.h"
#include "tc_gemm.cuh"

namespace spz {
namespace {

constexpr uint32_t S_ACT = 7;

struct PolicyShadow {  // one weight matrix: fp32 [rows x cols] at p_off -> operand [rows x ld] at s_off
  int64_t p_off, s_off;
  int rows, cols, ld;
};

template <typename T>
__global__ void policy_shadow_kernel(const PolicyShadow* __restrict__ ents, const float* __restrict__ P, T* __restrict__ S) {
  const PolicyShadow e = ents[blockIdx.y];
  const int64_t total = (int64_t)e.rows * e.ld;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = k / e.ld;
    const int c = (int)(k - r * e.ld);
    S[e.s_off + k] = from_f<T>(c < e.cols ? P[e.p_off + r * e.cols + c] : 0.f);
  }
}

// observations [n x o] fp32 -> layer-0 operand [n x ld0] (zero padding columns)
template <typename T>
__global__ void policy_obs_kernel(const float* __restrict__ obs, int64_t n, int o, int ld0, T* __restrict__ X) {
  const int64_t total = n * ld0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = k / ld0;
    const int c = (int)(k - r * ld0);
    X[k] = from_f<T>(c < o ? obs[r * o + c] : 0.f);
  }
}

struct ActArgs {
  const float* H;  // head pre-activations [n x nout]
  float* act;      // [n x m]
  int64_t n;
  int m, nout, td3, det;
  float lo, hi, expl;
  uint64_t seed, step;
};

__global__ void policy_act_kernel(const ActArgs a) {
  pdl_wait();
  const int64_t total = a.n * a.m;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = k / a.m;
    const int i = (int)(k - j * a.m);
    const float* h = a.H + j * a.nout;
    float out;
    if (!a.td3) {
      const float mu = h[i];
      if (a.det) {
        out = tanhf(mu);
      } else {
        const float lc = fminf(fmaxf(h[a.m + i], a.lo), a.hi);
        out = tanhf(fmaf(expf(lc), normal_q(a.seed, a.step, S_ACT, (uint64_t)j, i), mu));
      }
    } else {
      out = tanhf(h[i]);
      if (!a.det) out = fminf(fmaxf(out + a.expl * normal_q(a.seed, a.step, S_ACT, (uint64_t)j, i), -1.f), 1.f);
    }
    a.act[k] = out;
  }
}

bool on_device(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace
}  // namespace spz

using namespace spz;

struct spz_policy {
  int device = 0;
  bool td3 = false, bf16 = true;
  int o = 0, m = 0, h = 0, L = 0, nout = 0, ld0 = 0;
  int64_t max_batch = 0, np = 0;
  float lo = -20.f, hi = 2.f, expl = 0.1f;
  uint64_t version = 0;
  std::vector<int> ldw;              // shadow row pitch of each layer
  std::vector<int64_t> woff, boff;   // flat offsets of W_l and b_l in P
  std::vector<int64_t> soff;         // shadow offsets
  float* P = nullptr;                // fp32 flat actor
  void* S = nullptr;                 // operand shadow of the weights
  PolicyShadow* d_ents = nullptr;
  void* X = nullptr;                 // [max_batch x ld0]
  void* A[2] = {nullptr, nullptr};   // hidden activations (ping-pong) [max_batch x h]
  float* Hout = nullptr;             // [max_batch x nout]
  float* dobs = nullptr;             // staging for host observations
  float* dact = nullptr;             // staging for host actions
  uint8_t* hdr = nullptr;            // pinned: header + re-read seq word (seqlock read)
  cudaStream_t stream = nullptr;
  std::vector<void*> allocs;
  ~spz_policy() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : allocs) cudaFree(p);
    if (hdr) cudaFreeHost(hdr);
    if (stream) cudaStreamDestroy(stream);
    if (prev >= 0) cudaSetDevice(prev);
  }
};

namespace {

spz_status palloc(spz_policy* p, void** out, size_t bytes) {
  if (cudaMalloc(out, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(SPZ_ENOMEM, "spz_policy_create: cannot allocate " + std::to_string(bytes) + " device bytes");
  }
  p->allocs.push_back(*out);
  if (cudaMemsetAsync(*out, 0, bytes, p->stream) != cudaSuccess) return fail(SPZ_ECUDA, "cudaMemsetAsync failed");
  return SPZ_OK;
}

template <typename T>
spz_status forward(spz_policy* p, int64_t n) {
  const size_t E = sizeof(T);
  for (int l = 0; l <= p->L; ++l) {
    const bool head = l == p->L;
    GemmArgs a{};
    a.K = l == 0 ? p->ld0 : p->h;
    a.N = head ? p->nout : p->h;
    a.epi = head ? EPI_BIAS_F32 : EPI_BIAS_RELU;
    a.splits = 1;
    a.k_per_split = a.K;
    a.n_groups = 1;
    GemmGroup& g = a.g[0];
    g.A = l == 0 ? p->X : p->A[(l - 1) & 1];
    g.lda = l == 0 ? p->ld0 : p->h;
    g.B = static_cast<const uint8_t*>(p->S) + p->soff[l] * E;
    g.ldb = p->ldw[l];
    g.C = head ? (void*)p->Hout : p->A[l & 1];
    g.ldc = head ? p->nout : p->h;
    g.M = (int)n;
    g.N = a.N;
    g.bias = p->P + p->boff[l];
    cudaError_t e;  // one backend per precision (no SIMT dispatch): unsupported shapes are an error
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
      if (!tc_gemm_supported(a)) return fail(SPZ_EUNSUPPORTED, "spz_policy_act: layer GEMM not supported by the bf16 tcgen05 kernel");
      e = tc_gemm_bf16(a, p->stream);
    } else {
      if (!tc_gemm_tf32_supported(a)) return fail(SPZ_EUNSUPPORTED, "spz_policy_act: layer GEMM not supported by the 3xTF32 tcgen05 kernel");
      e = tc_gemm_tf32x3(a, p->stream);
    }
    if (e != cudaSuccess) return fail(SPZ_ECUDA, std::string("spz_policy_act: layer GEMM: ") + cudaGetErrorString(e));
  }
  return SPZ_OK;
}

template <typename T>
spz_status refresh(spz_policy* p) {
  policy_shadow_kernel<T><<<dim3(32, p->L + 1), 256, 0, p->stream>>>(p->d_ents, p->P, static_cast<T*>(p->S));
  SPZ_CUDA_TRY(cudaGetLastError());
  return SPZ_OK;
}

}  // namespace

extern "C" {

spz_status spz_policy_create(const spz_policy_desc* d, spz_policy** out) {
  if (!d || !out) return fail(SPZ_EINVAL, "spz_policy_create: NULL argument");
  *out = nullptr;
  if (d->obs_dim < 1 || d->act_dim < 1 || d->act_dim > 32 || d->hidden < 16 || d->hidden % 16 || d->n_hidden < 1 ||
      d->n_hidden > 6 || d->max_batch < 1)
    return fail(SPZ_EINVAL, "spz_policy_create: bad dims (act_dim 1..32, hidden multiple of 16, 1 <= n_hidden <= 6, max_batch >= 1)");
  if (d->algo != SPZ_SAC && d->algo != SPZ_TD3 && d->algo != SPZ_DDPG && d->algo != SPZ_SACV1)
    return fail(SPZ_EINVAL, "spz_policy_create: unknown algo");
  if (d->precision != SPZ_FP32 && d->precision != SPZ_BF16) return fail(SPZ_EINVAL, "spz_policy_create: unknown precision");
  spz_status st = check_device(d->device);
  if (st != SPZ_OK) return st;
  DeviceGuard dg(d->device);
  std::unique_ptr<spz_policy> p(new spz_policy());
  p->device = d->device;
  p->td3 = d->algo == SPZ_TD3 || d->algo == SPZ_DDPG;  // deterministic tanh actor (SAC v1: SAC's head)
  p->bf16 = d->precision == SPZ_BF16;
  p->o = d->obs_dim;
  p->m = d->act_dim;
  p->h = d->hidden;
  p->L = d->n_hidden;
  p->nout = p->td3 ? p->m : 2 * p->m;
  p->max_batch = d->max_batch;
  p->lo = (float)d->log_std_min;
  p->hi = (float)d->log_std_max;
  p->expl = (float)d->expl_noise;
  if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(SPZ_ECUDA, "spz_policy_create: stream creation failed");
  if (cudaMallocHost(&p->hdr, 128) != cudaSuccess) return fail(SPZ_ENOMEM, "spz_policy_create: pinned header");
  const size_t E = p->bf16 ? 2 : 4;
  // layer-0 pitch: 128-byte rows on the bf16 tensor-core path (full-row TMA boxes), else 16-byte rows
  p->ld0 = (int)round_up(p->o, p->bf16 ? 64 : 4);
  std::vector<PolicyShadow> ents;
  int64_t off = 0, soff = 0;
  for (int l = 0; l <= p->L; ++l) {
    const int in = l == 0 ? p->o : p->h, outd = l == p->L ? p->nout : p->h;
    const int ld = l == 0 ? p->ld0 : (int)round_up(in, p->bf16 ? 8 : 4);
    p->woff.push_back(off);
    p->boff.push_back(off + (int64_t)outd * in);
    p->soff.push_back(soff);
    p->ldw.push_back(ld);
    ents.push_back({off, soff, outd, in, ld});
    off += (int64_t)outd * in + outd;
    soff += round_up((int64_t)outd * ld, 64);
  }
  p->np = off;
  const int64_t Bm = p->max_batch;
  SPZ_TRY(palloc(p.get(), (void**)&p->P, (size_t)p->np * 4));
  SPZ_TRY(palloc(p.get(), &p->S, (size_t)soff * E));
  SPZ_TRY(palloc(p.get(), (void**)&p->d_ents, ents.size() * sizeof(PolicyShadow)));
  SPZ_TRY(palloc(p.get(), &p->X, (size_t)Bm * p->ld0 * E));
  for (int i = 0; i < 2; ++i) SPZ_TRY(palloc(p.get(), &p->A[i], (size_t)Bm * p->h * E));
  SPZ_TRY(palloc(p.get(), (void**)&p->Hout, (size_t)Bm * p->nout * 4));
  SPZ_TRY(palloc(p.get(), (void**)&p->dobs, (size_t)Bm * p->o * 4));
  SPZ_TRY(palloc(p.get(), (void**)&p->dact, (size_t)Bm * p->m * 4));
  SPZ_CUDA_TRY(cudaMemcpyAsync(p->d_ents, ents.data(), ents.size() * sizeof(PolicyShadow), cudaMemcpyHostToDevice, p->stream));
  SPZ_CUDA_TRY(cudaStreamSynchronize(p->stream));
  *out = p.release();
  return SPZ_OK;
}

spz_status spz_policy_load(spz_policy* p, const void* payload, int64_t bytes, uint64_t* version) {
  if (!p || !payload) return fail(SPZ_EINVAL, "spz_policy_load: NULL argument");
  if (bytes < SPZ_SYNC_BYTES(p->np))
    return fail(SPZ_EINVAL, "spz_policy_load: buffer smaller than SPZ_SYNC_BYTES(" + std::to_string(p->np) + ")");
  DeviceGuard dg(p->device);
  const uint8_t* src = static_cast<const uint8_t*>(payload);
  const cudaMemcpyKind hk = on_device(payload) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost;
  const cudaMemcpyKind pk = on_device(payload) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  // seqlock read of the newest version v (include/spz.h): header -> seq[v & 1] must be 2v (complete) ->
  // payload of slot v & 1 -> seq[v & 1] unchanged; otherwise a writer reached that slot again: restart
  uint64_t* h0 = reinterpret_cast<uint64_t*>(p->hdr);  // the 64-byte header
  uint64_t* s1 = h0 + 8;                                // seq word re-read after the payload
  for (int attempt = 0; attempt < 64; ++attempt) {
    SPZ_CUDA_TRY(cudaMemcpyAsync(h0, src, SPZ_SYNC_HEADER_BYTES, hk, p->stream));
    SPZ_CUDA_TRY(cudaStreamSynchronize(p->stream));
    const uint64_t v = h0[0];
    if (v == 0) return fail(SPZ_ESTATE, "spz_policy_load: nothing published yet (version 0)");
    if (h0[1] != (uint64_t)p->np)
      return fail(SPZ_EINVAL, "spz_policy_load: payload holds " + std::to_string(h0[1]) + " floats, the policy needs " +
                                  std::to_string(p->np));
    const int slot = (int)(v & 1);
    if (h0[2 + slot] != 2 * v) continue;  // slot already being rewritten with v + 2
    SPZ_CUDA_TRY(cudaMemcpyAsync(p->P, src + SPZ_SYNC_HEADER_BYTES + slot * SPZ_SYNC_SLOT_BYTES(p->np),
                                 (size_t)p->np * 4, pk, p->stream));
    SPZ_CUDA_TRY(cudaMemcpyAsync(s1, src + 16 + 8 * slot, 8, hk, p->stream));
    SPZ_CUDA_TRY(cudaStreamSynchronize(p->stream));
    if (*s1 != 2 * v) continue;
        p->version = v;
    SPZ_TRY(p->bf16 ? refresh<__nv_bfloat16>(p) : refresh<float>(p));
    SPZ_CUDA_TRY(cudaStreamSynchronize(p->stream));
    if (version) *version = p->version;
    return SPZ_OK;
  }
  return fail(SPZ_ETIMEOUT, "spz_policy_load: every attempt overlapped a writer");
}

spz_status spz_policy_get_params(spz_policy* p, float* host_out, int64_t n) {
  if (!p || !host_out) return fail(SPZ_EINVAL, "spz_policy_get_params: NULL argument");
  if (n < p->np) return fail(SPZ_EINVAL, "spz_policy_get_params: output holds fewer than " + std::to_string(p->np) + " floats");
  if (p->version == 0) return fail(SPZ_ESTATE, "spz_policy_get_params: no parameters loaded");
  DeviceGuard dg(p->device);
  SPZ_CUDA_TRY(cudaMemcpyAsync(host_out, p->P, (size_t)p->np * 4, cudaMemcpyDeviceToHost, p->stream));
  SPZ_CUDA_TRY(cudaStreamSynchronize(p->stream));
  return SPZ_OK;
}

spz_status spz_policy_act(spz_policy* p, int64_t n, const float* obs, int32_t deterministic, uint64_t seed,
                          uint64_t step, float* act) {
  if (!p || !obs || !act) return fail(SPZ_EINVAL, "spz_policy_act: NULL argument");
  if (n < 0 || n > p->max_batch) return fail(SPZ_EINVAL, "spz_policy_act: n outside [0, max_batch]");
  if (p->version == 0) return fail(SPZ_ESTATE, "spz_policy_act: no parameters loaded (spz_policy_load)");
  if (n == 0) return SPZ_OK;
  DeviceGuard dg(p->device);
  const bool obs_dev = on_device(obs), act_dev = on_device(act);
  const float* dobs = obs;
  if (!obs_dev) {
    SPZ_CUDA_TRY(cudaMemcpyAsync(p->dobs, obs, (size_t)n * p->o * 4, cudaMemcpyHostToDevice, p->stream));
    dobs = p->dobs;
  }
  const int64_t nx = n * p->ld0;
  const int bx = (int)std::min<int64_t>(cdiv(nx, 256), 148 * 8);
  if (p->bf16)
    policy_obs_kernel<__nv_bfloat16><<<bx, 256, 0, p->stream>>>(dobs, n, p->o, p->ld0, static_cast<__nv_bfloat16*>(p->X));
  else
    policy_obs_kernel<float><<<bx, 256, 0, p->stream>>>(dobs, n, p->o, p->ld0, static_cast<float*>(p->X));
  SPZ_CUDA_TRY(cudaGetLastError());
  SPZ_TRY(p->bf16 ? forward<__nv_bfloat16>(p, n) : forward<float>(p, n));
  ActArgs aa{};
  aa.H = p->Hout;
  aa.act = act_dev ? act : p->dact;
  aa.n = n;
  aa.m = p->m;
  aa.nout = p->nout;
  aa.td3 = p->td3;
  aa.det = deterministic != 0;
  aa.lo = p->lo;
  aa.hi = p->hi;
  aa.expl = p->expl;
  aa.seed = seed;
  aa.step = step;
  const int ba = (int)std::min<int64_t>(cdiv(n * p->m, 256), 148 * 8);
  SPZ_CUDA_TRY(launch_pdl(policy_act_kernel, dim3(ba), dim3(256), 0, p->stream, aa));
  if (!act_dev) SPZ_CUDA_TRY(cudaMemcpyAsync(act, p->dact, (size_t)n * p->m * 4, cudaMemcpyDeviceToHost, p->stream));
  SPZ_CUDA_TRY(cudaStreamSynchronize(p->stream));
  return SPZ_OK;
}

void spz_policy_destroy(spz_policy* p) { delete p; }

}  // extern "C"
