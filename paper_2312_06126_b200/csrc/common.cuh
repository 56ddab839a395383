// common.cuh -- shared device helpers of the spz library (product side only).
//
// Philox4x32-10 (Salmon et al., SC'11) is implemented here independently of the
// oracle (oracle/philox.py); both follow the published algorithm and are tied
// together only by the known-answer vectors and the bit-exact index parity test.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <utility>

namespace spz {

// ------------------------------------------------------------------ Philox4x32-10
// Counter (c0..c3) = (row j, block c, step k, stream S); key = (seed_lo, seed_hi)
// (reading #13).
enum Stream : uint32_t { S_IDX = 1, S_EPS = 2, S_EPS2 = 3, S_SMOOTH = 4, S_INIT = 5 };

__host__ __device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
#else
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// idx = floor((x1 * 2^32 + x0) * F / 2^64): one 64x64->128 multiply-high.
__device__ __forceinline__ int64_t sample_index(uint64_t seed, uint64_t step, uint64_t row, uint64_t fill) {
  const uint4 x = philox(make_uint4((uint32_t)row, 0u, (uint32_t)step, S_IDX), (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t X = ((uint64_t)x.y << 32) | (uint64_t)x.x;
  return (int64_t)__umul64hi(X, fill);
}

// U(x) = (floor(x / 2^9) + 0.5) * 2^-23 -- exact in fp32.
__device__ __forceinline__ float u01(uint32_t x) { return ((float)(x >> 9) + 0.5f) * 1.1920928955078125e-07f; }

// Standard normal number q of row j in stream S (Box-Muller on one Philox block).
__device__ __forceinline__ float normal_q(uint64_t seed, uint64_t step, uint32_t stream, uint64_t row, int q) {
  const uint4 x = philox(make_uint4((uint32_t)row, (uint32_t)(q >> 2), (uint32_t)step, stream), (uint32_t)seed,
                         (uint32_t)(seed >> 32));
  const int p = (q & 3) >> 1;
  const uint32_t a = p ? x.z : x.x, b = p ? x.w : x.y;
  const float R = sqrtf(-2.0f * logf(u01(a)));
  float s, c;
  sincospif(2.0f * u01(b), &s, &c);
  return (q & 1) ? R * s : R * c;
}

// The four normals q = 4c .. 4c+3 of row j (one Philox block, two Box-Muller pairs); n[k] equals
// normal_q(seed, step, stream, row, 4c + k) bit for bit.  `pairs` = 1 skips the second pair.
__device__ __forceinline__ void normals4(uint64_t seed, uint64_t step, uint32_t stream, uint64_t row, int c, int pairs,
                                         float (&n)[4]) {
  const uint4 x = philox(make_uint4((uint32_t)row, (uint32_t)c, (uint32_t)step, stream), (uint32_t)seed,
                         (uint32_t)(seed >> 32));
  float s, co;
  const float R0 = sqrtf(-2.0f * logf(u01(x.x)));
  sincospif(2.0f * u01(x.y), &s, &co);
  n[0] = R0 * co;
  n[1] = R0 * s;
  n[2] = n[3] = 0.f;
  if (pairs > 1) {
    const float R1 = sqrtf(-2.0f * logf(u01(x.z)));
    sincospif(2.0f * u01(x.w), &s, &co);
    n[2] = R1 * co;
    n[3] = R1 * s;
  }
}

// Box-Muller pair `half` (0: x.x, x.y; 1: x.z, x.w) of the same Philox draw as normals4: bit-identical to
// normals4's n[2 half], n[2 half + 1]
__device__ __forceinline__ void normals2(uint64_t seed, uint64_t step, uint32_t stream, uint64_t row, int c, int half,
                                         float (&n)[2]) {
  const uint4 x = philox(make_uint4((uint32_t)row, (uint32_t)c, (uint32_t)step, stream), (uint32_t)seed,
                         (uint32_t)(seed >> 32));
  float s, co;
  const float R = sqrtf(-2.0f * logf(u01(half ? x.z : x.x)));
  sincospif(2.0f * u01(half ? x.w : x.y), &s, &co);
  n[0] = R * co;
  n[1] = R * s;
}

// ------------------------------------------------------------------ element types
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
// two fp32 -> one 32-bit word of two RNE bf16 (lo in the low half)
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&p);
}
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }

__host__ __device__ __forceinline__ int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
__host__ __device__ __forceinline__ int64_t cdiv(int64_t x, int64_t a) { return (x + a - 1) / a; }

// ------------------------------------------------------------------ reductions
constexpr int NSTAT = 6;  // per-block partial sums: (q1-y)^2+(q2-y)^2, q1, q2, alpha logp - minQ~ (or -Q1~), logp, SAC v1 (V-y_V)^2

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ programmatic dependent launch
// Every kernel of the update chain is launched with programmatic stream serialization:
// its launch and pre-wait prologue overlap the previous kernel's tail; pdl_wait() blocks
// until the previous grid has completed and its writes are visible (so semantics equal
// plain stream order).  Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Release/acquire fence at GPU scope (cheaper than __threadfence's sequentially consistent fence):
// publishes this thread's prior writes before a subsequent atomic, or orders an atomic's
// observation before subsequent reads.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);

}  // namespace spz

#define SPZ_CUDA_TRY(expr)                                                                            \
  do {                                                                                                \
    cudaError_t _e = (expr);                                                                          \
    if (_e != cudaSuccess) {                                                                          \
      ::spz::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" + __FILE__ + ":" +  \
                       std::to_string(__LINE__) + ")");                                               \
      return SPZ_ECUDA;                                                                               \
    }                                                                                                 \
  } while (0)
