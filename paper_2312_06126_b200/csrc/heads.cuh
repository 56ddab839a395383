// heads.cuh -- per-row math of the actor heads, shared by the standalone
// head kernels and the fused tcgen05 GEMM epilogues.
#pragma once

#include "common.cuh"

namespace spz {

constexpr float LN2F = 0.69314718055994530942f;
constexpr float HALF_LN_2PI_F = 0.91893853320467274178f;

__device__ __forceinline__ float softplusf(float x) { return fmaxf(x, 0.f) + log1pf(expf(-fabsf(x))); }

// Everything a head epilogue writes, for local rows r in [0, 2 Bl) of the actor pass:
// r < Bl is the s2-row j = r, r >= Bl is the s-row j = r - Bl.
struct HeadEpi {
  int m, o, Bl, ldx;   // action dim, obs dim, local batch, critic-input row pitch
  int64_t row0;        // global row id of local row 0 (row sharding)
  uint64_t seed;
  const int64_t* step_p;
  float lo, hi;        // log-sigma clamp (SAC)
  float noise, clipc;  // target smoothing (TD3)
  void* Xc;            // critic inputs [3 Bl x ldx]: a~ -> rows Bl.., a' -> rows 2 Bl..
  float *u, *a, *eps, *sig, *l;  // s-row cache, action-major [m x Bl] (TD3 uses a only)
  float *logp, *logp2;
};

// SAC: [mu | l] -> lc = clamp(l), sigma = exp(lc), u = mu + sigma eps, a = tanh u,
// log pi = sum_i [-eps^2/2 - lc - ln(2 pi)/2 - 2 (ln 2 - u - softplus(-2u))].
// One Philox block c of row r: actions i = 4c .. 4c+3 (< m) from mu4 / l4 (registers, compile-time
// indexed); one Philox call and two Box-Muller pairs serve all four.  Returns their part of log pi.
template <typename T>
__device__ __forceinline__ float sac_head_block4(const HeadEpi& h, int r, const float (&mu4)[4], const float (&l4)[4], int c) {
  const bool s2row = r < h.Bl;
  const int j = s2row ? r : r - h.Bl;
  const uint64_t step = (uint64_t)*h.step_p;
  const uint32_t stream = s2row ? S_EPS2 : S_EPS;
  T* xa = static_cast<T*>(h.Xc) + (int64_t)(s2row ? 2 * h.Bl + j : h.Bl + j) * h.ldx + h.o;
  float e4[4];
  normals4(h.seed, step, stream, (uint64_t)(h.row0 + j), c, h.m - 4 * c > 2 ? 2 : 1, e4);
  float lp = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = 4 * c + k;
    if (i >= h.m) break;
    const float l = l4[k];
    const float lc = fminf(fmaxf(l, h.lo), h.hi);
    const float sg = expf(lc);
    const float e = e4[k];
    const float u = fmaf(sg, e, mu4[k]);
    const float a = tanhf(u);
    lp += -0.5f * e * e - lc - HALF_LN_2PI_F - 2.f * (LN2F - u - softplusf(-2.f * u));
    xa[i] = from_f<T>(a);
    if (!s2row) {
      const int64_t ci = (int64_t)i * h.Bl + j;  // action-major [m x Bl]: coalesced over a warp's rows
      h.u[ci] = u;
      h.a[ci] = a;
      h.eps[ci] = e;
      h.sig[ci] = sg;
      h.l[ci] = l;
    }
  }
  return lp;
}
// Half `half` of Philox block c of row r: actions 4c + 2 half + {0, 1} (< m) from the Box-Muller pair
// `half` of the block's draw (so the work of one block can be split over two warps).
template <typename T>
__device__ __forceinline__ float sac_head_half(const HeadEpi& h, int r, const float (&mu2)[2], const float (&l2)[2], int c, int half) {
  const bool s2row = r < h.Bl;
  const int j = s2row ? r : r - h.Bl;
  const uint64_t step = (uint64_t)*h.step_p;
  const uint32_t stream = s2row ? S_EPS2 : S_EPS;
  T* xa = static_cast<T*>(h.Xc) + (int64_t)(s2row ? 2 * h.Bl + j : h.Bl + j) * h.ldx + h.o;
  float e2[2];
  normals2(h.seed, step, stream, (uint64_t)(h.row0 + j), c, half, e2);
  float lp = 0.f;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = 4 * c + 2 * half + k;
    if (i >= h.m) break;
    const float l = l2[k];
    const float lc = fminf(fmaxf(l, h.lo), h.hi);
    const float sg = expf(lc);
    const float e = e2[k];
    const float u = fmaf(sg, e, mu2[k]);
    const float a = tanhf(u);
    lp += -0.5f * e * e - lc - HALF_LN_2PI_F - 2.f * (LN2F - u - softplusf(-2.f * u));
    xa[i] = from_f<T>(a);
    if (!s2row) {
      const int64_t ci = (int64_t)i * h.Bl + j;
      h.u[ci] = u;
      h.a[ci] = a;
      h.eps[ci] = e;
      h.sig[ci] = sg;
      h.l[ci] = l;
    }
  }
  return lp;
}
// Philox blocks c = b0, b0 + bstep, ... of row r from the head row arrays mu[0..m), lraw[0..m).
template <typename T>
__device__ __forceinline__ float sac_head_blocks(const HeadEpi& h, int r, const float* mu, const float* lraw, int b0,
                                                 int bstep) {
  float lp = 0.f;
  for (int c = b0; 4 * c < h.m; c += bstep) {
    float mu4[4], l4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = min(4 * c + k, h.m - 1);
      mu4[k] = mu[i];
      l4[k] = lraw[i];
    }
    lp += sac_head_block4<T>(h, r, mu4, l4, c);
  }
  return lp;
}
__device__ __forceinline__ void sac_head_logp(const HeadEpi& h, int r, float lp) {
  if (r < h.Bl) h.logp2[r] = lp;
  else h.logp[r - h.Bl] = lp;
}
template <typename T>
__device__ __forceinline__ void sac_head_row(const HeadEpi& h, int r, const float* mu, const float* lraw) {
  sac_head_logp(h, r, sac_head_blocks<T>(h, r, mu, lraw, 0, 1));
}

// TD3: rows r < Bl (target actor on s2): a' = clip(tanh z + clip(noise n, -c, c), -1, 1), n from
// S_SMOOTH; rows r >= Bl (online actor on s): a~ = tanh z (cached for the backward).  One Philox block
// c of row r: actions 4c .. 4c+3 (< m) from z4.
template <typename T>
__device__ __forceinline__ void td3_head_block4(const HeadEpi& h, int r, const float (&z4)[4], int c) {
  const uint64_t step = (uint64_t)*h.step_p;
  const bool trow = r < h.Bl;
  const int j = trow ? r : r - h.Bl;
  T* xa = static_cast<T*>(h.Xc) + (int64_t)(trow ? 2 * h.Bl + r : h.Bl + j) * h.ldx + h.o;
  float n4[4] = {0.f, 0.f, 0.f, 0.f};
  if (trow) normals4(h.seed, step, S_SMOOTH, (uint64_t)(h.row0 + r), c, h.m - 4 * c > 2 ? 2 : 1, n4);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = 4 * c + k;
    if (i >= h.m) break;
    if (trow) {
      const float xi = fminf(fmaxf(h.noise * n4[k], -h.clipc), h.clipc);
      xa[i] = from_f<T>(fminf(fmaxf(tanhf(z4[k]) + xi, -1.f), 1.f));
    } else {
      const float a = tanhf(z4[k]);
      xa[i] = from_f<T>(a);
      h.a[(int64_t)i * h.Bl + j] = a;
    }
  }
}
template <typename T>
__device__ __forceinline__ void td3_head_blocks(const HeadEpi& h, int r, const float* z, int b0, int bstep) {
  for (int c = b0; 4 * c < h.m; c += bstep) {
    float z4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) z4[k] = z[min(4 * c + k, h.m - 1)];
    td3_head_block4<T>(h, r, z4, c);
  }
}
template <typename T>
__device__ __forceinline__ void td3_head_row(const HeadEpi& h, int r, const float* z) {
  td3_head_blocks<T>(h, r, z, 0, 1);
}

}  // namespace spz
