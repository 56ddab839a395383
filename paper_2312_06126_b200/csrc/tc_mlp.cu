// tc_mlp.cu -- fused multi-layer MLP forward on the 5th-generation tensor cores (see tc_mlp.cuh).
//
// Warp roles (persistent CTA, one per SM):
//   warp 0      TMA producer: for every (unit, layer, k-block) one pipeline stage -- layer 0 loads the
//               input tile and the weight slab, deeper layers only the weight slab
//   warp 1      TMEM allocator + MMA issuer: A from the stage (layer 0) or from the hidden buffer H
//               (deeper layers), accumulator in TMEM buffer (unit & 1); one acc_full commit per layer
//   warps 2..  epilogue (4 x WPQ warps): TMEM lane quarter (warp % 4) x column slice; per hidden layer bias + ReLU ->
//               H (128B-swizzled K-major bf16, the next layer's A operand) + packed masks + row dot;
//               activations leave by TMA bulk stores from H; the actor head runs on the last MMA.
// Ordering: H is single-buffered.  The epilogue of (unit u, layer l) writes H only after the MMA of
// layer l (which read H) has completed (its acc_full), and after the TMA stores issued from H for
// layer l-1 have read it.  It writes H slab by slab (every warp its columns of each 64-column slab) and
// signals hs[slab] after each, so the MMA of layer l+1 starts on slab 0 while later slabs are still
// being written; the TMEM accumulator buffers alternate per layer so that MMA does not overwrite the
// accumulator being drained (acc_empty is signalled per layer).
#include "tc_mlp.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tc_common.cuh"

namespace spz {

namespace {

constexpr int MBM = 128, MBK = 64, MSTAGES = 4;
// Epilogue warps: WPQ per TMEM lane quarter (each owns H / WPQ columns of its 32 rows); 4 per quarter
// at h >= 128 (the per-layer epilogue is instruction-issue bound), 2 at h = 64 (a warp keeps whole
// 32-column mask words).
template <int H>
constexpr int mlp_wpq() { return H >= 128 ? 4 : 2; }
constexpr int mlp_threads(int wpq) { return 64 + 4 * wpq * 32; }
constexpr int MA_BYTES = MBM * MBK * 2;  // 16 KB input tile per k-block

struct MlpDev {
  int rows, row0;
  const float* bias[MLP_MAXL + 1];
  uint32_t* mask[MLP_MAXL];
  int store[MLP_MAXL];  // activations of hidden layer l stored (tact valid)
  const float* dot_w;
  const float* dot_b;
  float* dot_out;
};

// Diagnostics (spz_diag_tc_trace, modes >= 100): %globaltimer stamps per (CTA, unit, layer):
// 0 MMA starts the layer, 1 MMA issue done, 2 epilogue sees the accumulator, 3 epilogue done,
// 4 first weight slab of the layer present, 5 last weight slab present.
constexpr int MT_CTAS = 160, MT_UNITS = 4, MT_LAYERS = 3, MT_EV = 6;
__device__ unsigned long long g_mtrace[MT_CTAS * MT_UNITS * MT_LAYERS * MT_EV];
__device__ __forceinline__ void mtrace(int on, int ui, int l, int ev) {
  if (on && blockIdx.x < MT_CTAS && ui < MT_UNITS && l < MT_LAYERS) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_mtrace[((blockIdx.x * MT_UNITS + ui) * MT_LAYERS + l) * MT_EV + ev] = t;
  }
}

struct MlpParams {
  int n_pass, L, n_mma, k0, nh, head_n, head_epi, mask_ld, stages, trace;
  // super-unit schedule: group kind k covers super-units [su0[k], su0[k+1]); each runs passes
  // gpass[k][0..gn[k]) on row block (su - su0[k])
  int n_grp, total_su, any_loss;
  int su0[MLP_MAXN + 1];
  int gn[MLP_MAXN], gloss[MLP_MAXN], gpass[MLP_MAXN][4];
  HeadEpi head;
  MlpLoss loss;
  MlpDev d[MLP_MAXN];
  CUtensorMap tx[MLP_MAXN];
  CUtensorMap tw[MLP_MAXN][MLP_MAXL + 1];
  CUtensorMap tact[MLP_MAXN][MLP_MAXL];
  CUtensorMap tdz[2][2];  // dZ_L [critic][loss rows | actor rows]
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }


// relu(lo), relu(hi) -> packed bf16x2 (RNE) in one instruction
__device__ __forceinline__ uint32_t pack_relu_bf16(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// Hidden-layer epilogue of one warp: NB blocks of 32 accumulator columns of row r -> bias + ReLU ->
// bf16 into H (128B swizzle); MASK: packed ReLU-mask words (pre-activation > 0); DOT: row dot of the
// fp32 ReLU outputs with dot_s.
template <int NB, bool MASK, bool DOT>
__device__ __forceinline__ float hidden_epi(uint32_t trow, int c_lo, int r, uint8_t* Hs, const float* __restrict__ bias_s,
                                            const float* __restrict__ dot_s, uint32_t (&mw)[NB > 0 ? NB : 1]) {
  float dot = 0.f;
#pragma unroll
  for (int ib = 0; ib < NB; ++ib) {
    const int c = c_lo + ib * 2;  // first chunk of this 32-column block
    float v[2][16];
    tmem_ld32(trow + c * 16, v[0], v[1]);
    uint32_t word = 0u;
    uint32_t pk[16];
#pragma unroll
    for (int cc = 0; cc < 2; ++cc)
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const int bi = (ib * 2 + cc) * 16 + j;
        const float p0 = v[cc][j] + bias_s[bi], p1 = v[cc][j + 1] + bias_s[bi + 1];
        if constexpr (MASK) {
          word |= gt0_mask(p0) & (1u << (16 * cc + j));
          word |= gt0_mask(p1) & (1u << (16 * cc + j + 1));
        }
        if constexpr (DOT) {
          dot = fmaf(fmaxf(p0, 0.f), dot_s[bi], dot);
          dot = fmaf(fmaxf(p1, 0.f), dot_s[bi + 1], dot);
        }
        pk[cc * 8 + j / 2] = pack_relu_bf16(p0, p1);
      }
    if constexpr (MASK) mw[ib] = word;
    // 32 columns = four 16-byte units of row r in slab (c * 16) / 64 (128B swizzle)
    uint8_t* rowp = Hs + ((c * 16) / 64) * 16384 + r * 128;
    const int u0 = ((c * 16) % 64) / 8;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      *reinterpret_cast<uint4*>(rowp + (((u0 + k) ^ (r & 7)) << 4)) =
          make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
  }
  return dot;
}

// fixed-order sum of the WPQ per-warp partials of row r of a lane quarter
template <int WPQ>
__device__ __forceinline__ float quarter_sum(const float (*part)[MBM], int r) {
  if constexpr (WPQ == 4) return (part[0][r] + part[1][r]) + (part[2][r] + part[3][r]);
  else return part[0][r] + part[1][r];
}

// TMEM -> registers for one warp's CW columns (32 lanes x CW), issued without waiting: the caller's
// tmem_wait<CW>(r) ties the registers to the wait, so the next slab's load overlaps this slab's math
template <int CW>
__device__ __forceinline__ void tmem_issue(uint32_t taddr, uint32_t (&r)[CW]) {
  if constexpr (CW == 32) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
  }
}
template <int CW>
__device__ __forceinline__ void tmem_wait(uint32_t (&r)[CW]) {
  if constexpr (CW == 32) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
  } else {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
                 :
                 : "memory");
  }
}

// One warp's share of one 64-column slab of a hidden layer (tc_mlp_kernel), from its TMEM registers:
// CW columns of row r -> bias + ReLU -> bf16 into the slab of H; MASK: the CW mask bits (pre-activation
// > 0); DOT: row-dot partial with dot_s.  bias_s / dot_s hold this slab's CW entries of the warp.
template <int CW, bool MASK, bool DOT>
__device__ __forceinline__ uint32_t slab_math(const uint32_t (&v)[CW], int col0, int r, uint8_t* Hslab, const float* __restrict__ bias_s,
                                              const float* __restrict__ dot_s, float& dot) {
  static_assert(CW == 16 || CW == 32, "columns per warp and slab");
  uint32_t word = 0u, pk[CW / 2];
#pragma unroll
  for (int j = 0; j < CW; j += 2) {
    const float p0 = __uint_as_float(v[j]) + bias_s[j], p1 = __uint_as_float(v[j + 1]) + bias_s[j + 1];
    if constexpr (MASK) {
      word |= gt0_mask(p0) & (1u << j);
      word |= gt0_mask(p1) & (1u << (j + 1));
    }
    if constexpr (DOT) {
      dot = fmaf(fmaxf(p0, 0.f), dot_s[j], dot);
      dot = fmaf(fmaxf(p1, 0.f), dot_s[j + 1], dot);
    }
    pk[j / 2] = pack_relu_bf16(p0, p1);
  }
  uint8_t* rowp = Hslab + r * 128;
  const int u0 = (col0 % 64) / 8;
#pragma unroll
  for (int k = 0; k < CW / 8; ++k)
    *reinterpret_cast<uint4*>(rowp + (((u0 + k) ^ (r & 7)) << 4)) = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
  return word;
}

// A hidden layer's epilogue for one warp, slab by slab (every warp covers its CW = 64 / WPQ columns of
// every 64-column slab, so H fills slab by slab): the TMEM load of slab sl+1 is in flight while slab sl
// is processed; after each slab, hs[sl] is signalled (SIGNAL: the next layer's MMA reads H) and the
// warp's mask bits of the slab are stored.
template <int H, int WPQ, bool MASK, bool DOT>
__device__ __forceinline__ float hidden_epi_slabs(uint32_t trow, int hh, int r, uint8_t* Hs, const float* __restrict__ bias_s,
                                                  const float* __restrict__ dot_s, bool signal, uint64_t* hs, int lane,
                                                  uint32_t* mask_row) {
  constexpr int CW = 64 / WPQ, S = H / 64;
  float dot = 0.f;
  uint32_t cur[CW], nxt[CW];
  tmem_issue<CW>(trow + hh * CW, cur);
  tmem_wait<CW>(cur);
#pragma unroll
  for (int sl = 0; sl < S; ++sl) {
    const int col0 = sl * 64 + hh * CW;
    if (sl + 1 < S) tmem_issue<CW>(trow + col0 + 64, nxt);
    const uint32_t w = slab_math<CW, MASK, DOT>(cur, col0, r, Hs + sl * 16384, bias_s + sl * CW, dot_s + sl * CW, dot);
    if (signal) {
      fence_async_smem();  // this thread's H writes -> async proxy (the MMA)
      __syncwarp();
      if (lane == 0) mbar_arrive(&hs[sl]);
    }
    if constexpr (MASK) {
      if (mask_row) {
        if constexpr (CW == 32) mask_row[col0 / 32] = w;
        else reinterpret_cast<uint16_t*>(mask_row)[col0 / 16] = (uint16_t)w;
      }
    }
    if (sl + 1 < S) {
      tmem_wait<CW>(nxt);
#pragma unroll
      for (int k = 0; k < CW; ++k) cur[k] = nxt[k];
    }
  }
  return dot;
}

__device__ __forceinline__ int su_kind(const MlpParams& p, int su) {
  int k = 0;
  while (k + 1 < p.n_grp && su >= p.su0[k + 1]) ++k;
  return k;
}

// Fused critic loss of one super-unit (critic_loss_kernel's arithmetic): rows
// j = m0 + r of the block.  Loss rows: y = r + gamma (1-d)(min(q'1, q'2) - alpha log pi'), g_qi =
// 2 (q_i - y) / B; actor rows: g_qi = -w_i / B ((1,0) | (0,1) | (1/2,1/2) on a tie; TD3: q1 only,
// delayed steps).  Then dZ_L[ci] = g_qci w_ci 1[A_L > 0] (masks of this launch's online passes),
// written through H by TMA, and the block's statistics partial (fixed order).
template <int H, int WPQ>
__device__ __forceinline__ void loss_epilogue(const MlpParams& p, int kind, int su, int m0, int r, int hh, int e,
                                              int lane, uint8_t* Hs, float (*qv_s)[MBM], float* dot_s,
                                              double (*red_s)[NSTAT]) {
  constexpr int EW = 4 * WPQ, CPW = H / 16 / WPQ, NB = CPW / 2, SLICE = CPW * 16;
  const MlpLoss& a = p.loss;
  const int lk = p.gloss[kind];
  const int j = m0 + r;
  const bool valid = j < a.Bl;
  named_bar(1, EW * 32);  // every pass's q of this block is in qv_s
  double v[NSTAT] = {0, 0, 0, 0, 0, 0};
  float g[2] = {0.f, 0.f};
  if (valid) {
    if (lk == 1) {
      const float q1 = qv_s[0][r], q2 = qv_s[1][r], qt1 = qv_s[2][r], qt2 = qv_s[3][r];
      const float alpha = a.td3 ? 0.f : expf(*a.log_alpha);
      const float qmin = fminf(qt1, qt2);
      const float boot = a.td3 ? qmin : qmin - alpha * a.logp2[j];
      const float y = a.r[j] + a.gamma * (1.f - a.d[j]) * boot;
      const float e1 = q1 - y, e2 = q2 - y;
      g[0] = 2.f * e1 * a.invB;
      g[1] = 2.f * e2 * a.invB;
      if (hh == 0) {
        a.y[j] = y;
        a.gq1[j] = g[0];
        a.gq2[j] = g[1];
        if (a.gq16[0]) {
          a.gq16[0][(int64_t)j * 8] = __float2bfloat16_rn(g[0]);
          a.gq16[1][(int64_t)j * 8] = __float2bfloat16_rn(g[1]);
        }
        v[0] = (double)e1 * e1 + (double)e2 * e2;
        v[1] = q1;
        v[2] = q2;
      }
    } else {
      const float a1 = qv_s[0][r], a2 = qv_s[1][r];
      if (!a.td3) {
        const float alpha = expf(*a.log_alpha);
        const float w1 = a1 < a2 ? 1.f : (a1 > a2 ? 0.f : 0.5f);
        g[0] = -w1 * a.invB;
        g[1] = -(1.f - w1) * a.invB;
        if (hh == 0) {
          v[3] = (double)alpha * a.logp[j] - (double)fminf(a1, a2);
          v[4] = a.logp[j];
        }
      } else {
        const bool on = ((*a.step_p + 1) % a.delay) == 0;
        g[0] = on ? -a.invB : 0.f;
        if (hh == 0) v[3] = on ? -(double)a1 : 0.0;
      }
      if (hh == 0) {
        a.gq1[a.Bl + j] = g[0];
        a.gq2[a.Bl + j] = g[1];
      }
    }
  }
  const int c_lo = hh * CPW;
  for (int ci = 0; ci < 2; ++ci) {
    // this thread's mask words of row j (stored by this same thread in pass ci's last epilogue)
    uint32_t mw[NB > 0 ? NB : 1];
    const MlpDev& dd = p.d[p.gpass[kind][ci]];
#pragma unroll
    for (int i = 0; i < NB; ++i) mw[i] = valid ? dd.mask[p.L - 1][(int64_t)j * p.mask_ld + (c_lo * 16) / 32 + i] : 0u;
#pragma unroll
    for (int c = lane; c < SLICE; c += 32) dot_s[c] = a.w[ci][c_lo * 16 + c];
    if (e == 0 && lane == 0) bulk_wait_read0();  // H free of earlier TMA stores
    named_bar(1, EW * 32);
    const float gq = g[ci];
#pragma unroll
    for (int ib = 0; ib < NB; ++ib) {
      const int c = c_lo + ib * 2;
      uint32_t pk[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int n = 2 * k;
        const float z0 = (mw[ib] >> n) & 1u ? gq * dot_s[ib * 32 + n] : 0.f;
        const float z1 = (mw[ib] >> (n + 1)) & 1u ? gq * dot_s[ib * 32 + n + 1] : 0.f;
        pk[k] = pack_bf16(z0, z1);
      }
      uint8_t* rowp = Hs + ((c * 16) / 64) * 16384 + r * 128;
      const int u0 = ((c * 16) % 64) / 8;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        *reinterpret_cast<uint4*>(rowp + (((u0 + k) ^ (r & 7)) << 4)) =
            make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
    }
    fence_async_smem();
    named_bar(1, EW * 32);
    if (e == 0 && lane == 0) {
#pragma unroll
      for (int sl = 0; sl < H / 64; ++sl) tma_store_2d(&p.tdz[ci][lk - 1], Hs + sl * 16384, sl * 64, m0);
      bulk_commit();
    }
  }
  // statistics partial of this block: fixed shuffle tree per warp, warps in order
#pragma unroll
  for (int i = 0; i < NSTAT; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NSTAT; ++i) red_s[e][i] = v[i];
  named_bar(1, EW * 32);
  if (e == 0 && lane == 0)
    for (int i = 0; i < NSTAT; ++i) {
      double t = 0.0;
      for (int k = 0; k < EW; ++k) t += red_s[k][i];
      a.partials[(int64_t)su * NSTAT + i] = t;
    }
}

// After the last super-unit of every CTA: the last CTA to finish sums the statistics partials in
// block order into the step totals and snapshots the counters, log alpha and the Adam bias
// corrections for the optimizer (critic_loss_kernel's tail).
template <int EW>
__device__ __forceinline__ void loss_finish(const MlpParams& p, int e, int lane, double (*red_s)[NSTAT], bool& last) {
  const MlpLoss& a = p.loss;
  const int tid = e * 32 + lane;
  if (tid == 0) {
    fence_acq_rel_gpu();  // this thread wrote every partial of this CTA
    last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  }
  named_bar(1, EW * 32);
  if (!last) return;
  fence_acq_rel_gpu();
  double t[NSTAT] = {0, 0, 0, 0, 0, 0};
  for (int su = tid; su < p.total_su; su += EW * 32)
#pragma unroll
    for (int i = 0; i < NSTAT; ++i) t[i] += __ldcg(a.partials + (int64_t)su * NSTAT + i);
#pragma unroll
  for (int i = 0; i < NSTAT; ++i) t[i] = warp_sum(t[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NSTAT; ++i) red_s[e][i] = t[i];
  named_bar(1, EW * 32);
  if (tid < NSTAT) {
    double u = 0.0;
    for (int k = 0; k < EW; ++k) u += red_s[k][tid];
    a.totals[tid] = u;
  }
  if (tid == 0) *a.ticket = 0u;
  if (tid < 4) a.ctr_snap[tid] = a.step_p[tid];
  if (tid == 4) *a.la_snap = *a.log_alpha;
  if (tid >= 8 && tid < 14) {
    const int k = tid - 8, o = k % 3;
    const double beta = k < 3 ? (double)a.beta1 : (double)a.beta2;
    const double tt = (double)(a.step_p[1 + o] + 1);
    a.bc_snap[k] = (float)(-expm1(tt * log1p(beta - 1.0)));
  }
}

// H: hidden width of this instantiation; ACTOR: the last MMA layer is the actor head (else: critic,
// row-dot head fused into the last hidden layer's epilogue).
template <int H, bool ACTOR, int WPQ>
__global__ void __launch_bounds__(mlp_threads(WPQ), 1) tc_mlp_kernel(const __grid_constant__ MlpParams p) {
  constexpr int STAGE = H * MBK * 2;  // one weight slab (largest layer) per ring stage
  constexpr uint32_t BUF = H < 32 ? 32 : H;      // TMEM columns per accumulator buffer
  constexpr uint32_t TMEM_COLS = 2 * BUF <= 64 ? 64 : 2 * BUF <= 128 ? 128 : 2 * BUF <= 256 ? 256 : 512;
  constexpr int SLABS = H / 64;                  // 64-column slabs of H (16 KB each)
  constexpr int EW = 4 * WPQ;                    // epilogue warps
  constexpr int CPW = H / 16 / WPQ;              // 16-column chunks per epilogue warp
  constexpr int NB = CPW / 2;                    // 32-column blocks (= mask words) per warp
  constexpr int SLICE = CPW * 16;
  static_assert(H % 64 == 0 && H <= 256, "hidden width");
  __shared__ __align__(16) float bias_w[EW][SLICE > 64 ? SLICE : 64];  // (the actor head's nh <= 64 biases)
  __shared__ __align__(16) float dotw_w[EW][SLICE];
  __shared__ float dotpart[2][WPQ][MBM];
  __shared__ float qv_s[4][MBM];                    // critic groups: q of each pass, per row
  __shared__ double red_s[EW][NSTAT];      // statistics reduction
  __shared__ bool last_s;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NS = p.stages;
  uint8_t* Xs = smem + NS * STAGE;                  // layer-0 input tile: k0/64 x [128 rows x 128 B]
  uint8_t* Hs = Xs + (p.k0 / MBK) * MA_BYTES;       // hidden buffer: SLABS x [128 rows x 128 B]
  uint64_t* full = reinterpret_cast<uint64_t*>(Hs + SLABS * 16384);
  uint64_t* empty = full + MSTAGES;
  uint64_t* acc_full = empty + MSTAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* hs = acc_empty + 2;     // [4]: slab sl of H holds this layer's output (one arrival per epilogue warp)
  uint64_t* x_full = hs + 4;
  uint64_t* x_empty = x_full + 1;
  // actor: the head weights (<= 16 KB) are loaded into the input-tile region once layer 0 has consumed
  // it, early in the unit and outside the stage ring (whose slots free only as layer 1 completes)
  uint64_t* hw_full = x_empty + 1;
  uint64_t* hw_empty = hw_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hw_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TSU = p.total_su;
  const int L = p.L, NMMA = p.n_mma;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < p.n_pass; ++i) {
      tma_prefetch(&p.tx[i]);
      for (int l = 0; l < NMMA; ++l) tma_prefetch(&p.tw[i][l]);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], EW);
    }
    for (int sl = 0; sl < SLABS; ++sl) mbar_init(&hs[sl], EW);
    mbar_init(x_full, 1);
    mbar_init(x_empty, 1);
    mbar_init(hw_full, 1);
    mbar_init(hw_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Everything above overlapped the previous kernel (PDL).  The producer also issues the first ring
  // stages before its wait: they hold weight slabs only, written by the optimizer at least two
  // kernels back -- complete before the previous kernel passed its own wait, which precedes its
  // launch_dependents -- so they do not depend on the previous kernel.
  if (!(warp == 0 && lane == 0)) pdl_wait();
  pdl_launch();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: the input tile of each unit into Xs (freed by the MMA after
      //                  layer 0), every layer's weight slabs through the stage ring
      int pre = 0;  // ring stages issued before the PDL wait
      {
        bool stop = false;
        for (int su = blockIdx.x; su < TSU && !stop; su += gridDim.x) {
          const int k = su_kind(p, su);
          for (int j = 0; j < p.gn[k] && !stop; ++j) {
            const int g = p.gpass[k][j];
            for (int l = 0; l < NMMA && !stop; ++l) {
              if (ACTOR && l == L) continue;  // head weights go through the input-tile region
              const int nkb = l == 0 ? p.k0 / MBK : H / MBK;
              const int nrows = H;
              for (int kb = 0; kb < nkb; ++kb) {
                if (pre == NS) {
                  stop = true;
                  break;
                }
                mbar_expect_tx(&full[pre], (uint32_t)nrows * MBK * 2);
                tma_load_2d(smem + pre * STAGE, &p.tw[g][l], &full[pre], kb * MBK, 0);
                ++pre;
              }
            }
          }
        }
      }
      pdl_wait();
      int kg = 0, ui = 0;
      for (int su = blockIdx.x; su < TSU; su += gridDim.x) {
        const int k = su_kind(p, su);
        const int m0 = (su - p.su0[k]) * MBM;
        for (int j = 0; j < p.gn[k]; ++j, ++ui) {
          const int g = p.gpass[k][j];
          const int nx = p.k0 / MBK;
          for (int l = 0; l < NMMA; ++l) {
            if (l == 0) {
              // the region is free once the previous unit's head MMAs (actor) / layer 0 (critic) are done
              mbar_wait(ACTOR ? hw_empty : x_empty, ((uint32_t)ui & 1u) ^ 1u);
              mbar_expect_tx(x_full, (uint32_t)nx * MA_BYTES);
              for (int kb = 0; kb < nx; ++kb) tma_load_2d(Xs + kb * MA_BYTES, &p.tx[g], x_full, kb * MBK, m0);
            }
            if (ACTOR && l == L) {
              // head weights into the input-tile region as soon as layer 0 has consumed the input tile
              mbar_wait(x_empty, (uint32_t)ui & 1u);
              mbar_expect_tx(hw_full, (uint32_t)(H / MBK) * p.nh * 128);
              for (int kb = 0; kb < H / MBK; ++kb) tma_load_2d(Xs + kb * p.nh * 128, &p.tw[g][l], hw_full, kb * MBK, 0);
              continue;
            }
            const int nkb = l == 0 ? nx : H / MBK;
            const int nrows = H;
            for (int kb = 0; kb < nkb; ++kb, ++kg) {
              if (kg < pre) continue;  // issued before the PDL wait
              const int s = kg % NS;
              mbar_wait(&empty[s], ((uint32_t)(kg / NS) & 1u) ^ 1u);
              mbar_expect_tx(&full[s], (uint32_t)nrows * MBK * 2);
              tma_load_2d(smem + s * STAGE, &p.tw[g][l], &full[s], kb * MBK, 0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer.  Accumulator buffers alternate per layer (gl & 1), so layer l+1 can
      // run while the epilogue still drains layer l; its K-blocks wait for H slab by slab (hs[kb]).
      int kg = 0, ui = 0, hcnt = 0, gl = 0;
      uint32_t ause[2] = {0u, 0u};
      constexpr uint32_t IDESC_H = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(H >> 3) << 17) | ((uint32_t)(MBM >> 4) << 24);
      const uint32_t IDESC_HEAD = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.nh >> 3) << 17) | ((uint32_t)(MBM >> 4) << 24);
      const uint32_t sH = smem_u32(Hs), sX = smem_u32(Xs);
      for (int su = blockIdx.x; su < TSU; su += gridDim.x)
      for (int j = 0; j < p.gn[su_kind(p, su)]; ++j, ++ui) {
        for (int l = 0; l < NMMA; ++l, ++gl) {
          const int b = gl & 1;
          mbar_wait(&acc_empty[b], (ause[b] & 1u) ^ 1u);  // the epilogue drained this buffer's previous layer
          ++ause[b];
          tc_fence_after();
          const uint32_t acc = tmem + (uint32_t)b * BUF;
          mtrace(p.trace, ui, l, 0);
          const int nkb = l == 0 ? p.k0 / MBK : H / MBK;
          const uint32_t idesc = (ACTOR && l == L) ? IDESC_HEAD : IDESC_H;
          const uint32_t hph = (uint32_t)hcnt & 1u;  // phase of the H slabs of layer l-1
          if (l > 0) ++hcnt;
          if (l == 0) {
            mbar_wait(x_full, (uint32_t)ui & 1u);
            tc_fence_after();
          }
          if (ACTOR && l == L) {
            // head: B from the input-tile region (loaded there after layer 0), not from the ring
            mbar_wait(hw_full, (uint32_t)ui & 1u);
            tc_fence_after();
            mtrace(p.trace, ui, l, 4);
            mtrace(p.trace, ui, l, 5);
            for (int kb = 0; kb < nkb; ++kb) {
              mbar_wait(&hs[kb], hph);
              tc_fence_after();
              const uint32_t sB = sX + kb * p.nh * 128;
              const uint32_t aBase = sH + kb * 16384;
#pragma unroll
              for (int kk = 0; kk < MBK / 16; ++kk)
                umma_bf16(acc, desc_kmajor(aBase, kk), desc_kmajor(sB, kk), idesc, (kb | kk) != 0 ? 1u : 0u);
            }
            umma_commit(hw_empty);      // the region may take the next unit's input tile
            umma_commit(&acc_full[b]);  // head complete
            mtrace(p.trace, ui, l, 1);
            continue;
          }
          for (int kb = 0; kb < nkb; ++kb, ++kg) {
            const int s = kg % NS;
            mbar_wait(&full[s], (uint32_t)(kg / NS) & 1u);
            if (l > 0) mbar_wait(&hs[kb], hph);
            tc_fence_after();
            if (kb == 0) mtrace(p.trace, ui, l, 4);
            if (kb == nkb - 1) mtrace(p.trace, ui, l, 5);
            const uint32_t sB = smem_u32(smem + s * STAGE);
            const uint32_t aBase = l == 0 ? sX + kb * MA_BYTES : sH + kb * 16384;
#pragma unroll
            for (int kk = 0; kk < MBK / 16; ++kk)
              umma_bf16(acc, desc_kmajor(aBase, kk), desc_kmajor(sB, kk), idesc, (kb | kk) != 0 ? 1u : 0u);
            umma_commit(&empty[s]);
          }
          if (l == 0) umma_commit(x_empty);  // input tile consumed
          umma_commit(&acc_full[b]);  // layer l complete
          mtrace(p.trace, ui, l, 1);
        }
      }
    }
  } else {
    // ---------------- epilogue
    const int e = warp - 2;
    const int q = warp & 3;
    const int hh = e >> 2;
    const int c_lo = hh * CPW;      // first 16-column chunk of this warp
    const int r = q * 32 + lane;    // tile row of this thread
    float* bias_s = bias_w[e];
    float* dot_s = dotw_w[e];
    int ui = 0, dot_tiles = 0, gl = 0;
    uint32_t acnt[2] = {0u, 0u};    // acc_full commits consumed per buffer
    constexpr int CW = 64 / WPQ;    // columns of each 64-column slab owned by this warp
    for (int su = blockIdx.x; su < TSU; su += gridDim.x) {
    const int kind = su_kind(p, su);
    const int m0 = (su - p.su0[kind]) * MBM;
    const int m = m0 + r;
    for (int jp = 0; jp < p.gn[kind]; ++jp, ++ui) {
      const int g = p.gpass[kind][jp];
      const MlpDev& d = p.d[g];
      for (int l = 0; l < NMMA; ++l, ++gl) {
        const int b = gl & 1;  // accumulator buffers alternate per layer (the MMA issuer's order)
        const uint32_t trow = tmem + (uint32_t)b * BUF + ((uint32_t)(q * 32) << 16);
        const bool head = ACTOR && l == L;
        const bool last_hidden = !ACTOR && l == L - 1;
        const bool has_dot = last_hidden && d.dot_out != nullptr;
        // this warp's bias (and row-dot weight) entries of layer l, slab-major: entry sl * CW + c is
        // column sl * 64 + hh * CW + c; previous reads ordered by the __syncwarp that ends every layer
        if (!head) {
#pragma unroll
          for (int c = lane; c < SLICE; c += 32) {
            const int col = (c / CW) * 64 + hh * CW + c % CW;
            bias_s[c] = d.bias[l][col];
            dot_s[c] = has_dot ? d.dot_w[col] : 0.f;
          }
        } else if (lane < 16) {
          for (int c = lane; c < p.nh; c += 16) bias_s[c] = c < p.head_n ? d.bias[l][c] : 0.f;
        }
        __syncwarp();
        mbar_wait(&acc_full[b], acnt[b] & 1u);
        ++acnt[b];
        tc_fence_after();
        if (e == 0 && lane == 0) mtrace(p.trace, ui, l, 2);
        if (head) {
          // ---- actor head: the WPQ warps of a lane quarter take the row's Philox blocks of 4 actions
          //      in turn (warp hh: blocks hh, hh + WPQ, ...); SAC log pi = sum of the parts (fixed order)
          // per Philox block: the 4 mu (or z) and 4 log-sigma columns straight from TMEM into
          // registers (no per-row array, so nothing is indexed at run time)
          const int mh = p.head.m;
          const bool live = m < d.rows;
          const bool sac = p.head_epi == EPI_SAC_HEAD;
          float lp = 0.f;
          if (sac) {
            // SAC: work items = halves of Philox blocks (actions 2 it, 2 it + 1; one Box-Muller pair each),
            // taken in turn by the WPQ warps of the quarter (m = 6: 3 items instead of 2 blocks)
            for (int it = hh; 2 * it < mh; it += WPQ) {
              float v4[4], l4[4];
              tmem_ld1x4(trow + (uint32_t)(2 * it), v4);
              tmem_ld1x4(trow + (uint32_t)(mh + 2 * it), l4);
              float mu2[2], l2[2];
#pragma unroll
              for (int k = 0; k < 2; ++k) {
                const int i = min(2 * it + k, mh - 1);
                mu2[k] = v4[k] + bias_s[i];
                l2[k] = l4[k] + bias_s[mh + i];
              }
              if (!live) continue;
              lp += sac_head_half<__nv_bfloat16>(p.head, d.row0 + m, mu2, l2, it >> 1, it & 1);
            }
          } else {
            for (int c = hh; 4 * c < mh; c += WPQ) {
              float v4[4];
              tmem_ld1x4(trow + (uint32_t)(4 * c), v4);
#pragma unroll
              for (int k = 0; k < 4; ++k) v4[k] += bias_s[min(4 * c + k, mh - 1)];
              if (!live) continue;
              td3_head_block4<__nv_bfloat16>(p.head, d.row0 + m, v4, c);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[b]);  // head accumulator drained by this warp
          if (sac) {
            const int pb = dot_tiles & 1;
            dotpart[pb][hh][r] = lp;
            named_bar(2 + q, WPQ * 32);
            if (hh == 0 && live) sac_head_logp(p.head, d.row0 + m, quarter_sum<WPQ>(dotpart[pb], r));
            ++dot_tiles;
          }
          __syncwarp();
          if (e == 0 && lane == 0) mtrace(p.trace, ui, l, 3);
          continue;
        }
        // ---- hidden layer l: H must be free of the TMA stores issued from it for layer l-1
        if (e == 0 && lane == 0) bulk_wait_read0();
        named_bar(1, EW * 32);
        const bool want_mask = d.mask[l] != nullptr;
        const bool signal = l + 1 < NMMA;  // the next layer's MMA reads H slab by slab
        uint32_t* mrow = want_mask && m < d.rows ? d.mask[l] + (int64_t)m * p.mask_ld : nullptr;
        float dot;
        if (has_dot) {
          dot = want_mask ? hidden_epi_slabs<H, WPQ, true, true>(trow, hh, r, Hs, bias_s, dot_s, signal, hs, lane, mrow)
                          : hidden_epi_slabs<H, WPQ, false, true>(trow, hh, r, Hs, bias_s, dot_s, signal, hs, lane, mrow);
        } else {
          dot = want_mask ? hidden_epi_slabs<H, WPQ, true, false>(trow, hh, r, Hs, bias_s, dot_s, signal, hs, lane, mrow)
                          : hidden_epi_slabs<H, WPQ, false, false>(trow, hh, r, Hs, bias_s, dot_s, signal, hs, lane, mrow);
        }
        tc_fence_before();  // TMEM reads of this layer done: the buffer may take layer l+2
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[b]);
        if (d.store[l]) {
          // activations leave by TMA bulk stores from H once every warp has written its slabs
          if (!signal) fence_async_smem();
          named_bar(1, EW * 32);
          if (e == 0 && lane == 0) {
#pragma unroll
            for (int sl = 0; sl < SLABS; ++sl) tma_store_2d(&p.tact[g][l], Hs + sl * 16384, sl * 64, m0);
            bulk_commit();
          }
        }
        if (e == 0 && lane == 0) mtrace(p.trace, ui, l, 3);
        if (has_dot) {
          // the warps of this lane quarter combine their slices in a fixed order
          const int pb = dot_tiles & 1;
          dotpart[pb][hh][r] = dot;
          named_bar(2 + q, WPQ * 32);
          const float qv = quarter_sum<WPQ>(dotpart[pb], r) + d.dot_b[0];
          if (hh == 0 && m < d.rows) d.dot_out[m] = qv;
          if (hh == 0) qv_s[jp][r] = qv;
          ++dot_tiles;
        }
      }
      __syncwarp();
    }
    if constexpr (!ACTOR) {
      if (p.gloss[kind]) loss_epilogue<H, WPQ>(p, kind, su, m0, r, hh, e, lane, Hs, qv_s, dot_s, red_s);
    }
    }
    if constexpr (!ACTOR) {
      if (p.any_loss) loss_finish<EW>(p, e, lane, red_s, last_s);
    }
  }
  if (warp >= 2 && lane == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

int g_mtrace_mode = 0;
long g_mtrace_count = 0;

// ---------------------------------------------------------------------------------------------------
// Critic forward with two row blocks in flight per CTA ("pair" schedule).  The plain schedule above
// runs the layers of one block back to back, so the tensor pipe idles during every epilogue and
// the epilogue warps idle during every layer's MMAs (~7.5 us per block at WLK, ~2.6 blocks per
// CTA).  Here the blocks of a CTA are taken in pairs (A, B) and interleaved layer by layer --
//   MMA:      L0(A) L0(B) L1(A) L1(B) ...        epilogue: E0(A) E0(B) E1(A) E1(B) ...
// -- so E0(B) runs under L1(A), E1(A) under L1(B), and so on.  Each block of a pair owns a TMEM
// accumulator buffer and a hidden buffer H (two H buffers: 2 x 64 KB at h = 256, which leaves room
// for a 2-stage weight ring).  Critic passes only (no actor head, no fused loss groups).
template <int H, int WPQ>
__global__ void __launch_bounds__(mlp_threads(WPQ), 1) tc_mlp_pair_kernel(const __grid_constant__ MlpParams p) {
  constexpr int STAGE = H * MBK * 2;
  constexpr uint32_t BUF = H < 32 ? 32 : H;
  constexpr uint32_t TMEM_COLS = 2 * BUF <= 64 ? 64 : 2 * BUF <= 128 ? 128 : 2 * BUF <= 256 ? 256 : 512;
  constexpr int SLABS = H / 64;
  constexpr int EW = 4 * WPQ;
  constexpr int CPW = H / 16 / WPQ;
  constexpr int NB = CPW / 2;
  constexpr int SLICE = CPW * 16;
  constexpr int HBYTES = SLABS * 16384;
  constexpr uint32_t IDESC_H = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(H >> 3) << 17) | ((uint32_t)(MBM >> 4) << 24);
  __shared__ __align__(16) float bias_w[EW][SLICE];
  __shared__ __align__(16) float dotw_w[EW][SLICE];
  __shared__ float dotpart[2][WPQ][MBM];
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NS = p.stages;
  uint8_t* Xs = smem + NS * STAGE;
  uint8_t* Hs0 = Xs + (p.k0 / MBK) * MA_BYTES;  // H buffer of pair slot x: Hs0 + x * HBYTES
  uint64_t* full = reinterpret_cast<uint64_t*>(Hs0 + 2 * HBYTES);
  uint64_t* empty = full + MSTAGES;
  uint64_t* acc_full = empty + MSTAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint64_t* h_full = acc_empty + 2;      // [2]
  uint64_t* x_full = h_full + 2;
  uint64_t* x_empty = x_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_empty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TSU = p.total_su, L = p.L;
  const int U = TSU > (int)blockIdx.x ? (TSU - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;  // this CTA's blocks
  const int nx = p.k0 / MBK;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < p.n_pass; ++i) {
      tma_prefetch(&p.tx[i]);
      for (int l = 0; l < L; ++l) tma_prefetch(&p.tw[i][l]);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], EW);
      mbar_init(&h_full[b], 1);
    }
    mbar_init(x_full, 1);
    mbar_init(x_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch();

  // block i of this CTA: super-unit su = blockIdx.x + i * gridDim.x (every group has one pass)
  auto block_of = [&](int i, int& g, int& m0) {
    const int su = (int)blockIdx.x + i * (int)gridDim.x;
    const int k = su_kind(p, su);
    g = p.gpass[k][0];
    m0 = (su - p.su0[k]) * MBM;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer: per pair, layer by layer, block by block (the MMA's order)
      int kg = 0, xc = 0;
      for (int i0 = 0; i0 < U; i0 += 2) {
        const int nu = min(2, U - i0);
        for (int l = 0; l < L; ++l)
          for (int x = 0; x < nu; ++x) {
            int g, m0;
            block_of(i0 + x, g, m0);
            if (l == 0) {
              mbar_wait(x_empty, ((uint32_t)xc & 1u) ^ 1u);
              mbar_expect_tx(x_full, (uint32_t)nx * MA_BYTES);
              for (int kb = 0; kb < nx; ++kb) tma_load_2d(Xs + kb * MA_BYTES, &p.tx[g], x_full, kb * MBK, m0);
              ++xc;
            }
            const int nkb = l == 0 ? nx : H / MBK;
            for (int kb = 0; kb < nkb; ++kb, ++kg) {
              const int s = kg % NS;
              mbar_wait(&empty[s], ((uint32_t)(kg / NS) & 1u) ^ 1u);
              mbar_expect_tx(&full[s], (uint32_t)H * MBK * 2);
              tma_load_2d(smem + s * STAGE, &p.tw[g][l], &full[s], kb * MBK, 0);
            }
          }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      int kg = 0, xc = 0;
      int ae[2] = {0, 0}, hf[2] = {0, 0};  // acc_empty / h_full waits per buffer
      const uint32_t sX = smem_u32(Xs);
      for (int i0 = 0; i0 < U; i0 += 2) {
        const int nu = min(2, U - i0);
        for (int l = 0; l < L; ++l)
          for (int x = 0; x < nu; ++x) {
            const uint32_t acc = tmem + (uint32_t)x * BUF;
            const uint32_t sH = smem_u32(Hs0 + x * HBYTES);
            if (l == 0) {
              mbar_wait(&acc_empty[x], ((uint32_t)ae[x] & 1u) ^ 1u);  // the previous pair's block x drained
              ++ae[x];
              tc_fence_after();
              mbar_wait(x_full, (uint32_t)xc & 1u);
              ++xc;
              tc_fence_after();
            } else {
              mbar_wait(&h_full[x], (uint32_t)hf[x] & 1u);  // H_x holds layer l-1 of block x
              ++hf[x];
              tc_fence_after();
            }
            const int nkb = l == 0 ? nx : H / MBK;
            for (int kb = 0; kb < nkb; ++kb, ++kg) {
              const int s = kg % NS;
              mbar_wait(&full[s], (uint32_t)(kg / NS) & 1u);
              tc_fence_after();
              const uint32_t sB = smem_u32(smem + s * STAGE);
              const uint32_t aBase = l == 0 ? sX + kb * MA_BYTES : sH + kb * 16384;
#pragma unroll
              for (int kk = 0; kk < MBK / 16; ++kk)
                umma_bf16(acc, desc_kmajor(aBase, kk), desc_kmajor(sB, kk), IDESC_H, (kb | kk) != 0 ? 1u : 0u);
              umma_commit(&empty[s]);
            }
            if (l == 0) umma_commit(x_empty);
            umma_commit(&acc_full[x]);
          }
      }
    }
  } else {
    // ---------------- epilogue
    const int e = warp - 2, q = warp & 3, hh = e >> 2;
    const int c_lo = hh * CPW;
    const int r = q * 32 + lane;
    float* bias_s = bias_w[e];
    float* dot_s = dotw_w[e];
    int af[2] = {0, 0}, dot_tiles = 0;
    for (int i0 = 0; i0 < U; i0 += 2) {
      const int nu = min(2, U - i0);
      for (int l = 0; l < L; ++l)
        for (int x = 0; x < nu; ++x) {
          int g, m0;
          block_of(i0 + x, g, m0);
          const MlpDev& d = p.d[g];
          const int m = m0 + r;
          const bool last_hidden = l == L - 1;
          const bool has_dot = last_hidden && d.dot_out != nullptr;
          uint8_t* Hx = Hs0 + x * HBYTES;
          const uint32_t trow = tmem + (uint32_t)x * BUF + ((uint32_t)(q * 32) << 16);
#pragma unroll
          for (int c = lane; c < SLICE; c += 32) {
            bias_s[c] = d.bias[l][c_lo * 16 + c];
            dot_s[c] = has_dot ? d.dot_w[c_lo * 16 + c] : 0.f;
          }
          __syncwarp();
          mbar_wait(&acc_full[x], (uint32_t)af[x] & 1u);
          ++af[x];
          tc_fence_after();
          // H_x must be free of the TMA stores issued from it (conservatively: every store so far)
          if (e == 0 && lane == 0) bulk_wait_read0();
          named_bar(1, EW * 32);
          uint32_t mw[NB > 0 ? NB : 1];
          const bool want_mask = d.mask[l] != nullptr;
          float dot;
          if (has_dot) {
            dot = want_mask ? hidden_epi<NB, true, true>(trow, c_lo, r, Hx, bias_s, dot_s, mw)
                            : hidden_epi<NB, false, true>(trow, c_lo, r, Hx, bias_s, dot_s, mw);
          } else {
            dot = want_mask ? hidden_epi<NB, true, false>(trow, c_lo, r, Hx, bias_s, dot_s, mw)
                            : hidden_epi<NB, false, false>(trow, c_lo, r, Hx, bias_s, dot_s, mw);
          }
          tc_fence_before();
          fence_async_smem();
          named_bar(1, EW * 32);
          if (e == 0 && lane == 0) {
            if (l + 1 < L) mbar_arrive(&h_full[x]);
            if (d.store[l]) {
#pragma unroll
              for (int sl = 0; sl < SLABS; ++sl) tma_store_2d(&p.tact[g][l], Hx + sl * 16384, sl * 64, m0);
              bulk_commit();
            }
          }
          if (d.mask[l] != nullptr && m < d.rows) {
            uint32_t* dst = d.mask[l] + (int64_t)m * p.mask_ld + (c_lo * 16) / 32;
            if constexpr (NB == 4) {
              *reinterpret_cast<uint4*>(dst) = make_uint4(mw[0], mw[1 % NB], mw[2 % NB], mw[3 % NB]);
            } else if constexpr (NB == 2) {
              *reinterpret_cast<uint2*>(dst) = make_uint2(mw[0], mw[1 % NB]);
            } else {
#pragma unroll
              for (int i = 0; i < NB; ++i) dst[i] = mw[i];
            }
          }
          if (has_dot) {
            const int pb = dot_tiles & 1;
            dotpart[pb][hh][r] = dot;
            named_bar(2 + q, WPQ * 32);
            const float qv = quarter_sum<WPQ>(dotpart[pb], r) + d.dot_b[0];
            if (hh == 0 && m < d.rows) d.dot_out[m] = qv;
            ++dot_tiles;
          }
          if (last_hidden) {  // accumulator x drained for this block
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[x]);
          }
        }
    }
  }
  if (warp >= 2 && lane == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

template <int H, int WPQ>
cudaError_t launch_mlp_pair(MlpParams& p, cudaStream_t st) {
  constexpr int STAGE = H * MBK * 2;
  const int xbytes = (p.k0 / MBK) * MA_BYTES;
  const int fixed = 1024 + xbytes + 2 * (H / 64) * 16384 + 1024;
  constexpr int STATIC = 2 * 4 * H * 4 + 2 * WPQ * MBM * 4;  // bias / dot slices + dot partials
  const int ns = std::min(MSTAGES, (227 * 1024 - STATIC - 512 - fixed) / STAGE);
  if (ns < 2) return cudaErrorInvalidValue;
  auto kern = tc_mlp_pair_kernel<H, WPQ>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once(attr, kern, 227 * 1024 - STATIC - 512); e != cudaSuccess) return e;
  p.stages = ns;
  int grid = std::min(p.total_su, num_sms());
  if (grid == 0) return cudaSuccess;
  return launch_pdl(kern, dim3(grid), dim3(mlp_threads(WPQ)), (size_t)(ns * STAGE + fixed), st, p);
}

template <int H, bool ACTOR, int WPQ>
cudaError_t launch_mlp(MlpParams& p, cudaStream_t st) {
  constexpr int STAGE = H * MBK * 2;
  // dynamic: alignment slack + weight ring + input tile + H + barriers; static: bias / dot slices,
  // dot partials, q values, statistics (+ slack)
  constexpr int STATIC = 2 * 4 * WPQ * (H / WPQ > 64 ? H / WPQ : 64) * 4 + 2 * WPQ * MBM * 4 + 4 * MBM * 4 + 4 * WPQ * NSTAT * 8 + 1024;
  const int xbytes = (p.k0 / MBK) * MA_BYTES;
  const int fixed = 1024 + xbytes + (H / 64) * 16384 + 1024;
  const int ns = std::min(MSTAGES, (227 * 1024 - STATIC - fixed) / STAGE);
  if (ns < 2) return cudaErrorInvalidValue;
  constexpr int SMEM_ATTR = 227 * 1024 - STATIC;
  auto kern = tc_mlp_kernel<H, ACTOR, WPQ>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once(attr, kern, SMEM_ATTR); e != cudaSuccess) return e;
  p.stages = ns;
  p.trace = g_mtrace_mode == 1 || (g_mtrace_mode >= 2 && g_mtrace_count == g_mtrace_mode - 2);
  ++g_mtrace_count;
  int grid = std::min(p.total_su, num_sms());
  if (const char* cap = std::getenv("SPZ_DIAG_MLP_GRID")) grid = std::max(1, std::min(grid, std::atoi(cap)));  // diagnostics
  if (grid == 0) return cudaSuccess;
  return launch_pdl(kern, dim3(grid), dim3(mlp_threads(WPQ)), (size_t)(ns * STAGE + fixed), st, p);
}

// bf16 [rows x inner] map with a 64 x box_rows box, 128-byte swizzle (load or store)
bool map_rows(CUtensorMap* m, const void* ptr, int inner, int rows, int ld, int box_rows) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld % 8)) return false;
  return make_map(m, ptr, (uint64_t)inner, (uint64_t)rows, (uint64_t)ld, 64, (uint32_t)box_rows);
}

}  // namespace

cudaError_t mlp_trace(int on, unsigned long long* out, int n) {
  g_mtrace_mode = on;
  g_mtrace_count = 0;
  cudaError_t e = cudaSuccess;
  if (on) {
    static std::vector<unsigned long long> zeros(MT_CTAS * MT_UNITS * MT_LAYERS * MT_EV, 0ull);
    e = cudaMemcpyToSymbol(g_mtrace, zeros.data(), zeros.size() * sizeof(unsigned long long));
  }
  if (e != cudaSuccess || !out) return e;
  n = std::min(n, MT_CTAS * MT_UNITS * MT_LAYERS * MT_EV);
  return cudaMemcpyFromSymbol(out, g_mtrace, n * sizeof(unsigned long long));
}

bool tc_mlp_supported(const MlpArgs& a) {
  if (!get_encode()) return false;
  if (a.n_pass < 1 || a.n_pass > MLP_MAXN || a.L < 1 || a.L > MLP_MAXL) return false;
  if (a.h != 64 && a.h != 128 && a.h != 256) return false;
  if (a.k0 < 64 || a.k0 % 64 || a.k0 > 256) return false;
  if (a.head_n > 32 || (a.head_n == 0 && a.mask_ld * 32 < a.h)) return false;
  if (a.mask_ld % 4) return false;
  for (int i = 0; i < a.n_pass; ++i) {
    const MlpPass& s = a.p[i];
    if ((reinterpret_cast<uintptr_t>(s.X) & 15) || s.ldx % 8) return false;
    for (int l = 0; l <= a.L; ++l)
      if (l < a.L || a.head_n > 0)
        if ((reinterpret_cast<uintptr_t>(s.W[l]) & 15) || s.ldw[l] % 8) return false;
    for (int l = 0; l < a.L; ++l)
      if (s.mask[l] && (reinterpret_cast<uintptr_t>(s.mask[l]) & 15)) return false;
    if (a.head_n == 0 && !s.dot_out) return false;
  }
  if (a.n_group < 0 || a.n_group > MLP_MAXG) return false;
  for (int k = 0; k < a.n_group; ++k) {
    const MlpGroup& gr = a.grp[k];
    if (gr.n < 1 || gr.n > 4 || gr.rows < 0) return false;
    for (int jj = 0; jj < gr.n; ++jj)
      if (gr.pass[jj] < 0 || gr.pass[jj] >= a.n_pass || a.p[gr.pass[jj]].rows != gr.rows) return false;
    if (gr.loss) {
      if (a.head_n != 0 || gr.n != (gr.loss == 1 ? 4 : 2)) return false;
      for (int ci = 0; ci < 2; ++ci)
        if (!a.p[gr.pass[ci]].mask[a.L - 1] || (reinterpret_cast<uintptr_t>(a.loss.dZ[ci]) & 15)) return false;
    }
  }
  return true;
}

cudaError_t tc_mlp_fwd(const MlpArgs& a, cudaStream_t st) {
  MlpParams p;
  std::memset(&p, 0, sizeof(p));
  const bool actor = a.head_n > 0;
  p.n_pass = a.n_pass;
  p.L = a.L;
  p.n_mma = actor ? a.L + 1 : a.L;
  p.k0 = a.k0;
  p.head_n = a.head_n;
  p.nh = actor ? (a.head_n + 15) / 16 * 16 : 16;
  p.head_epi = a.head_epi;
  p.mask_ld = a.mask_ld;
  p.head = a.head;
  for (int i = 0; i < a.n_pass; ++i) {
    const MlpPass& s = a.p[i];
    MlpDev& d = p.d[i];
    d.rows = s.rows;
    d.row0 = s.row0;
    d.dot_w = s.dot_w;
    d.dot_b = s.dot_b;
    d.dot_out = s.dot_out;
    if (s.rows < 1) continue;
    if (!map_rows(&p.tx[i], s.X, a.k0, s.rows, s.ldx, MBM)) return cudaErrorInvalidValue;
    for (int l = 0; l < p.n_mma; ++l) {
      const int in = l == 0 ? a.k0 : a.h;
      const int out = (actor && l == a.L) ? a.head_n : a.h;
      const int box = (actor && l == a.L) ? p.nh : a.h;
      if (!map_rows(&p.tw[i][l], s.W[l], in, out, s.ldw[l], box)) return cudaErrorInvalidValue;
    }
    for (int l = 0; l <= a.L; ++l) d.bias[l] = s.bias[l];
    for (int l = 0; l < a.L; ++l) {
      d.mask[l] = s.mask[l];
      d.store[l] = s.act != nullptr && s.act[l] != nullptr;
      if (d.store[l] && !map_rows(&p.tact[i][l], s.act[l], a.h, s.rows, a.h, MBM)) return cudaErrorInvalidValue;
    }
  }
  // super-unit schedule
  int TSU = 0;
  if (a.n_group == 0) {
    p.n_grp = a.n_pass;
    for (int i = 0; i < a.n_pass; ++i) {
      p.su0[i] = TSU;
      p.gn[i] = 1;
      p.gpass[i][0] = i;
      TSU += (int)cdiv(a.p[i].rows, MBM);
    }
  } else {
    p.n_grp = a.n_group;
    for (int k = 0; k < a.n_group; ++k) {
      const MlpGroup& gr = a.grp[k];
      p.su0[k] = TSU;
      p.gn[k] = gr.n;
      p.gloss[k] = gr.loss;
      for (int jj = 0; jj < gr.n; ++jj) p.gpass[k][jj] = gr.pass[jj];
      TSU += (int)cdiv(gr.rows, MBM);
      if (gr.loss) {
        p.any_loss = 1;
        const int koff = gr.loss == 1 ? 0 : 1;
        for (int ci = 0; ci < 2; ++ci) {
          const void* base = static_cast<const __nv_bfloat16*>(a.loss.dZ[ci]) + (int64_t)koff * a.loss.Bl * a.h;
          if (!map_rows(&p.tdz[ci][koff], base, a.h, a.loss.Bl, a.h, MBM)) return cudaErrorInvalidValue;
        }
      }
    }
  }
  p.su0[p.n_grp] = TSU;
  p.total_su = TSU;
  p.loss = a.loss;
  if (TSU == 0) return cudaSuccess;
  // critic passes without loss groups and >= 2 row blocks per CTA: two blocks in flight per CTA (ANT:
  // critic forward 83.9 -> 76.1 us; WLK, ~2.6 blocks per CTA, since the 4-warps-per-quarter epilogue:
  // 103.0 -> 101.8 us per update -- with 2 epilogue warps per quarter the plain schedule had won there,
  // 29.7 vs 31.8 us, the pair schedule's 2-stage weight ring starving layer 1).  SPZ_MLP_PAIR=0 / 1 forces.
  const char* pe = std::getenv("SPZ_MLP_PAIR");  // read per launch (plans are built once)
  const int pair_env = pe ? (pe[0] == '1' ? 1 : 0) : -1;
  const bool pair = pair_env >= 0 ? pair_env == 1 : TSU >= 2 * num_sms();
  // SPZ_MLP_WPQ=2: two epilogue warps per lane quarter at every width (diagnostics; default mlp_wpq)
  const char* we = std::getenv("SPZ_MLP_WPQ");
  const bool w2 = we && we[0] == '2';
  if (!actor && a.n_group == 0 && pair) {
    switch (a.h) {
      case 64: return launch_mlp_pair<64, 2>(p, st);
      case 128: return w2 ? launch_mlp_pair<128, 2>(p, st) : launch_mlp_pair<128, mlp_wpq<128>()>(p, st);
      default: return w2 ? launch_mlp_pair<256, 2>(p, st) : launch_mlp_pair<256, mlp_wpq<256>()>(p, st);
    }
  }
  switch (a.h) {
    case 64: return actor ? launch_mlp<64, true, 2>(p, st) : launch_mlp<64, false, 2>(p, st);
    case 128:
      if (w2) return actor ? launch_mlp<128, true, 2>(p, st) : launch_mlp<128, false, 2>(p, st);
      return actor ? launch_mlp<128, true, mlp_wpq<128>()>(p, st) : launch_mlp<128, false, mlp_wpq<128>()>(p, st);
    default:
      if (w2) return actor ? launch_mlp<256, true, 2>(p, st) : launch_mlp<256, false, 2>(p, st);
      return actor ? launch_mlp<256, true, mlp_wpq<256>()>(p, st) : launch_mlp<256, false, mlp_wpq<256>()>(p, st);
  }
}

}  // namespace spz
