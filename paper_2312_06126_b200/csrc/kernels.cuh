// kernels.cuh -- the non-GEMM kernels of one update step.
//
// Each kernel cites the step it implements.  All reductions are fixed-order
// (warp shuffles in a fixed tree, per-block partials summed in block order), so
// an update is bit-reproducible run to run on a given device count (reading #16).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "heads.cuh"

namespace spz {


// ------------------------------------------------------------------ a1 + a2: index + gather
// Block = 32 rows.  Records are read with 128-bit loads into shared memory; the operands leave with
// 128-bit stores, each row's written columns rounded up to whole 32-byte sectors.  Writes (local row j,
// global row row0 + j):
//   Xa[j] = s2, Xa[Bl + j] = s                           (actor input, [s2; s])
//   Xc[j] = [s | a], Xc[Bl + j] = [s | 0], Xc[2Bl + j] = [s2 | 0]  (critic inputs; the action columns of
//                                                         the last two are written by the actor heads)
//   r[j], d[j]
// Columns past the rounded-up width are padding: zeroed once at allocation and never written.
constexpr int GATHER_ROWS = 32;

template <typename T>
__device__ __forceinline__ uint4 pack_chunk(const float* src, int c0, int n) {
  // 16 bytes of the operand: elements c0 .. c0 + 16/sizeof(T) - 1 of a row, zero past n
  constexpr int EPC = 16 / sizeof(T);
  float v[EPC];
#pragma unroll
  for (int i = 0; i < EPC; ++i) v[i] = c0 + i < n ? src[c0 + i] : 0.f;
  uint4 u;
  if constexpr (std::is_same<T, float>::value) {
    u.x = __float_as_uint(v[0]);
    u.y = __float_as_uint(v[1]);
    u.z = __float_as_uint(v[2]);
    u.w = __float_as_uint(v[3]);
  } else {
    u.x = pack_bf16x2(v[0], v[1]);
    u.y = pack_bf16x2(v[2], v[3]);
    u.z = pack_bf16x2(v[4], v[5]);
    u.w = pack_bf16x2(v[6], v[7]);
  }
  return u;
}

__device__ __forceinline__ uint32_t smem_u32_(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// 16-byte asynchronous global -> shared copy (LDGSTS, L1 bypass) and its group fences
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32_(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Grid-stride over groups of GATHER_ROWS rows with NBUF shared-memory record buffers: the Philox indices and the
// asynchronous record copies of the next group are issued before the current group is packed and stored, so
// the random-row round trip to HBM overlaps the operand stores (large batches: several groups per block).
template <typename T>
__global__ void __launch_bounds__(256) gather_kernel(const float* __restrict__ rec, int R, int o, int m,
                                                     const int64_t* __restrict__ fill_p, uint64_t seed,
                                                     const int64_t* __restrict__ step_p, int64_t row0, int Bl,
                                                     T* __restrict__ Xa, int lda, T* __restrict__ Xc, int ldc,
                                                     float* __restrict__ r, float* __restrict__ d,
                                                     int32_t* __restrict__ idx_out, uint32_t* __restrict__ tags,
                                                     int nbuf) {
  pdl_wait();
  pdl_launch();
  extern __shared__ float4 sm4[];
  __shared__ int64_t sidx[2][GATHER_ROWS];
  const int64_t fill = *fill_p;
  const uint64_t step = (uint64_t)*step_p;
  const int R4 = R >> 2;
  const int ngroups = (Bl + GATHER_ROWS - 1) / GATHER_ROWS;
  // indices of group gi into sidx[b], then its records into buffer b (one commit group)
  auto issue = [&](int gi, int b) {
    const int j0 = gi * GATHER_ROWS;
    const int nr = min(GATHER_ROWS, Bl - j0);
    if (threadIdx.x < nr) {
      const int64_t i = sample_index(seed, step, (uint64_t)(row0 + j0 + threadIdx.x), (uint64_t)fill);
      sidx[b][threadIdx.x] = i;
      if (idx_out) idx_out[j0 + threadIdx.x] = (int32_t)i;
      if (tags) atomicOr(&tags[i >> 5], 1u << (i & 31));  // transmission-loss tags (spz_replay_track)
    }
    __syncthreads();
    float4* buf = sm4 + (size_t)b * GATHER_ROWS * R4;
    for (int e = threadIdx.x; e < nr * R4; e += blockDim.x) {
      const int rr = e / R4, q = e - rr * R4;
      cp_async16(buf + e, reinterpret_cast<const float4*>(rec + sidx[b][rr] * R) + q);
    }
    cp_async_commit();
  };
  // 16-byte chunks per operand row, rounded up to whole 32-byte sectors (and capped by the row pitch)
  constexpr int EPC = 16 / sizeof(T), EPS = 32 / sizeof(T);
  const int s2c = o + m + 2;
  const int ca = min((o + EPS - 1) / EPS * EPS, lda) / EPC;          // s / s2 columns (actor, critic [s|0])
  const int cb = min((o + m + EPS - 1) / EPS * EPS, ldc) / EPC;      // [s | a]
  const int cs = min((o + EPS - 1) / EPS * EPS, ldc) / EPC;
  const int J = 2 * ca + cb + 2 * cs;                                 // chunks per row
  // operand of chunk k of a row: 0 Xa s2-row j, 1 Xa s-row Bl + j, 2 Xc [s | a] row j, 3 Xc [s | (a~)] row Bl + j,
  // 4 Xc [s2 | (a')] row 2 Bl + j -- destination base / pitch / row offset, 16-byte unit, source column, width
  struct Chunk {
    T* base;
    int64_t rowoff;
    int ld, kk, src0, n;
  };
  auto chunk_of = [&](int k) {
    int op, kk;
    if (k < 2 * ca) {
      op = k >= ca;
      kk = k - op * ca;
    } else if ((k -= 2 * ca) < cb) {
      op = 2;
      kk = k;
    } else {
      k -= cb;
      op = k >= cs ? 4 : 3;
      kk = k - (op - 3) * cs;
    }
    Chunk c;
    c.base = op < 2 ? Xa : Xc;
    c.ld = op < 2 ? lda : ldc;
    c.rowoff = (op == 1 || op == 3) ? (int64_t)Bl : op == 4 ? 2 * (int64_t)Bl : 0;
    c.kk = kk;
    c.src0 = (op == 0 || op == 4) ? s2c : 0;
    c.n = op == 2 ? o + m : o;
    return c;
  };
  const bool fixed_chunk = J <= (int)blockDim.x;
  const int rows_per_pass = fixed_chunk ? (int)blockDim.x / J : 0, t_row = fixed_chunk ? (int)threadIdx.x / J : 0;
  const Chunk tc = chunk_of(fixed_chunk ? (int)threadIdx.x % J : 0);
  T* const t_base = tc.base;
  const int64_t t_rowoff = tc.rowoff;
  const int t_ld = tc.ld, t_kk = tc.kk, t_src0 = tc.src0, t_n = tc.n;
  int it = 0;
  if ((int)blockIdx.x < ngroups) issue(blockIdx.x, 0);
  for (int gi = blockIdx.x; gi < ngroups; gi += gridDim.x, ++it) {
    const int b = nbuf > 1 ? (it & 1) : 0;
    const int gn = gi + (int)gridDim.x;
    if (nbuf > 1 && gn < ngroups) {
      issue(gn, b ^ 1);   // the next group's copies in flight while this one is stored
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int j0 = gi * GATHER_ROWS;
    const int nr = min(GATHER_ROWS, Bl - j0);
    const float* sm = reinterpret_cast<const float*>(sm4 + (size_t)b * GATHER_ROWS * R4);
    if (fixed_chunk) {
      // J <= blockDim.x: thread t keeps chunk t % J for rows t / J, t / J + rows_per_pass, ... -- its operand,
      // destination and source columns are loop invariants (no per-item division or operand selection)
      if (t_row < rows_per_pass)
        for (int rr = t_row; rr < nr; rr += rows_per_pass)
          *(reinterpret_cast<uint4*>(t_base + (t_rowoff + j0 + rr) * t_ld) + t_kk) =
              pack_chunk<T>(sm + rr * R + t_src0, t_kk * EPC, t_n);
    } else {
      for (int e = threadIdx.x; e < nr * J; e += blockDim.x) {
        const int rr = e / J;
        const Chunk c = chunk_of(e - rr * J);
        *(reinterpret_cast<uint4*>(c.base + (c.rowoff + j0 + rr) * c.ld) + c.kk) =
            pack_chunk<T>(sm + rr * R + c.src0, c.kk * EPC, c.n);
      }
    }
    if (threadIdx.x < nr) {
      r[j0 + threadIdx.x] = sm[threadIdx.x * R + o + m];
      d[j0 + threadIdx.x] = sm[threadIdx.x * R + o + m + 1];
    }
    __syncthreads();  // buffer b (and sidx[b]) free for the group after next
    if (nbuf == 1 && gn < ngroups) issue(gn, 0);
  }
}

// ------------------------------------------------------------------ a3: SAC actor head (forward)
// Row r < Bl is the s2-row j = r (noise eps' from S_EPS2) and produces a', log pi';
// row r >= Bl is the s-row j = r - Bl (eps from S_EPS) and produces a~, log pi~ plus
// the per-element cache the head backward needs.  [mu | l] = H[r, 0:2m];
// lc = clamp(l, lo, hi); sigma = exp(lc); u = mu + sigma eps; a = tanh u;
// log pi = sum_i [-eps^2/2 - lc - ln(2 pi)/2 - 2 (ln 2 - u - softplus(-2u))].
struct HeadCache {
  float *u, *a, *eps, *sig, *l;  // [m x Bl] each (action-major: a warp's rows store contiguously), s-rows only
};

template <typename T>
__global__ void sac_head_fwd_kernel(const float* __restrict__ H, int ldh, HeadEpi h, int M) {
  pdl_wait();
  pdl_launch();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  float mu[32], l[32];
  for (int i = 0; i < h.m; ++i) {
    mu[i] = H[(int64_t)r * ldh + i];
    l[i] = H[(int64_t)r * ldh + h.m + i];
  }
  sac_head_row<T>(h, r, mu, l);
}

// ------------------------------------------------------------------ a3: TD3 actor heads (forward)
// Rows r < Bl: target actor on s2, a' = clip(tanh(z) + clip(noise * n, -c, c), -1, 1) with n from
// S_SMOOTH (written into Xc[2Bl + r]); rows Bl <= r < M: online actor on s, a~ = tanh(z)
// (written into Xc[r], cached for the backward).  P:576, reading #18.
template <typename T>
__global__ void td3_head_fwd_kernel(const float* __restrict__ H, int ldh, HeadEpi h, int M) {
  pdl_wait();
  pdl_launch();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  float z[32];
  for (int i = 0; i < h.m; ++i) z[i] = H[(int64_t)r * ldh + i];
  td3_head_row<T>(h, r, z);
}

// TD3 actor head backward: dZ_out = g_a (1 - a~^2) with g_a the Q1 input gradient's action columns.
template <typename T>
__global__ void td3_head_bwd_kernel(const float* __restrict__ dX1, int ldx, int o, int m, int Bl,
                                    const float* __restrict__ a_cache, T* __restrict__ dH, int ldh) {
  pdl_wait();
  pdl_launch();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)Bl * m) return;
  const int64_t j = e / m;
  const int i = (int)(e - j * m);
  const float a = a_cache[(int64_t)i * Bl + j];  // head cache: action-major [m x Bl]
  dH[j * ldh + i] = from_f<T>(dX1[j * ldx + o + i] * (1.f - a * a));
}

// ------------------------------------------------------------------ a4/a5: critic head (N = 1) row dot
// q[r] = sum_n A[r, n] w[n] + b, one warp per row, fixed shuffle tree.
struct RowdotGroup {
  const void* A;
  const float* w;
  const float* b;
  float* q;
};
struct RowdotArgs {
  int M, h, ld;
  RowdotGroup g[4];
};

template <typename T>
__global__ void __launch_bounds__(256) rowdot_kernel(const __grid_constant__ RowdotArgs a) {
  pdl_wait();
  pdl_launch();
  const RowdotGroup& g = a.g[blockIdx.y];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= a.M) return;
  const T* row = static_cast<const T*>(g.A) + (int64_t)warp * a.ld;
  float s = 0.f;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    // h % 8 == 0: each lane takes 8 adjacent columns per pass (16-byte loads)
    for (int n = lane * 8; n < a.h; n += 256) {
      const uint4 u = *reinterpret_cast<const uint4*>(row + n);
      const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(x[i]);
        s = fmaf(f.x, g.w[n + 2 * i], s);
        s = fmaf(f.y, g.w[n + 2 * i + 1], s);
      }
    }
  } else {
    for (int n = lane; n < a.h; n += 32) s = fmaf(to_f(row[n]), g.w[n], s);
  }
  s = warp_sum(s);
  if (lane == 0) g.q[warp] = s + g.b[0];
}

// ------------------------------------------------------------------ block reduction of NSTAT doubles
template <int NT>
__device__ __forceinline__ void block_stats(double (&v)[NSTAT], double* __restrict__ out) {
  __shared__ double red[NT / 32][NSTAT];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NSTAT; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NSTAT; ++i) red[w][i] = v[i];
  __syncthreads();
  if (threadIdx.x < NSTAT) {
    double s = 0.0;
    for (int k = 0; k < NT / 32; ++k) s += red[k][threadIdx.x];
    out[blockIdx.x * NSTAT + threadIdx.x] = s;
  }
}

// ------------------------------------------------------------------ a4 + a5 + a6 head: Bellman target, losses, critic head backward
// Block = LOSS_ROWS rows j of [0, Bl).  Per row:
//   y = r + gamma (1-d) (min(q'1, q'2) - alpha log pi');     (TD3: no entropy term)
//   loss rows:  g_qi[j] = 2 (q_i(s,a) - y) / B
//   actor rows: g_qi[Bl + j] = -w_i / B, (w1, w2) = (1,0) | (0,1) | (1/2,1/2) on a tie
//               (TD3: Q1 only, g = -1/B, and only on delayed steps)
// then the critic head backward for those rows: dZ_L[r, n] = g_q[r] w_out[n] 1[A_L[r, n] > 0].
// Loss statistics: per-block partials; the last block to finish sums them in block order into
// `totals` (this rank's loss totals; all-reduced across a row-sharded group).
constexpr int LOSS_NT = 256, LOSS_WARPS = LOSS_NT / 32;
constexpr int LOSS_MIN_ROWS = LOSS_WARPS;  // rows per block at RPW = 1 (sizes the statistics partials)

struct LossArgs {
  const float *qt1, *qt2, *q1, *q2, *logp2, *logp, *r, *d, *log_alpha;
  const int64_t* step_p;
  float *gq1, *gq2, *y;
  __nv_bfloat16* gq16[2];  // optional: bf16 copies of the loss-row g_q (pitch 8, column 0) -- the A operand
                           // of the critic-head weight / bias gradients on the tensor cores
  double* partials;
  double* totals;
  int64_t* ctr_snap;  // the step's counters (step, t_c, t_a, t_al) as read before the optimizer advances them
  float* la_snap;     // the step's log alpha (statistics), likewise
  float* bc_snap;     // Adam bias corrections 1 - beta^t of the three optimizers: [bc1 x 3 | bc2 x 3]
  float beta1, beta2;
  unsigned* ticket;
  const void* A[2];          // last hidden activations (mask source when mask[] is null)
  const uint32_t* mask[2];   // packed ReLU masks of the last hidden layer (tcgen05 path)
  const float* w[2];
  void* dZ[2];
  float gamma, invB;
  int Bl, td3, delay, loss_rows, actor_rows, h, ld, mask_ld;
  int q2_no_actor;        // TD3: Q2 has no actor rows (its dZ_L there is never read)
  int defer_totals;       // 1: no grid-wide reduction here -- the optimizer sums the block partials itself (off the
                          //    critical path, before its dependency wait); block 0 writes the optimizer snapshot;
  unsigned* bad2;         //    a block with a non-finite partial ORs 1 into bad2[step & 1] (block 0 clears the
                          //    other word for the next step), so the optimizer's blocks decide without the totals
  int diag;               // diagnostics only (SPZ_DIAG_LOSS_CUT; results are wrong): 1 skip the grid-wide statistics
                          // reduction, 2 no work at all
  // SAC v1 (reading #24): qt1 = qt2 = V'(s2) and the bootstrap drops the entropy term; the actor rows
  // also give the value target y_V = min(q1~, q2~) - alpha log pi~, g_V = 2 (V(s) - y_V) / B
  int v1;
  const float* vo;        // V(s) of the s rows (qp partials, stride vps)
  float* gv;              // g_V [Bl]
  __nv_bfloat16* gv16;    // optional bf16 copy (pitch 8), like gq16
  int64_t vps;
  int qp;                 // q partials per row (fused row dot over qp 256-column tiles), summed in tile order
  int64_t qps_tg, qps_on;  // partial strides of the target / online q buffers
};

__device__ __forceinline__ float ld_q(const float* __restrict__ q, int64_t j, int qp, int64_t ps) {
  // qp <= 4 (h <= 1024): predicated loads, so every row scalar's loads can issue back to back
  float s = __ldg(q + j), t[3];
#pragma unroll
  for (int p = 1; p < 4; ++p) t[p - 1] = p < qp ? __ldg(q + p * ps + j) : 0.f;
#pragma unroll
  for (int p = 1; p < 4; ++p)
    if (p < qp) s += t[p - 1];
  return s;
}

// Loss totals from the per-block statistics partials, in a fixed order: thread t sums blocks t, t + NT, ...; then
// each warp's shuffle tree; then the warps in order.  Called by the loss kernel's last block, or by every block of
// the optimizer (deferred totals) -- the same NT gives bit-identical totals.  Thread i < NSTAT writes total i to
// out[i] (out may be shared or global); red: [NT / 32][NSTAT] shared scratch.
template <int NT>
__device__ __forceinline__ void stat_totals(const double* __restrict__ partials, unsigned nblocks, double (*red)[NSTAT],
                                            double* out) {
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  double t[NSTAT] = {0, 0, 0, 0, 0, 0};
  for (unsigned b = threadIdx.x; b < nblocks; b += NT)
#pragma unroll
    for (int i = 0; i < NSTAT; ++i) t[i] += __ldcg(partials + b * NSTAT + i);
#pragma unroll
  for (int i = 0; i < NSTAT; ++i) t[i] = warp_sum(t[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NSTAT; ++i) red[wi][i] = t[i];
  __syncthreads();
  if (threadIdx.x < NSTAT) {
    double u = 0.0;
    for (int k = 0; k < NT / 32; ++k) u += red[k][threadIdx.x];
    out[threadIdx.x] = u;
  }
}

// Block = LOSS_ROWS rows, warp w owns rows w, w + 8, ... (LOSS_RPW of them).  Every lane loads the
// row scalars (broadcast) and computes g_q itself; with DZ (h <= 256: one 8-column chunk per lane) it
// then writes its chunk of dZ_L, otherwise critic_dz_kernel does that afterwards.  All of a warp's
// loads are issued before any of its arithmetic.  Lane 0 accumulates the statistics of the warp's
// rows in row order; the block partial sums the warps in order.
template <typename T, bool DZ, int LOSS_RPW, bool Q1 = DZ>
__global__ void __launch_bounds__(LOSS_NT) critic_loss_kernel(const __grid_constant__ LossArgs a) {
  constexpr int LOSS_ROWS = LOSS_WARPS * LOSS_RPW;
  pdl_wait();
  pdl_launch();
  if (a.diag) {  // diagnostics: block 0 writes the optimizer snapshot (finite totals, counters, bias corrections)
    if (blockIdx.x == 0) {
      if (threadIdx.x < NSTAT) a.totals[threadIdx.x] = 0.0;
      if (threadIdx.x < 4) a.ctr_snap[threadIdx.x] = a.step_p[threadIdx.x];
      if (threadIdx.x == 4) *a.la_snap = *a.log_alpha;
      if (threadIdx.x >= 8 && threadIdx.x < 14) {
        const int k = threadIdx.x - 8, o = k % 3;
        const double beta = k < 3 ? (double)a.beta1 : (double)a.beta2;
        a.bc_snap[k] = (float)(-expm1((double)(a.step_p[1 + o] + 1) * log1p(beta - 1.0)));
      }
    }
    if (a.diag == 2) return;
  }
  __shared__ double red[LOSS_NT / 32][NSTAT];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const bool lr = a.loss_rows, ar = a.actor_rows;
  const float alpha = a.td3 ? 0.f : expf(*a.log_alpha);
  const bool td3_on = a.td3 && ((*a.step_p + 1) % a.delay) == 0;
  double v[NSTAT] = {0, 0, 0, 0, 0, 0};
  // a grid of a few blocks per SM walks the row blocks (few grid-wide ticket atomics: one same-address
  // atomic per block serialises in L2, ~20 ns each at thousands of blocks); each warp's statistics
  // accumulate in row-block order, the block partials are summed in block order -- deterministic
  for (int jb = blockIdx.x; jb * LOSS_ROWS < a.Bl; jb += gridDim.x) {
  const int j0 = jb * LOSS_ROWS;
  // q partials per row: Q1 (always with DZ, which runs only at h <= 256, one lane per 8 columns) -- the row dot is
  // one tile; a compile-time 1 drops the predicated partial loads and their 64-bit address arithmetic
  const int qp = Q1 ? 1 : a.qp;
  // ---- loads, all issued before any use: row scalars of the warp's rows (row index clamped, so
  //      every address is valid; rows past Bl are discarded below)
  float qt1[LOSS_RPW], qt2[LOSS_RPW], q1[LOSS_RPW], q2[LOSS_RPW], lp2[LOSS_RPW], rw[LOSS_RPW], dn[LOSS_RPW];
  float a1[LOSS_RPW], a2[LOSS_RPW], lp[LOSS_RPW], vo[LOSS_RPW];
  const bool notemp = a.td3 || a.v1;  // no entropy term in the bootstrap (TD3; v1 bootstraps V')
#pragma unroll
  for (int i = 0; i < LOSS_RPW; ++i) {
    const int j = min(j0 + wi + 8 * i, a.Bl - 1);
    qt1[i] = ld_q(a.qt1, j, qp, a.qps_tg);
    qt2[i] = ld_q(a.qt2, j, qp, a.qps_tg);
    q1[i] = ld_q(a.q1, j, qp, a.qps_on);
    q2[i] = ld_q(a.q2, j, qp, a.qps_on);
    rw[i] = __ldg(a.r + j);
    dn[i] = __ldg(a.d + j);
    lp2[i] = notemp ? 0.f : __ldg(a.logp2 + j);
    a1[i] = ld_q(a.q1, a.Bl + j, qp, a.qps_on);
    a2[i] = ld_q(a.q2, a.Bl + j, qp, a.qps_on);
    lp[i] = a.td3 ? 0.f : __ldg(a.logp + j);
    vo[i] = a.v1 ? ld_q(a.vo, j, qp, a.vps) : 0.f;
  }
  // ---- DZ: mask bytes (bit k = column n0 + k) and head weights of this lane's chunk
  const int n0 = lane * 8;
  const bool has_chunk = DZ && n0 < a.h;
  const int nc = has_chunk ? n0 : 0;
  uint32_t mk[DZ ? LOSS_RPW : 1][2][2];
  float wv[2][8];
  if constexpr (DZ) {
    const bool bits = std::is_same<T, __nv_bfloat16>::value && a.mask[0] != nullptr;
#pragma unroll
    for (int i = 0; i < LOSS_RPW; ++i)
#pragma unroll
      for (int ci = 0; ci < 2; ++ci)
#pragma unroll
        for (int kind = 0; kind < 2; ++kind) {
          const int64_t row = (int64_t)(kind ? a.Bl : 0) + min(j0 + wi + 8 * i, a.Bl - 1);
          if (bits) {
            mk[i][ci][kind] = (__ldg(a.mask[ci] + row * a.mask_ld + nc / 32) >> (nc & 31)) & 0xFFu;
          } else {
            const T* A = static_cast<const T*>(a.A[ci]) + row * a.ld + nc;
            uint32_t mb = 0u;
#pragma unroll
            for (int k = 0; k < 8; ++k) mb |= (to_f(__ldg(A + k)) > 0.f ? 1u : 0u) << k;
            mk[i][ci][kind] = mb;
          }
        }
#pragma unroll
    for (int ci = 0; ci < 2; ++ci) {
      const float4 w0 = __ldg(reinterpret_cast<const float4*>(a.w[ci] + nc));
      const float4 w1 = __ldg(reinterpret_cast<const float4*>(a.w[ci] + nc + 4));
      wv[ci][0] = w0.x, wv[ci][1] = w0.y, wv[ci][2] = w0.z, wv[ci][3] = w0.w;
      wv[ci][4] = w1.x, wv[ci][5] = w1.y, wv[ci][6] = w1.z, wv[ci][7] = w1.w;
    }
  }
  // ---- per row: g_q (every lane), statistics (lane 0), dZ_L chunk of this lane
#pragma unroll
  for (int i = 0; i < LOSS_RPW; ++i) {
    const int rr = wi + 8 * i, j = j0 + rr;
    if (j >= a.Bl) break;  // warp-uniform
    float g[2][2] = {{0.f, 0.f}, {0.f, 0.f}};  // [critic][loss | actor row]
    if (lr) {
      const float qmin = fminf(qt1[i], qt2[i]);
      const float boot = notemp ? qmin : qmin - alpha * lp2[i];
      const float y = rw[i] + a.gamma * (1.f - dn[i]) * boot;
      const float e1 = q1[i] - y, e2 = q2[i] - y;
      g[0][0] = 2.f * e1 * a.invB;
      g[1][0] = 2.f * e2 * a.invB;
      if (lane == 0) {
        a.y[j] = y;
        a.gq1[j] = g[0][0];
        a.gq2[j] = g[1][0];
        if (a.gq16[0]) {
          a.gq16[0][(int64_t)j * 8] = __float2bfloat16_rn(g[0][0]);
          a.gq16[1][(int64_t)j * 8] = __float2bfloat16_rn(g[1][0]);
        }
        v[0] += (double)e1 * e1 + (double)e2 * e2;
        v[1] += q1[i];
        v[2] += q2[i];
      }
    }
    if (ar) {
      if (!a.td3) {
        const float w1 = a1[i] < a2[i] ? 1.f : (a1[i] > a2[i] ? 0.f : 0.5f);
        g[0][1] = -w1 * a.invB;
        g[1][1] = -(1.f - w1) * a.invB;
      } else {
        g[0][1] = td3_on ? -a.invB : 0.f;
      }
      if (lane == 0) {
        a.gq1[a.Bl + j] = g[0][1];
        a.gq2[a.Bl + j] = g[1][1];
        if (!a.td3) {
          v[3] += (double)alpha * lp[i] - (double)fminf(a1[i], a2[i]);
          v[4] += lp[i];
          if (a.v1) {
            const float ev = vo[i] - (fminf(a1[i], a2[i]) - alpha * lp[i]);
            const float gv = 2.f * ev * a.invB;
            a.gv[j] = gv;
            if (a.gv16) a.gv16[(int64_t)j * 8] = __float2bfloat16_rn(gv);
            v[5] += (double)ev * ev;
          }
        } else {
          v[3] += td3_on ? -(double)a1[i] : 0.0;
        }
      }
    }
    if constexpr (DZ) {
      if (!has_chunk) continue;
#pragma unroll
      for (int ci = 0; ci < 2; ++ci)
#pragma unroll
        for (int kind = 0; kind < 2; ++kind) {
          if (kind == 0 ? !lr : !ar) continue;
          if (kind == 1 && ci == 1 && a.q2_no_actor) continue;
          const int64_t row = (int64_t)(kind ? a.Bl : 0) + j;
          const float gq = g[ci][kind];
          const uint32_t mb = mk[i][ci][kind];
          T* dZ = static_cast<T*>(a.dZ[ci]) + row * a.ld + n0;
          if constexpr (std::is_same<T, __nv_bfloat16>::value) {
            uint4 o;
            __nv_bfloat162* yv = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              yv[k] = __floats2bfloat162_rn((mb >> (2 * k)) & 1u ? gq * wv[ci][2 * k] : 0.f,
                                            (mb >> (2 * k + 1)) & 1u ? gq * wv[ci][2 * k + 1] : 0.f);
            *reinterpret_cast<uint4*>(dZ) = o;
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) dZ[k] = (mb >> k) & 1u ? gq * wv[ci][k] : 0.f;
          }
        }
    }
  }
  }  // row blocks
  // block partial of the statistics: warps in order
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NSTAT; ++k) red[wi][k] = v[k];
  __syncthreads();
  if (threadIdx.x < NSTAT) {
    double t = 0.0;
    for (int k = 0; k < LOSS_NT / 32; ++k) t += red[k][threadIdx.x];
    a.partials[blockIdx.x * NSTAT + threadIdx.x] = t;
    if (a.defer_totals && !isfinite(t)) atomicOr(a.bad2 + (*a.step_p & 1), 1u);
  }
  // the last block sums every block's partial (fixed order: strided per thread, then a fixed tree)
  __syncthreads();
  if (a.diag == 1) return;
  if (a.defer_totals) {
    // the optimizer reduces the partials (stat_totals, same order); the snapshot depends on no other block
    if (blockIdx.x == 0) {
      if (threadIdx.x == 15) a.bad2[(*a.step_p + 1) & 1] = 0u;
      if (threadIdx.x < 4) a.ctr_snap[threadIdx.x] = a.step_p[threadIdx.x];
      if (threadIdx.x == 4) *a.la_snap = *a.log_alpha;
      if (threadIdx.x >= 8 && threadIdx.x < 14) {
        const int k = threadIdx.x - 8, o = k % 3;
        const double beta = k < 3 ? (double)a.beta1 : (double)a.beta2;
        const double t = (double)(a.step_p[1 + o] + 1);
        a.bc_snap[k] = (float)(-expm1(t * log1p(beta - 1.0)));
      }
    }
    return;
  }
  if (threadIdx.x == 0) {
    // two-level ticket: same-address atomics serialise in L2, so the blocks count in groups of 32 on
    // separate counters (ticket[1 + group]) and only each group's last block counts on ticket[0]
    fence_acq_rel_gpu();
    const unsigned grp = blockIdx.x / 32u, ngrp = (gridDim.x + 31u) / 32u;
    const unsigned in_grp = min(32u, gridDim.x - grp * 32u);
    last = false;
    if (atomicAdd(a.ticket + 1 + grp, 1u) == in_grp - 1) {
      a.ticket[1 + grp] = 0u;  // ready for the next launch (nobody else touches it in this one)
      fence_acq_rel_gpu();
      last = atomicAdd(a.ticket, 1u) == ngrp - 1;
    }
  }
  __syncthreads();
  if (last) {
    fence_acq_rel_gpu();
    stat_totals<LOSS_NT>(a.partials, gridDim.x, red, a.totals);
    if (threadIdx.x == 0) *a.ticket = 0u;
    if (threadIdx.x < 4) a.ctr_snap[threadIdx.x] = a.step_p[threadIdx.x];
    if (threadIdx.x == 4) *a.la_snap = *a.log_alpha;
    if (threadIdx.x >= 8 && threadIdx.x < 14) {
      // 1 - beta^t = -expm1(t log1p(beta - 1)) without cancellation, t = the optimizer's next step
      const int k = threadIdx.x - 8, o = k % 3;
      const double beta = k < 3 ? (double)a.beta1 : (double)a.beta2;
      const double t = (double)(a.step_p[1 + o] + 1);
      a.bc_snap[k] = (float)(-expm1(t * log1p(beta - 1.0)));
    }
  }
}

// ------------------------------------------------------------------ a6 head backward for wide layers (h > 256)
// dZ_L[r, n] = g_q[r] w_out[n] 1[z_L[r, n] > 0] over rows [r0, r0 + rows) of both critics; one thread per
// (row, 8-column chunk): every load (g_q, mask byte, head weights) is independent and issued up front,
// then one 16-byte store per critic.  Runs after critic_loss_kernel (which wrote g_q).
struct DzArgs {
  const float* gq[2];
  const uint32_t* mask[2];  // packed ReLU masks (tcgen05 path), or null: sign of A
  const void* A[2];
  const float* w[2];
  void* dZ[2];
  int64_t r0, rows;
  int64_t q2_end;  // critic 1 (Q2) rows end here (TD3: the loss rows only)
  int hv, ld, mask_ld;
};

template <typename T>
__global__ void __launch_bounds__(256) critic_dz_kernel(const __grid_constant__ DzArgs a) {
  pdl_wait();
  pdl_launch();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.rows * a.hv) return;
  const int64_t row = a.r0 + t / a.hv;
  const int n = (int)(t % a.hv) * 8;
  float g[2], wk[2][8];
  uint32_t mb[2];
#pragma unroll
  for (int ci = 0; ci < 2; ++ci) {
    g[ci] = __ldg(a.gq[ci] + row);
    const float4 w0 = __ldg(reinterpret_cast<const float4*>(a.w[ci] + n));
    const float4 w1 = __ldg(reinterpret_cast<const float4*>(a.w[ci] + n + 4));
    wk[ci][0] = w0.x, wk[ci][1] = w0.y, wk[ci][2] = w0.z, wk[ci][3] = w0.w;
    wk[ci][4] = w1.x, wk[ci][5] = w1.y, wk[ci][6] = w1.z, wk[ci][7] = w1.w;
    if (a.mask[ci]) {
      mb[ci] = (__ldg(a.mask[ci] + row * a.mask_ld + n / 32) >> (n & 31)) & 0xFFu;
    } else {
      const T* A = static_cast<const T*>(a.A[ci]) + row * a.ld + n;
      uint32_t m = 0u;
#pragma unroll
      for (int k = 0; k < 8; ++k) m |= (to_f(A[k]) > 0.f ? 1u : 0u) << k;
      mb[ci] = m;
    }
  }
#pragma unroll
  for (int ci = 0; ci < 2; ++ci) {
    if (ci == 1 && row >= a.q2_end) continue;
    T* dZ = static_cast<T*>(a.dZ[ci]) + row * a.ld + n;
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
      uint4 o;
      __nv_bfloat162* yv = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        yv[k] = __floats2bfloat162_rn((mb[ci] >> (2 * k)) & 1u ? g[ci] * wk[ci][2 * k] : 0.f,
                                      (mb[ci] >> (2 * k + 1)) & 1u ? g[ci] * wk[ci][2 * k + 1] : 0.f);
      *reinterpret_cast<uint4*>(dZ) = o;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) dZ[k] = (mb[ci] >> k) & 1u ? g[ci] * wk[ci][k] : 0.f;
    }
  }
}

// ------------------------------------------------------------------ a7: SAC actor head backward (eq. H)
// g_a = dL/da~ = sum over critics of the input-gradient action columns; g_lp = alpha / B.
// g_u = g_a (1 - a^2) + 2 a g_lp;  g_mu = g_u;  g_l = (g_u sigma eps - g_lp) 1[lo <= l <= hi].
template <typename T>
__global__ void sac_head_bwd_kernel(const float* __restrict__ dX1, const float* __restrict__ dX2, int ldx, int o, int m,
                                    int Bl, HeadCache cache, const float* __restrict__ log_alpha, float invB, float lo,
                                    float hi, T* __restrict__ dH, int ldh) {
  pdl_wait();
  pdl_launch();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)Bl * m) return;
  const int64_t j = e / m;
  const int i = (int)(e - j * m);
  const float g_lp = expf(*log_alpha) * invB;
  const float ga = dX1[j * ldx + o + i] + dX2[j * ldx + o + i];
  const int64_t ci = (int64_t)i * Bl + j;  // head cache: action-major [m x Bl]
  const float a = cache.a[ci];
  const float gu = ga * (1.f - a * a) + 2.f * a * g_lp;
  const float l = cache.l[ci];
  const float gl = (l >= lo && l <= hi) ? (gu * cache.sig[ci] * cache.eps[ci] - g_lp) : 0.f;
  dH[j * ldh + i] = from_f<T>(gu);
  dH[j * ldh + m + i] = from_f<T>(gl);
}

// ------------------------------------------------------------------ bias / head-weight gradients: column sums
// One launch covers several tensors (jobs).  Block (split s, job j) sums rows
// [s*rps, (s+1)*rps) of X (optionally weighted by w[r]) for every column and writes
// partial[s][n]; the fused Adam kernel adds the splits in a fixed order.  Threads own 8
// adjacent columns (one 16-byte load per row for bf16 rows) x 8 row lanes.
struct ColsumJob {
  const void* X;
  const float* w;
  float* out;
  int ld, N, M, f32;
};
constexpr int MAX_COLSUM_JOBS = 16;
struct ColsumArgs {
  int n_jobs, rps;
  ColsumJob j[MAX_COLSUM_JOBS];
};
constexpr int CS_VEC = 8, CS_TX = 32, CS_TY = 8;

template <typename T>
__device__ __forceinline__ void load8(const T* row, int n, int N, int ld_aligned, float (&v)[CS_VEC]) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (ld_aligned && n + CS_VEC <= N) {
      const uint4 u = *reinterpret_cast<const uint4*>(row + n);
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int i = 0; i < CS_VEC; ++i) v[i] = __bfloat162float(b[i]);
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < CS_VEC; ++i) v[i] = n + i < N ? to_f(row[n + i]) : 0.f;
}

template <typename T>
__global__ void __launch_bounds__(CS_TX* CS_TY) colsum_multi_kernel(const __grid_constant__ ColsumArgs a) {
  pdl_wait();
  pdl_launch();
  __shared__ float red[CS_TY][CS_TX * CS_VEC + 1];
  const ColsumJob& jb = a.j[blockIdx.y];
  const int s = blockIdx.x;
  const int r0 = s * a.rps, r1 = min(jb.M, r0 + a.rps);
  const int tx = threadIdx.x % CS_TX, ty = threadIdx.x / CS_TX;
  for (int c0 = 0; c0 < jb.N; c0 += CS_TX * CS_VEC) {
    const int n = c0 + tx * CS_VEC;
    float acc[CS_VEC] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (n < jb.N) {
#pragma unroll 4
      for (int r = r0 + ty; r < r1; r += CS_TY) {
        float v[CS_VEC];
        if (jb.f32) load8<float>(static_cast<const float*>(jb.X) + (int64_t)r * jb.ld, n, jb.N, 0, v);
        else load8<T>(static_cast<const T*>(jb.X) + (int64_t)r * jb.ld, n, jb.N, (jb.ld & 7) == 0, v);
        const float wr = jb.w ? jb.w[r] : 1.f;
#pragma unroll
        for (int i = 0; i < CS_VEC; ++i) acc[i] = fmaf(wr, v[i], acc[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < CS_VEC; ++i) red[ty][tx * CS_VEC + i] = acc[i];
    __syncthreads();
    for (int c = threadIdx.x; c < CS_TX * CS_VEC; c += blockDim.x) {
      if (c0 + c < jb.N) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < CS_TY; ++k) t += red[k][c];
        jb.out[(int64_t)s * jb.N + c0 + c] = t;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ a7 (alpha) + statistics
// Sums the per-block partials in block order; writes the step statistics, the
// log-alpha gradient g = -(mean log pi~ + H_bar) and the non-finite flag.
struct StatsOut {
  double step, critic_loss, actor_loss, alpha, alpha_loss, q1_mean, q2_mean, logp_mean, value_loss;
};

// ------------------------------------------------------------------ a9: fused multi-tensor Adam + Polyak
// Per element of every trained tensor:
// g = sum_s partial[s] (fixed order); Adam with the optimizer's own t; master,
// m, v updated; operand shadow (T, padded row stride) refreshed; if the tensor
// has a target: theta' = tau theta_new + (1 - tau) theta' (+ its shadow).
#ifndef SPZ_ADAM_EPT
#define SPZ_ADAM_EPT 2
#endif
#ifndef SPZ_ADAM_NT
#define SPZ_ADAM_NT 256
#endif
#ifndef SPZ_ADAM_CH4
#define SPZ_ADAM_CH4 8  // float4 split partials loaded per round (16: slower at TD3 / HUM, profiles/r02_adam_ab2.txt)
#endif
#ifndef SPZ_ADAM_MINB
#define SPZ_ADAM_MINB 4
#endif
constexpr int ADAM_NT = SPZ_ADAM_NT, ADAM_EPT = SPZ_ADAM_EPT, ADAM_SEG = ADAM_NT * ADAM_EPT;  // elements per block
static_assert(ADAM_NT == LOSS_NT, "deferred loss totals must sum in the loss kernel's order (stat_totals<NT>)");

struct AdamTensor {
  int64_t p_off;      // master offset of element 0
  int64_t numel;
  const float* partials;
  int32_t n_partials;
  int32_t opt;        // 0 critic, 1 actor, 2 alpha
  int32_t cols;       // > 0: weight matrix with shadow row stride ld
  int32_t ld;
  int64_t s_off;      // shadow offset (elements) of element 0, -1 if none
  int64_t t_off;      // target master offset, -1 if none
  int64_t ts_off;     // target shadow offset, -1 if none
  int64_t red_off;    // offset of this tensor in the contiguous (all-reduced) gradient buffer
  int64_t pstride;    // elements between split partials
  int32_t pld;        // partial row pitch: weight (r, c) at r * pld + c; bias i at i * pld
  int32_t pad_;
};

// Split-K partial sum of element i of tensor tn (fixed split order, left to right; 32-bit offsets).  The
// loads of up to 16 splits are all issued before the first add: one memory round trip per 16 splits.
__device__ __forceinline__ float partial_sum(const float* __restrict__ partials, int n_partials, int pstride, int pld,
                                             int cols, int i) {
  int idx;
  if (cols > 0) {
    const int row = i / cols;
    idx = row * pld + (i - row * cols);
  } else {
    idx = i * pld;
  }
  const float* src = partials + idx;
  constexpr int CH = 16;
  float g = 0.f;
  for (int s0 = 0; s0 < n_partials; s0 += CH) {
    float t[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) t[u] = s0 + u < n_partials ? __ldg(src + (s0 + u) * pstride) : 0.f;
#pragma unroll
    for (int u = 0; u < CH; ++u)
      if (s0 + u < n_partials) g += t[u];
  }
  return g;
}
// The same for 4 consecutive elements i..i+3 of one row, contiguous and 16-byte aligned in every partial.
template <int CH = SPZ_ADAM_CH4>
__device__ __forceinline__ float4 partial_sum4(const float* __restrict__ partials, int n_partials, int pstride, int pld,
                                               int cols, int i) {
  int idx;
  if (cols > 0) {
    const int row = i / cols;
    idx = row * pld + (i - row * cols);
  } else {
    idx = i * pld;
  }
  const float4* src = reinterpret_cast<const float4*>(partials + idx);
  const int ps4 = pstride >> 2;
  float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s0 = 0; s0 < n_partials; s0 += CH) {
    float4 t[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) t[u] = s0 + u < n_partials ? __ldg(src + (s0 + u) * ps4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < CH; ++u)
      if (s0 + u < n_partials) g.x += t[u].x, g.y += t[u].y, g.z += t[u].z, g.w += t[u].w;
  }
  return g;
}
__device__ __forceinline__ float partial_sum(const AdamTensor& tn, int64_t i) {
  return partial_sum(tn.partials, tn.n_partials, (int)tn.pstride, tn.pld, tn.cols, (int)i);
}

struct AdamSegment {
  AdamTensor t;       // the tensor (embedded: one dependent load per segment)
  int64_t start;      // element index within the tensor
  int32_t count;
  int32_t vec;        // 1: float4 layout (4 consecutive elements per thread, 16-byte loads and stores; the host
                      //    checked every alignment and that 4 consecutive elements share one row), 0: scalar
};
struct AdamHyper {
  float lr[3];
  float beta1, beta2, eps, tau;
  int td3, delay;
  // statistics + counter advance folded into this kernel
  double* totals;  // loss totals of the step (this rank's, or the group's after the allreduce)
  const float* log_alpha;  // as of the start of the step (loss-kernel snapshot)
  StatsOut* stats;
  double target_entropy, B;
  const int64_t* snap;  // counters of this step (written by the loss kernel); the kernel advances `counters`
  const float* bc;      // bias corrections of this step (loss-kernel snapshot): [bc1 x 3 | bc2 x 3]
  int alpha_auto, critic_on, actor_on;
  int diag_nowork;  // diagnostics only (SPZ_DIAG_ADAM_NOWORK): statistics and counters, no parameter update
  const double* stat_partials;  // deferred totals: the loss kernel's block partials (n_stat_blocks of them), summed by
  int n_stat_blocks;            // block 0 (publishes them to `totals`: statistics, diagnostics) and the log-alpha
  const unsigned* bad2;         // block; every other block decides from bad2[step & 1] (a partial was non-finite)
  int prewait;      // 1: the loss totals / counter snapshot are complete before this kernel's grid-dependency wait
                    //    (their writer is >= 2 kernels back behind wait-before-trigger kernels; set by the plan)
};

// 4 consecutive shadow elements (8-byte bf16 or 16-byte fp32 store; alignment checked by the host).
__device__ __forceinline__ void store4(__nv_bfloat16* d, float4 x) {
  *reinterpret_cast<uint2*>(d) = make_uint2(pack_bf16x2(x.x, x.y), pack_bf16x2(x.z, x.w));
}
__device__ __forceinline__ void store4(float* d, float4 x) { *reinterpret_cast<float4*>(d) = x; }

// One block per segment of ADAM_SEG elements (ADAM_EPT per thread, independent).  Every load of a
// thread is issued before the block barrier behind which thread 0 decides whether the step is
// applied (non-finite loss totals or an earlier halt); block 0 also publishes the statistics and
// advances the counters from the loss kernel's snapshot -- no block reads `counters` here, so no
// grid-wide handshake is needed.  (A non-finite gradient element sets the sticky flag 2: the step
// itself counts, every later step is skipped.)
// WIDE (small grids, at most two blocks per SM, e.g. WLK's 232): all <= 16 float4 split partials of a thread in one
// round (64 registers of loads; 2 blocks per SM) -- large grids keep 8 per round at 4 blocks per SM
template <typename T, bool WIDE>
__global__ void __launch_bounds__(ADAM_NT, WIDE ? 2 : SPZ_ADAM_MINB) adam_polyak_kernel(const AdamSegment* __restrict__ segs, AdamHyper hp,
                                                                 float* __restrict__ P, float* __restrict__ Mo,
                                                                 float* __restrict__ Vo, T* __restrict__ S,
                                                                 int64_t* __restrict__ counters,  // step, t_c, t_a, t_al
                                                                 int* __restrict__ flag) {
  // Prologue before the grid dependency wait (overlaps the weight-gradient kernel's tail): the segment
  // descriptor (host-written) and the optimizer state m, v, theta, theta' -- written only by the previous
  // step's Adam, which completed before any kernel of this step passed its own wait.
  __shared__ bool skip;
  const AdamSegment* sg = segs + blockIdx.x;
  const int opt = __ldg(&sg->t.opt);
  const int count = hp.diag_nowork ? 0 : __ldg(&sg->count);
  const int start = (int)__ldg(&sg->start);
  const int p_off = (int)__ldg(&sg->t.p_off);
  const int t_off = (int)__ldg(&sg->t.t_off);
  const float* partials = reinterpret_cast<const float*>(__ldg(reinterpret_cast<const unsigned long long*>(&sg->t.partials)));
  const int n_partials = __ldg(&sg->t.n_partials), pld = __ldg(&sg->t.pld), cols = __ldg(&sg->t.cols);
  const int pstride = (int)__ldg(&sg->t.pstride);
  const bool vec = __ldg(&sg->vec) != 0;
  float g[ADAM_EPT], m0[ADAM_EPT], v0[ADAM_EPT], p0[ADAM_EPT], tp0[ADAM_EPT];
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 g4 = z4, m4 = z4, v4 = z4, p4 = z4, tp4 = z4;
  const int k4 = 4 * threadIdx.x;  // vec: this thread's first element in the segment
  if (vec) {
    if (k4 < count) {
      const int pi = p_off + start + k4;
      m4 = *reinterpret_cast<const float4*>(Mo + pi);
      v4 = *reinterpret_cast<const float4*>(Vo + pi);
      p4 = *reinterpret_cast<const float4*>(P + pi);
      if (t_off >= 0) tp4 = *reinterpret_cast<const float4*>(P + t_off + start + k4);
    }
  } else {
#pragma unroll
    for (int u = 0; u < ADAM_EPT; ++u) {
      const int k = threadIdx.x + u * ADAM_NT;
      g[u] = m0[u] = v0[u] = p0[u] = tp0[u] = 0.f;
      if (k < count) {
        const int i = start + k, pi = p_off + i;
        m0[u] = Mo[pi];
        v0[u] = Vo[pi];
        p0[u] = P[pi];
        if (t_off >= 0) tp0[u] = P[t_off + i];
      }
    }
  }
  // Also before the wait: the loss totals, counter snapshot and bias corrections (written by the loss kernel,
  // three kernels back: complete once the weight-gradient kernel, this kernel's prerequisite, passed its own wait;
  // in a row-sharded group the non-PDL allreduce precedes this kernel, which then starts after it) and the skip
  // decision -- so after the wait only the split-K partials are loaded.
  __shared__ double stot[NSTAT];
  __shared__ double sred[ADAM_NT / 32][NSTAT];
  const double* tot = hp.n_stat_blocks > 0 ? stot : hp.totals;
  int64_t step = 0;
  float bc1 = 1.f, bc2 = 1.f;
  bool delayed = true;
  const bool need_totals = hp.n_stat_blocks > 0 && (blockIdx.x == 0 || opt == 2);
  auto decide = [&]() {
    if (need_totals) {
      stat_totals<ADAM_NT>(hp.stat_partials, (unsigned)hp.n_stat_blocks, sred, stot);
      __syncthreads();
      if (blockIdx.x == 0 && threadIdx.x < NSTAT) hp.totals[threadIdx.x] = stot[threadIdx.x];
    }
    step = __ldg(hp.snap);
    bc1 = __ldg(hp.bc + opt);
    bc2 = __ldg(hp.bc + 3 + opt);
    if (hp.td3) delayed = ((step + 1) % hp.delay) == 0;
    if (threadIdx.x == 0) {
      // the step's losses are finite iff their totals are (B > 0); TD3 has no log-prob total.  Deferred totals:
      // iff every block partial is (the loss kernel's flag word), except where this block summed them anyway
      const bool bad = hp.n_stat_blocks > 0 && !need_totals
                           ? __ldcg(hp.bad2 + (step & 1)) != 0u
                           : !isfinite(tot[0]) || !isfinite(tot[1]) || !isfinite(tot[2]) || !isfinite(tot[3]) ||
                                 (!hp.td3 && !isfinite(tot[4])) || !isfinite(tot[5]);
      const int f = *flag;
      if (bad && blockIdx.x == 0) atomicExch(flag, 1);
      skip = bad || f;  // halted: parameters stay at the state before the failing step
    }
    __syncthreads();
  };
  if (hp.prewait) decide();
  pdl_wait();
  pdl_launch();
  if (!hp.prewait) decide();
  // after the wait: this step's gradient partials
  if (vec) {
    if (k4 < count) g4 = partial_sum4<WIDE ? 16 : SPZ_ADAM_CH4>(partials, n_partials, pstride, pld, cols, start + k4);
  } else {
#pragma unroll
    for (int u = 0; u < ADAM_EPT; ++u) {
      const int k = threadIdx.x + u * ADAM_NT;
      if (k < count) {
        const int i = start + k;
        g[u] = opt == 2 ? (float)(-(tot[4] / hp.B + hp.target_entropy))  // log-alpha gradient
                        : partial_sum(partials, n_partials, pstride, pld, cols, i);
      }
    }
  }
  const bool active = !skip && !(hp.td3 && opt == 1 && !delayed);  // TD3 actor: delayed steps only
  if (active) {
    const float lr = hp.lr[opt];
    const int s_off = (int)__ldg(&sg->t.s_off), ts_off = (int)__ldg(&sg->t.ts_off), ld = __ldg(&sg->t.ld);
    const bool polyak = t_off >= 0 && (!hp.td3 || delayed);
    // one element: Adam (m, v, theta) and Polyak (theta'); false (nothing changes) on a non-finite gradient
    // bias corrections as per-block reciprocals and one approximate divide per element (each within 2 ulp of the
    // IEEE divisions; tests/parity.py's Adam identity allows 1e-5 of the step): WLK -1 us per update
    const float ib1 = 1.f / bc1, ib2 = 1.f / bc2;
    auto elem = [&](float ge, float me, float ve, float pe, float tpe, float& m, float& v, float& p, float& tp) {
      if (!isfinite(ge)) {
        atomicExch(flag, 2);
        m = me, v = ve, p = pe, tp = tpe;
        return false;
      }
      m = hp.beta1 * me + (1.f - hp.beta1) * ge;
      v = hp.beta2 * ve + (1.f - hp.beta2) * ge * ge;
      p = pe - __fdividef(lr * (m * ib1), sqrtf(v * ib2) + hp.eps);
      tp = hp.tau * p + (1.f - hp.tau) * tpe;
      return true;
    };
    if (vec) {
      if (k4 < count) {
        const int i = start + k4, pi = p_off + i;
        float4 m, v, p, tp;
        elem(g4.x, m4.x, v4.x, p4.x, tp4.x, m.x, v.x, p.x, tp.x);
        elem(g4.y, m4.y, v4.y, p4.y, tp4.y, m.y, v.y, p.y, tp.y);
        elem(g4.z, m4.z, v4.z, p4.z, tp4.z, m.z, v.z, p.z, tp.z);
        elem(g4.w, m4.w, v4.w, p4.w, tp4.w, m.w, v.w, p.w, tp.w);
        *reinterpret_cast<float4*>(Mo + pi) = m;
        *reinterpret_cast<float4*>(Vo + pi) = v;
        *reinterpret_cast<float4*>(P + pi) = p;
        int so = -1;
        if (cols > 0) {
          const int row = i / cols, col = i - row * cols;
          so = row * ld + col;
          store4(S + s_off + so, p);
        }
        if (polyak) {
          *reinterpret_cast<float4*>(P + t_off + i) = tp;
          if (so >= 0) store4(S + ts_off + so, tp);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < ADAM_EPT; ++u) {
        const int k = threadIdx.x + u * ADAM_NT;
        if (k >= count) continue;
        float m, v, p, tp;
        if (!elem(g[u], m0[u], v0[u], p0[u], tp0[u], m, v, p, tp)) continue;
        const int i = start + k, pi = p_off + i;
        Mo[pi] = m;
        Vo[pi] = v;
        P[pi] = p;
        int so = -1;
        if (cols > 0) {
          const int row = i / cols, col = i - row * cols;
          so = row * ld + col;
          S[s_off + so] = from_f<T>(p);
        }
        if (polyak) {
          P[t_off + i] = tp;
          if (so >= 0) S[ts_off + so] = from_f<T>(tp);
        }
      }
    }
  }
  // block 0: statistics (one field per thread) and the counter advance
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const double B = hp.B;
    const double la = (double)*hp.log_alpha;
    const double lpm = hp.td3 ? 0.0 : tot[4] / B;
    double* o = reinterpret_cast<double*>(hp.stats);
    switch (threadIdx.x) {
      case 0: o[0] = (double)(step + 1); break;
      case 1: o[1] = tot[0] / B; break;
      case 2: o[2] = tot[3] / B; break;
      case 3: o[3] = hp.td3 ? 0.0 : exp(la); break;
      case 4: o[4] = hp.td3 ? 0.0 : -la * (lpm + hp.target_entropy); break;
      case 5: o[5] = tot[1] / B; break;
      case 6: o[6] = tot[2] / B; break;
      case 7: o[7] = lpm; break;
      case 9: o[8] = tot[5] / B; break;  // SAC v1 value loss (the spare total is 0 otherwise)
      case 8:
        if (!skip) {
          counters[1] = hp.snap[1] + (hp.critic_on ? 1 : 0);
          counters[2] = hp.snap[2] + (hp.actor_on && delayed ? 1 : 0);
          counters[3] = hp.snap[3] + (hp.actor_on && hp.alpha_auto && !hp.td3 ? 1 : 0);
          counters[0] = step + 1;
        }
        break;
      default: break;
    }
  }
}
// Row-sharded learners: sum each tensor's split partials (fixed order) into the contiguous
// gradient buffer that is then all-reduced across the group.
__global__ void __launch_bounds__(ADAM_NT) reduce_partials_kernel(const AdamSegment* __restrict__ segs,
                                                                 float* __restrict__ Gred) {
  pdl_wait();
  pdl_launch();
  const AdamTensor tn = segs[blockIdx.x].t;
  for (int k = threadIdx.x; k < segs[blockIdx.x].count; k += blockDim.x) {
    const int64_t i = segs[blockIdx.x].start + k;
    Gred[tn.red_off + i] = partial_sum(tn, i);
  }
}

// Measurement: holds the stream until the host has queued a whole profiled step (the host-mapped word
// reaches `target`); gives up after ~5 s so a failed host never leaves the GPU spinning.
__global__ void gate_kernel(const volatile int* word, int target) {
  if (threadIdx.x != 0) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*word < target) {
    __nanosleep(2000);
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 5000000000ull) break;
  }
}

// Diagnostics: an empty kernel in the PDL chain (SPZ_DIAG_NOOP_OPS) to measure the cost of one
// kernel boundary inside the graph replay.
__global__ void noop_kernel(int) {
  pdl_wait();
  pdl_launch();
}

// ------------------------------------------------------------------ shadow refresh + init
struct ShadowEntry {
  int64_t p_off;  // master offset of W
  int32_t rows, cols, ld;
  int64_t s_off;
};

template <typename T>
__global__ void shadow_refresh_kernel(const ShadowEntry* __restrict__ ents, int n_ents, const float* __restrict__ P,
                                      T* __restrict__ S) {
  const ShadowEntry e = ents[blockIdx.y];
  const int64_t total = (int64_t)e.rows * e.ld;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = k / e.ld;
    const int col = (int)(k - row * e.ld);
    S[e.s_off + k] = from_f<T>(col < e.cols ? P[e.p_off + row * e.cols + col] : 0.f);
  }
}

// W, b ~ U(+-bound) with bound = 1/sqrt(fan_in), from Philox(init_seed, ctr = (e, net, 0, S_INIT)).
__global__ void init_uniform_kernel(float* __restrict__ P, int64_t off, int64_t n, float bound, uint64_t seed,
                                    uint32_t net, int64_t e0) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t e = (uint64_t)(e0 + k);
    const uint4 x = philox(make_uint4((uint32_t)e, (uint32_t)(e >> 32), net, S_INIT), (uint32_t)seed, (uint32_t)(seed >> 32));
    P[off + k] = (2.f * u01(x.x) - 1.f) * bound;
  }
}

}  // namespace spz
