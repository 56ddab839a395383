// tc_gemm.cu -- bf16 GEMM on the 5th-generation tensor cores (sm_100a): TMA -> SMEM (128 B
// swizzle) -> tcgen05.mma (accumulator in TMEM) -> tcgen05.ld epilogue, with the shared
// GemmArgs epilogues (bias + ReLU, dgrad ReLU mask, fp32 head / split-K partial stores).
//
// One CTA computes a 128 x BN output tile (UMMA M = 128, N = BN, K = 16 per instruction)
// over a 64-deep K slab per pipeline stage:
//   warp 0      TMA producer (one elected lane), 4-stage mbarrier ring (full / empty)
//   warp 1      TMEM allocator + MMA issuer (one lane issues tcgen05.mma, commits to mbarriers)
//   warps 2..5  epilogue: TMEM lane quarter (warp % 4) -> 32 rows x BN fp32 columns
// Operands may be K-major (activations [rows x K], weights [out x in] in the forward) or
// MN-major (weights in dgrad; activations and dZ in wgrad, where the contraction runs over the
// batch) -- both are native UMMA smem-descriptor layouts, so no transposed copies exist.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <vector>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tc_gemm.cuh"

namespace spz {

namespace {

constexpr int BM = 128, BK = 64, STAGES = 4;
// producer warp, MMA warp, WPQ epilogue warps per TMEM lane quarter (each a slice of the columns)
#ifndef SPZ_TC_WPQ
#define SPZ_TC_WPQ 2
#endif
constexpr int WPQ = SPZ_TC_WPQ, NUM_EPI_WARPS = 4 * WPQ, NTHREADS = 64 + NUM_EPI_WARPS * 32;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB

struct TcParams {
  GemmArgs a;
  int stages;       // pipeline depth actually used (<= STAGES)
  int total_tiles;  // persistent schedule
  int tile0[MAX_GROUPS + 1];
  int mtiles[MAX_GROUPS], ntiles[MAX_GROUPS];
  int trace;      // diagnostics: record per-tile timestamps in this launch
  int tma_out;    // 1: outputs leave through TMA bulk tensor stores (tc[] valid), 0: direct stores
  int out_bytes;  // 2 (bf16) or 4 (fp32) output elements
  CUtensorMap ta[MAX_GROUPS];
  CUtensorMap tb[MAX_GROUPS];
  CUtensorMap tc[MAX_GROUPS];  // C as [splits][M][N]; box = 64 bytes x 32 rows, 64-byte swizzle
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Diagnostics: per-CTA, per-tile %globaltimer stamps (spz_diag_tc_trace).  Event e of the i-th tile of
// CTA c lands in g_trace[(c * TRACE_TILES + i) * 4 + e]: 0 producer starts the tile, 1 MMA issue done,
// 2 epilogue sees the accumulator, 3 epilogue done.
constexpr int TRACE_CTAS = 160, TRACE_TILES = 8;
__device__ unsigned long long g_trace[TRACE_CTAS * TRACE_TILES * 4];
#define trace(tile_i, ev) trace_(p.trace, tile_i, ev)
__device__ __forceinline__ void trace_(int on, int tile_i, int ev) {
  if (on && blockIdx.x < TRACE_CTAS && tile_i < TRACE_TILES) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[(blockIdx.x * TRACE_TILES + tile_i) * 4 + ev] = t;
  }
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// UMMA shared-memory descriptor (sm_100): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version 1 [46,48), base offset 0, layout SWIZZLE_128B (2) [61,64).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// K-major SW128 tile (rows x 64 bf16, 128 B rows): 8-row atoms 1024 B apart; K step of 16 = +32 B.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int kk) { return umma_desc(base + kk * 32, 16, 1024); }
// MN-major SW128 tile (64 K-rows x 64-element MN chunks, chunks 8 KB apart): 8-K-row groups
// 1024 B apart (SBO), MN chunks 8192 B apart (LBO); K step of 16 = +2048 B.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int kk) { return umma_desc(base + kk * 2048, 8192, 1024); }

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&p);
}

// Epilogue of 16 consecutive accumulator columns n..n+15 of row m (bias / dot vectors staged
// in shared memory for this column chunk).  Returns the chunk's contribution to the row dot.
__device__ __forceinline__ float epi16(const GemmArgs& a, const GemmGroup& g, int split, int m, int n, const float (&v)[16],
                                       const float* __restrict__ bias, const float* __restrict__ dotw, uint32_t& bits) {
  const bool full = n + 16 <= g.N;
  const int64_t off = (int64_t)m * g.ldc + n;
  float dot = 0.f;
  switch (a.epi) {
    case EPI_MASK_BITS: {
      // bits: this chunk's 16 ReLU-mask bits (prefetched by the caller)
      __nv_bfloat16* C = static_cast<__nv_bfloat16*>(g.C);
      if (full && (g.ldc & 7) == 0) {
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          pk[j] = pack_bf16((bits >> (2 * j)) & 1u ? v[2 * j] : 0.f, (bits >> (2 * j + 1)) & 1u ? v[2 * j + 1] : 0.f);
        uint4* dst = reinterpret_cast<uint4*>(C + off);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      } else {
        for (int j = 0; j < 16 && n + j < g.N; ++j) C[off + j] = __float2bfloat16_rn((bits >> j) & 1u ? v[j] : 0.f);
      }
      break;
    }
    case EPI_BIAS_RELU: {
      __nv_bfloat16* C = static_cast<__nv_bfloat16*>(g.C);
      float z[16];
      bits = 0u;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float pre = v[j] + bias[j];
        z[j] = fmaxf(pre, 0.f);
        bits |= (pre > 0.f && n + j < g.N ? 1u : 0u) << j;
      }
      if (dotw) {
#pragma unroll
        for (int j = 0; j < 16; ++j) dot = fmaf(z[j], dotw[j], dot);  // dotw is zero past g.N
      }
      if (full && (g.ldc & 7) == 0) {
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) pk[j] = pack_bf16(z[2 * j], z[2 * j + 1]);
        uint4* dst = reinterpret_cast<uint4*>(C + off);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      } else {
        for (int j = 0; j < 16 && n + j < g.N; ++j) C[off + j] = __float2bfloat16_rn(z[j]);
      }
      break;
    }
    case EPI_MASK: {
      __nv_bfloat16* C = static_cast<__nv_bfloat16*>(g.C);
      const __nv_bfloat16* X = static_cast<const __nv_bfloat16*>(g.aux) + (int64_t)m * g.ldaux + n;
      if (full && (g.ldc & 7) == 0 && (g.ldaux & 7) == 0) {
        const uint4 x0 = reinterpret_cast<const uint4*>(X)[0], x1 = reinterpret_cast<const uint4*>(X)[1];
        const __nv_bfloat162* xs0 = reinterpret_cast<const __nv_bfloat162*>(&x0);
        const __nv_bfloat162* xs1 = reinterpret_cast<const __nv_bfloat162*>(&x1);
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 f = __bfloat1622float2(j < 4 ? xs0[j] : xs1[j - 4]);
          pk[j] = pack_bf16(f.x > 0.f ? v[2 * j] : 0.f, f.y > 0.f ? v[2 * j + 1] : 0.f);
        }
        uint4* dst = reinterpret_cast<uint4*>(C + off);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      } else {
        for (int j = 0; j < 16 && n + j < g.N; ++j)
          C[off + j] = __float2bfloat16_rn(__bfloat162float(X[j]) > 0.f ? v[j] : 0.f);
      }
      break;
    }
    case EPI_BIAS_F32: {
      float* C = static_cast<float*>(g.C) + off;
      for (int j = 0; j < 16 && n + j < g.N; ++j) C[j] = v[j] + bias[j];
      break;
    }
    default: {
      float* C = static_cast<float*>(g.C) + off + (int64_t)split * g.split_stride;
      if (full && (g.ldc & 3) == 0 && ((reinterpret_cast<uintptr_t>(C) & 15) == 0)) {
        float4* d4 = reinterpret_cast<float4*>(C);
#pragma unroll
        for (int j = 0; j < 4; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      } else {
        for (int j = 0; j < 16 && n + j < g.N; ++j) C[j] = v[j];
      }
      break;
    }
  }
  return dot;
}

// Linear tile index -> (group, m0, n0, split).  Tiles of group g occupy [tile0[g], tile0[g+1]);
// within a group the M tile varies fastest, then the N tile, then the split.
struct TileInfo {
  int grp, m0, n0, split;
};
__device__ __forceinline__ TileInfo decode_tile(const TcParams& p, int t, int bn) {
  int g = 0;
  while (g + 1 < p.a.n_groups && t >= p.tile0[g + 1]) ++g;
  const int r = t - p.tile0[g];
  const int mt = r % p.mtiles[g];
  const int rest = r / p.mtiles[g];
  const int nt = rest % p.ntiles[g];
  return {g, mt * BM, nt * bn, rest / p.ntiles[g]};
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void epi_bar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(NUM_EPI_WARPS * 32) : "memory"); }

// Persistent, warp-specialized: each CTA walks tiles blockIdx.x, +gridDim.x, ...; the TMA producer
// and the MMA issuer run ahead into the next tile while the epilogue drains the previous one
// from the other TMEM accumulator buffer.
// Output values of 16 accumulator columns (TMA-store path): v is overwritten with what C receives.
__device__ __forceinline__ float epi16_vals(int epi, int n, int N, float (&v)[16], const float* __restrict__ bias,
                                            const float* __restrict__ dotw, uint32_t& bits) {
  float dot = 0.f;
  if (epi == EPI_BIAS_RELU) {
    uint32_t b = 0u;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float pre = v[j] + bias[j];
      v[j] = fmaxf(pre, 0.f);
      b |= (pre > 0.f && n + j < N ? 1u : 0u) << j;
    }
    if (dotw) {
#pragma unroll
      for (int j = 0; j < 16; ++j) dot = fmaf(v[j], dotw[j], dot);  // dotw is zero past N
    }
    bits = b;
  } else if (epi == EPI_MASK_BITS) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = (bits >> j) & 1u ? v[j] : 0.f;
  } else if (epi == EPI_BIAS_F32) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] += bias[j];
  }
  return dot;
}

// Write 16 output values of row `row` into a 64-byte-row staging block (64-byte TMA swizzle:
// 16-byte unit u of row r sits at unit u ^ ((r >> 1) & 3)); `unit0` = first 16-byte unit.
__device__ __forceinline__ void stage16(uint8_t* blk, int row, int unit0, const float (&v)[16], bool bf16) {
  uint8_t* rp = blk + row * 64;
  const int sw = (row >> 1) & 3;
  if (bf16) {
    const uint4 u0 = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
    const uint4 u1 = make_uint4(pack_bf16(v[8], v[9]), pack_bf16(v[10], v[11]), pack_bf16(v[12], v[13]),
                                pack_bf16(v[14], v[15]));
    *reinterpret_cast<uint4*>(rp + (((unit0 + 0) ^ sw) << 4)) = u0;
    *reinterpret_cast<uint4*>(rp + (((unit0 + 1) ^ sw) << 4)) = u1;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      *reinterpret_cast<float4*>(rp + (((unit0 + k) ^ sw) << 4)) = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  }
}

template <int BN, bool AMN, bool BMN>
__global__ void __launch_bounds__(NTHREADS, 1) tc_gemm_kernel(const __grid_constant__ TcParams p) {
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr uint32_t ACC_COLS = BN < 32 ? 32 : BN;  // one accumulator buffer
  constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;       // double-buffered
  constexpr int NW = (BN + 31) / 32, MSTR = NW + 1;
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((AMN ? 1u : 0u) << 15) | ((BMN ? 1u : 0u) << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NS = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* bias_s = reinterpret_cast<float*>(tmem_slot + 4);     // [BN] epilogue bias of the current tile
  float* dot_s = bias_s + BN;                                  // [BN] fused row-dot weights
  float* dotpart = dot_s + BN;                                 // [WPQ][BM] row-dot slices
  uint32_t* mask_s = reinterpret_cast<uint32_t*>(dotpart + WPQ * BM);  // [BM][MSTR] packed ReLU masks
  // per epilogue warp: two 32-row x 64-byte staging blocks for the TMA stores (1024-byte aligned)
  uint8_t* stage_s = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(mask_s + BM * MSTR) + 1023) & ~uintptr_t(1023));

  const GemmArgs& a = p.a;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = p.total_tiles;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < a.n_groups; ++i) {
      tma_prefetch(&p.ta[i]);
      tma_prefetch(&p.tb[i]);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], NUM_EPI_WARPS);
    }
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
  // everything above overlapped the previous kernel (PDL); from here on we read its outputs
  pdl_wait();
  pdl_launch();
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) g_trace[TRACE_CTAS * TRACE_TILES * 4 - 1] = (unsigned long long)T;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: a continuous stream of k-blocks over this CTA's tiles
      int kg = 0, tile_p = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x, ++tile_p) {
        trace(tile_p, 0);
        const TileInfo ti = decode_tile(p, t, BN);
        const int k_begin = ti.split * a.k_per_split;
        const int k_end = min(a.K, k_begin + a.k_per_split);
        const int nkb = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;
        for (int kb = 0; kb < nkb; ++kb, ++kg) {
          const int s = kg % NS;
          const uint32_t ph = (uint32_t)(kg / NS) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* sA = smem + s * STAGE;
          uint8_t* sB = sA + A_BYTES;
          mbar_expect_tx(&full[s], STAGE);
          const int k = k_begin + kb * BK;
          if (!AMN) {
            tma_load_2d(sA, &p.ta[ti.grp], &full[s], k, ti.m0);
          } else {
            tma_load_2d(sA, &p.ta[ti.grp], &full[s], ti.m0, k);
            tma_load_2d(sA + 8192, &p.ta[ti.grp], &full[s], ti.m0 + 64, k);
          }
          if (!BMN) {
            tma_load_2d(sB, &p.tb[ti.grp], &full[s], k, ti.n0);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i) tma_load_2d(sB + i * 8192, &p.tb[ti.grp], &full[s], ti.n0 + 64 * i, k);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: accumulator buffer (tile_i & 1), freed by the epilogue warps
      int kg = 0, tile_i = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x, ++tile_i) {
        const TileInfo ti = decode_tile(p, t, BN);
        const int k_begin = ti.split * a.k_per_split;
        const int k_end = min(a.K, k_begin + a.k_per_split);
        const int nkb = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;
        const int b = tile_i & 1;
        mbar_wait(&acc_empty[b], (((uint32_t)tile_i >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)b * ACC_COLS;
        for (int kb = 0; kb < nkb; ++kb, ++kg) {
          const int s = kg % NS;
          const uint32_t ph = (uint32_t)(kg / NS) & 1u;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sA = smem_u32(smem + s * STAGE);
          const uint32_t sB = sA + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = AMN ? desc_mnmajor(sA, kk) : desc_kmajor(sA, kk);
            const uint64_t bd = BMN ? desc_mnmajor(sB, kk) : desc_kmajor(sB, kk);
            umma_bf16(acc, ad, bd, IDESC, (kb | kk) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[s]);  // frees the smem stage once these MMAs have read it
        }
        umma_commit(&acc_full[b]);  // accumulator complete (immediately if the split is empty)
        trace(tile_i, 1);
      }
    }
  } else {
    // ---------------- epilogue: 8 warps; warp % 4 selects the TMEM lane quarter (32 rows) and
    //                  the two warps of a quarter split the columns (heads: one warp takes the row)
    const int e = warp - 2;
    const int q = warp & 3;
    const int hh = e >> 2;
    const bool head = a.epi == EPI_SAC_HEAD || a.epi == EPI_TD3_HEAD;
    // 16-column chunks per warp: whole 32-bit mask words per warp (>= 2 chunks)
    constexpr int CPW = (BN / 16) / WPQ >= 2 ? (BN / 16) / WPQ : 2;
    const bool split_cols = BN >= 64 && !head;
    const int c_lo = split_cols ? min(hh * CPW, BN / 16) : 0;    // first 16-column chunk of this warp
    const int c_hi = split_cols ? min((hh + 1) * CPW, BN / 16) : (hh == 0 ? BN / 16 : 0);
    const int r = q * 32 + lane;  // tile row of this thread
    uint32_t* mrow = mask_s + r * MSTR;
    int tile_i = 0;
    int st_count = 0;  // TMA store blocks issued by this warp
    for (int t = blockIdx.x; t < T; t += gridDim.x, ++tile_i) {
      const TileInfo ti = decode_tile(p, t, BN);
      const GemmGroup& g = a.g[ti.grp];
      const int m = ti.m0 + r;
      const int n0 = ti.n0;
      const int k_begin = ti.split * a.k_per_split;
      const int nkb = min(a.K, k_begin + a.k_per_split) > k_begin ? 1 : 0;
      const bool has_bias = a.epi == EPI_BIAS_RELU || a.epi == EPI_BIAS_F32 || head;
      const bool has_dot = a.epi == EPI_BIAS_RELU && g.dot_out != nullptr;
      const bool mask_in = a.epi == EPI_MASK_BITS;
      const bool mask_out = a.epi == EPI_BIAS_RELU && g.mask_out != nullptr;
      // stage this tile's bias / row-dot weights (after every epilogue warp left the previous tile)
      epi_bar(1);
      if (has_bias)
        for (int c = e * 32 + lane; c < BN; c += NUM_EPI_WARPS * 32) {
          bias_s[c] = n0 + c < g.N ? g.bias[n0 + c] : 0.f;
          dot_s[c] = (has_dot && n0 + c < g.N) ? g.dot_w[n0 + c] : 0.f;
        }
      if (mask_in) {  // this warp's words of the row's packed mask, prefetched before the accumulator wait
        const uint32_t* src = static_cast<const uint32_t*>(g.aux) + (int64_t)m * g.ldaux + n0 / 32;
        for (int i = c_lo / 2; i < (c_hi + 1) / 2; ++i) mrow[i] = (m < g.M && n0 + 32 * i < g.N) ? src[i] : 0u;
      }
      if (mask_out)
        for (int i = c_lo / 2; i < (c_hi + 1) / 2; ++i) mrow[i] = 0u;
      epi_bar(1);
      const int b = tile_i & 1;
      mbar_wait(&acc_full[b], ((uint32_t)tile_i >> 1) & 1u);
      tc_fence_after();
      if (e == 0 && lane == 0) trace(tile_i, 2);
      const uint32_t trow = tmem + (uint32_t)b * ACC_COLS + ((uint32_t)(q * 32) << 16);
      if (head) {
        if constexpr (BN <= 64) {
          if (hh == 0) {
            float hrow[BN];
#pragma unroll
            for (int c = 0; c < BN / 16; ++c) {
              float v[16];
              if (nkb > 0) tmem_ld16(trow + c * 16, v);
              else
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = 0.f;
#pragma unroll
              for (int j = 0; j < 16; ++j) hrow[c * 16 + j] = v[j] + bias_s[c * 16 + j];
            }
            tc_fence_before();
            if (m < g.M) {
              if (a.epi == EPI_SAC_HEAD) sac_head_row<__nv_bfloat16>(a.head, g.row0 + m, hrow, hrow + a.head.m);
              else td3_head_row<__nv_bfloat16>(a.head, g.row0 + m, hrow);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[b]);
      } else if (p.tma_out) {
        // ---- outputs staged in shared memory, written by TMA bulk tensor stores (64-byte x 32-row
        //      blocks, double-buffered per warp)
        float dot = 0.f;
        const bool obf = p.out_bytes == 2;
        const int cpb = obf ? 2 : 1;  // 16-column chunks per 64-byte store block
        uint8_t* wstage = stage_s + e * 4096;
#pragma unroll 1
        for (int c = c_lo; c < c_hi; c += cpb) {
          if (n0 + c * 16 >= g.N) break;  // warp-uniform
          if (st_count >= 2) {
            if (lane == 0) bulk_wait_read1();  // the block issued two stores ago has left this slot
            __syncwarp();
          }
          uint8_t* blk = wstage + (st_count & 1) * 2048;
          for (int cc = 0; cc < cpb; ++cc) {
            const int ch = c + cc;
            const int n = n0 + ch * 16;
            float v[16];
            if (nkb > 0 && n < g.N) {
              tmem_ld16(trow + ch * 16, v);
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = 0.f;
            }
            uint32_t bits = mask_in ? (mrow[ch >> 1] >> (16 * (ch & 1))) & 0xFFFFu : 0u;
            const float d = epi16_vals(a.epi, n, g.N, v, bias_s + ch * 16, has_dot ? dot_s + ch * 16 : nullptr, bits);
            if (m < g.M) {
              dot += d;
              if (mask_out) mrow[ch >> 1] |= bits << (16 * (ch & 1));
            }
            stage16(blk, lane, cc * (obf ? 2 : 4), v, obf);
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&p.tc[ti.grp], blk, n0 + c * 16, ti.m0 + q * 32, ti.split);
            bulk_commit();
          }
          ++st_count;
        }
        if (e == 0 && lane == 0) trace(tile_i, 3);
        // accumulator buffer drained by this warp
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[b]);
        if (has_dot) {
          dotpart[hh * BM + r] = dot;
          epi_bar(2);
          if (hh == 0 && m < g.M) {
            float tot = dot;
            if (split_cols) {
              tot = 0.f;
              for (int k = 0; k < WPQ; ++k) tot += dotpart[k * BM + r];  // fixed order
            }
            g.dot_out[m] = tot + g.dot_b[0];
          }
        }
        if (mask_out && m < g.M) {
          const int w_lo = c_lo / 2, w_hi = min((c_hi + 1) / 2, (g.N - n0 + 31) / 32);
          uint32_t* dst = g.mask_out + (int64_t)m * g.mask_ld + n0 / 32;
          if (w_hi - w_lo == 4 && ((reinterpret_cast<uintptr_t>(dst + w_lo) & 15) == 0)) {
            *reinterpret_cast<uint4*>(dst + w_lo) = make_uint4(mrow[w_lo], mrow[w_lo + 1], mrow[w_lo + 2], mrow[w_lo + 3]);
          } else {
            for (int i = w_lo; i < w_hi; ++i) dst[i] = mrow[i];
          }
        }
      } else {
        float dot = 0.f;
#pragma unroll 1
        for (int c = c_lo; c < c_hi; ++c) {
          const int n = n0 + c * 16;
          if (n >= g.N) break;  // warp-uniform
          float v[16];
          if (nkb > 0) {
            tmem_ld16(trow + c * 16, v);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.f;
          }
          uint32_t bits = mask_in ? (mrow[c >> 1] >> (16 * (c & 1))) & 0xFFFFu : 0u;
          if (m < g.M) {
            dot += epi16(a, g, ti.split, m, n, v, bias_s + c * 16, has_dot ? dot_s + c * 16 : nullptr, bits);
            if (mask_out) mrow[c >> 1] |= bits << (16 * (c & 1));
          }
        }
        // accumulator buffer drained by this warp
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[b]);
        if (has_dot) {
          dotpart[hh * BM + r] = dot;
          epi_bar(2);
          if (hh == 0 && m < g.M) {
            float tot = dot;
            if (split_cols) {
              tot = 0.f;
              for (int k = 0; k < WPQ; ++k) tot += dotpart[k * BM + r];  // fixed order
            }
            g.dot_out[m] = tot + g.dot_b[0];
          }
        }
        if (e == 0 && lane == 0) trace(tile_i, 3);
        if (mask_out && m < g.M) {
          const int w_lo = c_lo / 2, w_hi = min((c_hi + 1) / 2, (g.N - n0 + 31) / 32);
          uint32_t* dst = g.mask_out + (int64_t)m * g.mask_ld + n0 / 32;
          if (w_hi - w_lo == 4 && ((reinterpret_cast<uintptr_t>(dst + w_lo) & 15) == 0)) {
            *reinterpret_cast<uint4*>(dst + w_lo) = make_uint4(mrow[w_lo], mrow[w_lo + 1], mrow[w_lo + 2], mrow[w_lo + 3]);
          } else if (w_hi - w_lo == 2 && ((reinterpret_cast<uintptr_t>(dst + w_lo) & 7) == 0)) {
            *reinterpret_cast<uint2*>(dst + w_lo) = make_uint2(mrow[w_lo], mrow[w_lo + 1]);
          } else {
            for (int i = w_lo; i < w_hi; ++i) dst[i] = mrow[i];
          }
        }
      }
    }
  }
  if (warp >= 2 && lane == 0) bulk_wait_all();  // every TMA store of this warp has completed
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

// ------------------------------------------------------------------ host side
// tile tracing: 0 off; 1 every launch records (the last one wins); k >= 2 only the (k-2)-th launch from now
int g_trace_mode = 0;
long g_trace_count = 0;

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// 2-D bf16 tensor map: inner (contiguous) extent, outer extent, row pitch in elements, box.
bool make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
              uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN>
constexpr int smem_extras() {
  return 1024 /* alignment */ + 128 /* barriers + TMEM slot */ + BN * 8 /* bias, dot */ + WPQ * BM * 4 /* dot slices */ +
         BM * ((BN + 31) / 32 + 1) * 4 /* masks */ + 1024 + NUM_EPI_WARPS * 4096 /* TMA store staging */;
}

template <int BN, bool AMN, bool BMN>
cudaError_t launch(TcParams& p, int maxM, cudaStream_t st) {
  constexpr int STAGE = A_BYTES + BN * BK * 2;
  constexpr int MAX_ST = std::min(STAGES, (227 * 1024 - smem_extras<BN>()) / STAGE);
  static_assert(MAX_ST >= 1, "shared memory budget");
  constexpr int SMEM_MAX = MAX_ST * STAGE + smem_extras<BN>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  (void)maxM;
  // persistent schedule: tiles of every group, one CTA per SM (or more when TMEM and smem allow)
  int T = 0;
  for (int i = 0; i < p.a.n_groups; ++i) {
    const GemmGroup& g = p.a.g[i];
    p.tile0[i] = T;
    p.mtiles[i] = g.M > 0 && g.N > 0 ? (int)cdiv(g.M, BM) : 0;
    p.ntiles[i] = g.M > 0 && g.N > 0 ? (int)cdiv(g.N, BN) : 1;
    if (p.mtiles[i] == 0) p.mtiles[i] = 1, p.ntiles[i] = 0;
    T += p.mtiles[i] * p.ntiles[i] * p.a.splits;
  }
  p.tile0[p.a.n_groups] = T;
  p.total_tiles = T;
  if (T == 0) return cudaSuccess;
  constexpr int TMEM_COLS = 2 * (BN < 32 ? 32 : BN);
  static int occ = [] {
    int o = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, tc_gemm_kernel<BN, AMN, BMN>, NTHREADS, STAGE + smem_extras<BN>());
    return std::max(1, o);
  }();
  const int per_sm = std::max(1, std::min(512 / TMEM_COLS, occ));
  const int budget = 227 * 1024 / per_sm;
  const int kspan = p.a.splits > 1 ? p.a.k_per_split : p.a.K;
  const int want = (int)std::min<int64_t>(STAGES, std::max<int64_t>(1, cdiv(kspan, BK)));
  p.stages = std::max(1, std::min(std::min(want, MAX_ST), (budget - smem_extras<BN>()) / STAGE));
  const int smem = p.stages * STAGE + smem_extras<BN>();
  const int grid = std::min(T, num_sms() * per_sm);
  p.trace = g_trace_mode == 1 || (g_trace_mode >= 2 && g_trace_count == g_trace_mode - 2);
  ++g_trace_count;
  return launch_pdl(tc_gemm_kernel<BN, AMN, BMN>, dim3(grid), dim3(NTHREADS), (size_t)smem, st, p);
}

template <bool AMN, bool BMN>
cudaError_t launch_bn(TcParams& p, int bn, int maxM, cudaStream_t st) {
  switch (bn) {
    case 16: if constexpr (!BMN) return launch<16, AMN, BMN>(p, maxM, st); break;
    case 32: if constexpr (!BMN) return launch<32, AMN, BMN>(p, maxM, st); break;
    case 64: return launch<64, AMN, BMN>(p, maxM, st);
    case 128: return launch<128, AMN, BMN>(p, maxM, st);
    default: return launch<256, AMN, BMN>(p, maxM, st);
  }
  return cudaErrorInvalidValue;
}

int pick_bn(int N, bool bmn) {
  if (N > 128) return 256;
  if (N > 64) return 128;
  if (N > 32 || bmn) return 64;
  if (N > 16) return 32;
  return 16;
}

}  // namespace

bool tc_gemm_available() { return get_encode(); }

cudaError_t tc_trace(int on, unsigned long long* out, int n) {
  g_trace_mode = on;
  g_trace_count = 0;
  cudaError_t e = cudaSuccess;
  if (on) {
    static std::vector<unsigned long long> zeros(TRACE_CTAS * TRACE_TILES * 4, 0ull);
    e = cudaMemcpyToSymbol(g_trace, zeros.data(), zeros.size() * sizeof(unsigned long long));
  }
  if (e != cudaSuccess || !out) return e;
  n = std::min(n, TRACE_CTAS * TRACE_TILES * 4);
  return cudaMemcpyFromSymbol(out, g_trace, n * sizeof(unsigned long long));
}

bool tc_gemm_supported(const GemmArgs& a) {
  if (a.N < 1 || a.K < 1 || a.n_groups < 1 || a.n_groups > MAX_GROUPS) return false;
  if (a.splits > 1 && (a.k_per_split % BK)) return false;
  if (a.a_mn && !a.b_mn) return false;  // layout combination not instantiated
  const int bn = pick_bn(a.N, a.b_mn);
  if ((a.epi == EPI_SAC_HEAD || a.epi == EPI_TD3_HEAD) && bn > 64) return false;
  for (int i = 0; i < a.n_groups; ++i) {
    const GemmGroup& g = a.g[i];
    if ((g.lda & 7) || (g.ldb & 7)) return false;
    if ((reinterpret_cast<uintptr_t>(g.A) & 15) || (reinterpret_cast<uintptr_t>(g.B) & 15)) return false;
    if (g.dot_out && g.N > bn) return false;  // fused row dot needs the whole row in one tile
  }
  return get_encode();
}

// Output C of a group as a 3-D tensor [splits][M][N] for TMA bulk stores (64-byte inner box).
bool make_map_out(CUtensorMap* m, void* ptr, int esz, uint64_t N, uint64_t M, uint64_t splits, uint64_t ld,
                  uint64_t split_stride) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * esz) % 16 || (splits > 1 && (split_stride * esz) % 16)) return false;
  cuuint64_t dims[3] = {N, M, splits};
  cuuint64_t strides[2] = {ld * esz, (splits > 1 ? split_stride : ld * M) * esz};
  cuuint32_t box[3] = {(cuuint32_t)(64 / esz), 32, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t tc_gemm_bf16(const GemmArgs& a, cudaStream_t st) {
  TcParams p;
  std::memset(&p, 0, sizeof(p));
  p.a = a;
  // epilogue stores through TMA when every group's C qualifies (heads store nothing through C)
  const bool f32out = a.epi == EPI_F32 || a.epi == EPI_BIAS_F32;
  p.out_bytes = f32out ? 4 : 2;
  p.tma_out = (a.epi == EPI_BIAS_RELU || a.epi == EPI_MASK_BITS || f32out) ? 1 : 0;
  for (int i = 0; i < a.n_groups && p.tma_out; ++i) {
    const GemmGroup& g = a.g[i];
    if (g.M < 1 || g.N < 1) continue;
    if (!g.C || !make_map_out(&p.tc[i], g.C, p.out_bytes, g.N, g.M, a.splits, g.ldc, g.split_stride)) p.tma_out = 0;
  }
  const int bn = pick_bn(a.N, a.b_mn);
  int maxM = 0;
  for (int i = 0; i < a.n_groups; ++i) {
    const GemmGroup& g = a.g[i];
    maxM = g.M > maxM ? g.M : maxM;
    if (g.M < 1 || g.N < 1) continue;
    bool ok;
    if (!a.a_mn) ok = make_map(&p.ta[i], g.A, a.K, g.M, g.lda, BK, BM);      // A [M x K]
    else ok = make_map(&p.ta[i], g.A, g.M, a.K, g.lda, 64, BK);             // A stored [K x M]
    if (ok) {
      if (!a.b_mn) ok = make_map(&p.tb[i], g.B, a.K, g.N, g.ldb, BK, bn);    // B [N x K]
      else ok = make_map(&p.tb[i], g.B, g.N, a.K, g.ldb, 64, BK);           // B stored [K x N]
    }
    if (!ok) return cudaErrorInvalidValue;
  }
  if (maxM == 0) return cudaSuccess;
  if (!a.a_mn && !a.b_mn) return launch_bn<false, false>(p, bn, maxM, st);
  if (!a.a_mn && a.b_mn) return launch_bn<false, true>(p, bn, maxM, st);
  return launch_bn<true, true>(p, bn, maxM, st);
}

}  // namespace spz
