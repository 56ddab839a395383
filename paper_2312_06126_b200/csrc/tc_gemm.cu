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
#include "tc_common.cuh"

namespace spz {

namespace {

#ifndef SPZ_TC_STAGES
#define SPZ_TC_STAGES 4
#endif
constexpr int BM = 128, BK = 64, STAGES = SPZ_TC_STAGES;  // pipeline depth cap (shared memory decides below it)
// producer warp, MMA warp, WPQ epilogue warps per TMEM lane quarter (each a slice of the columns)
// Each launch picks 2 or 4 epilogue warps per lane quarter (template WPQ): 4 drain a tile's accumulator faster
// where the launch has under two tiles per SM (the WLK step's dgrad / wgrad: 100.8 -> 99.9 us per update), 2
// keep more shared memory for pipeline stages where many tiles stream (HUM: 1993 vs 2029 us per update with 4).
constexpr int gemm_threads(int w) { return 64 + 4 * w * 32; }
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
  int pair;       // 1: CTA-pair kernel (cta_group::2, M = 256 pair tiles; tb boxes hold BN / 2 rows)
  int wpq;        // epilogue warps per TMEM lane quarter (2 or 4)
  int dyn;        // 1: dynamic tile schedule (atomic counter a.sched), 0: static round robin
  int n_pre;      // dynamic schedule: linear tiles [0, n_pre) need no grid-dependency wait
  CUtensorMap ta[MAX_GROUPS];
  CUtensorMap tb[MAX_GROUPS];
  CUtensorMap tc[MAX_GROUPS];  // C as [splits][M][N]; box = 64 bytes x 32 rows, 64-byte swizzle
};

// Diagnostics: per-CTA, per-tile %globaltimer stamps (spz_diag_tc_trace).  Event e of the i-th tile of
// CTA c lands in g_trace[(c * TRACE_TILES + i) * 4 + e]: 0 producer starts the tile, 1 MMA issue done,
// 2 epilogue sees the accumulator, 3 epilogue done.
constexpr int TRACE_CTAS = 160, TRACE_TILES = 8;
__device__ unsigned long long g_trace[TRACE_CTAS * TRACE_TILES * 4];
__device__ int g_trace_tile[TRACE_CTAS * TRACE_TILES];  // linear tile index of each traced tile
__device__ unsigned long long g_trace_cta[TRACE_CTAS * 2];  // per CTA: kernel entry, producer past the dependency wait
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define trace(tile_i, ev) trace_(p.trace, tile_i, ev)
__device__ __forceinline__ void trace_(int on, int tile_i, int ev) {
  if (on && blockIdx.x < TRACE_CTAS && tile_i < TRACE_TILES) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[(blockIdx.x * TRACE_TILES + tile_i) * 4 + ev] = t;
  }
}

// Linear tile index -> (group, m0, n0, split).  Tiles of group g occupy [tile0[g], tile0[g+1]);
// within a group the N tile varies fastest, then the M tile, then the split: the N tiles of one row
// block run at the same time on neighbouring CTAs, so their common A tile comes from DRAM once and
// from L2 for the others (h = 512 forward: the 403 MB activation operand is no longer read twice).
struct TileInfo {
  int grp, m0, n0, split;
};
// CTA pair (p.pair): tiles are 256-row pair tiles (mtiles counts row-block PAIRS); CTA `rank` of the cluster
// takes row block 2 mt + rank (past M: TMA zero-fills it, the epilogue stores nothing).
__device__ __forceinline__ TileInfo decode_tile(const TcParams& p, int t, int bn, int rank = 0) {
  int g = 0;
  while (g + 1 < p.a.n_groups && t >= p.tile0[g + 1]) ++g;
  const int r = t - p.tile0[g];
  const int nt = r % p.ntiles[g];
  const int rest = r / p.ntiles[g];
  const int mt = rest % p.mtiles[g];
  return {g, (p.pair ? 2 * mt + rank : mt) * BM, nt * bn, rest / p.mtiles[g]};
}

// Write 16 output values of row `row` into a 64-byte-row staging block (64-byte TMA swizzle:
// 16-byte unit u of row r sits at unit u ^ ((r >> 1) & 3)); `unit0` = first 16-byte unit.
template <bool OBF>
__device__ __forceinline__ void stage16(uint8_t* blk, int row, int unit0, const float (&v)[16]) {
  uint8_t* rp = blk + row * 64;
  const int sw = (row >> 1) & 3;
  if constexpr (OBF) {
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

// Direct (non-TMA) store of 16 output values at C(m, n..n+15) + split partial offset; used when
// an output pitch cannot be described by a tensor map.
template <bool OBF>
__device__ __forceinline__ void direct16(const GemmGroup& g, int split, int m, int n, const float (&v)[16]) {
  if (m >= g.M) return;
  const int64_t off = (int64_t)m * g.ldc + n;
  const bool full = n + 16 <= g.N;
  if constexpr (OBF) {
    __nv_bfloat16* C = static_cast<__nv_bfloat16*>(g.C) + off;
    if (full && (reinterpret_cast<uintptr_t>(C) & 15) == 0) {
      uint4* d = reinterpret_cast<uint4*>(C);
      d[0] = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
      d[1] = make_uint4(pack_bf16(v[8], v[9]), pack_bf16(v[10], v[11]), pack_bf16(v[12], v[13]), pack_bf16(v[14], v[15]));
    } else {
      for (int j = 0; j < 16 && n + j < g.N; ++j) C[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* C = static_cast<float*>(g.C) + off + (int64_t)split * g.split_stride;
    if (full && (reinterpret_cast<uintptr_t>(C) & 15) == 0) {
      float4* d4 = reinterpret_cast<float4*>(C);
#pragma unroll
      for (int j = 0; j < 4; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
      for (int j = 0; j < 16 && n + j < g.N; ++j) C[j] = v[j];
    }
  }
}

// Epilogue shape of one (BN, EK) instantiation.
template <int BN, int EK, int WPQ>
struct EpiShape {
  static constexpr bool HEAD = EK == EPI_SAC_HEAD;
  static constexpr bool RELU = EK == EPI_BIAS_RELU;
  static constexpr bool MASKB = EK == EPI_MASK_BITS;
  static constexpr bool BIASCOL = EK == EPI_WGRAD_BIAS;  // + row sums of A through an all-ones MMA
  static constexpr bool BIAS = RELU || HEAD || EK == EPI_BIAS_F32;
  static constexpr bool OBF = RELU || MASKB;            // bf16 output, else fp32
  static constexpr bool SPLIT = BN >= 64 && !HEAD;      // the WPQ warps of a lane quarter split the columns
  static constexpr int CPW = SPLIT ? BN / 16 / WPQ : BN / 16;  // 16-column chunks per warp
  static constexpr int CPB = OBF ? 2 : 1;               // chunks per 64-byte store block (= one mask word)
  static constexpr int NB = (CPW + CPB - 1) / CPB;      // store blocks per warp
  static constexpr int SLICE = CPW * 16;                // columns per warp
  static_assert(!SPLIT || CPW >= CPB || BN < 64 || WPQ == 2,
                "a warp's column slice must fill whole 64-byte store blocks (4 warps per quarter need BN >= 128)");
  // TMEM: NBUF accumulator buffers of BUF_COLS columns (BIASCOL: + 16 row-sum columns at BN)
  static constexpr int ACC_COLS = BN < 32 ? 32 : BN;
  static constexpr int BUF_COLS = BIASCOL ? ACC_COLS + 16 : ACC_COLS;
  static constexpr int NBUF = 2 * BUF_COLS <= 512 ? 2 : 1;
  static constexpr int TMEM_COLS = NBUF * BUF_COLS <= 32 ? 32 : NBUF * BUF_COLS <= 64 ? 64 : NBUF * BUF_COLS <= 128 ? 128
                                   : NBUF * BUF_COLS <= 256 ? 256 : 512;
};

// Persistent, warp-specialized: each CTA walks tiles blockIdx.x, +gridDim.x, ...; the TMA producer
// and the MMA issuer run ahead into the next tile while the epilogue drains the previous one
// from the other TMEM accumulator buffer.  EK (the epilogue kind) is a template parameter so the
// epilogue compiles to straight-line code for exactly one kind (SAC_HEAD also covers TD3_HEAD).
// PAIR: a 2-CTA cluster on one TPC computes 256 x BN pair tiles with cta_group::2 MMAs issued by the even
// (leader) CTA: each CTA stages its own 128 A rows and half of the B tile's rows (BN / 2) per k-block -- 32 KB
// per CTA per k-block instead of 48 KB at BN = 256, which the k-block pipeline (TMA latency x stages) was
// bound by -- and drains its own 128 accumulator rows from its own TMEM with the unchanged epilogue.
template <int BN, bool AMN, bool BMN, int EK, bool PAIR, int WPQ>
__global__ void __launch_bounds__(gemm_threads(WPQ), 1) tc_gemm_kernel(const __grid_constant__ TcParams p) {
  constexpr int NUM_EPI_WARPS = 4 * WPQ, NTHREADS = gemm_threads(WPQ);
  using S = EpiShape<BN, EK, WPQ>;
  static_assert(!PAIR || (!AMN && !BMN && !S::HEAD && !S::BIASCOL && BN == 256), "CTA pair: K-major forward tiles only");
  constexpr int B_BYTES = PAIR ? BN * BK * 2 / 2 : BN * BK * 2;  // this CTA's share of the B tile
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr uint32_t BUF_COLS = S::BUF_COLS;    // one accumulator buffer
  constexpr uint32_t TMEM_COLS = S::TMEM_COLS;
  constexpr int NBUF = S::NBUF;
  // all-ones operand (N = 16, K-major) for the row sums of A
  constexpr uint32_t IDESC1 = (1u << 4) | (1u << 7) | (1u << 10) | ((AMN ? 1u : 0u) << 15) | (2u << 17) |
                              ((uint32_t)(BM >> 4) << 24);
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((AMN ? 1u : 0u) << 15) | ((BMN ? 1u : 0u) << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((PAIR ? 2 * BM : BM) >> 4) << 24);
  // per epilogue warp: its slice of the tile's bias / row-dot weights; row-dot partials per quarter
  __shared__ __align__(16) float bias_w[S::BIAS ? NUM_EPI_WARPS : 1][S::BIAS ? S::SLICE : 4];
  __shared__ __align__(16) float dotw_w[S::RELU ? NUM_EPI_WARPS : 1][S::RELU ? S::SLICE : 4];
  __shared__ float dotpart[S::RELU ? 2 : 1][S::RELU ? WPQ : 1][S::RELU ? BM : 1];
  __shared__ float headpart[S::HEAD ? 2 : 1][S::HEAD ? WPQ : 1][S::HEAD ? BM : 1];  // SAC log-pi parts
  // dynamic schedule: the producer's tile sequence, handed to the MMA issuer and the epilogue warps
  constexpr int TQ = 8;
  __shared__ int tq[TQ];
  __shared__ __align__(8) uint64_t tq_full[TQ], tq_empty[TQ];
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NS = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // per epilogue warp: two 32-row x 64-byte staging blocks for the TMA stores (1024-byte aligned)
  uint8_t* stage_s = smem + NS * STAGE + 1024;
  uint8_t* ones_s = stage_s + NUM_EPI_WARPS * 4096;  // 16 x 64 bf16 ones (2 KB, 1024-aligned)
  if constexpr (S::BIASCOL) {
    for (int i = threadIdx.x; i < 2048 / 16; i += NTHREADS)
      reinterpret_cast<uint4*>(ones_s)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    fence_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
  }

  const GemmArgs& a = p.a;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = p.total_tiles;
  const int crank = PAIR ? (int)cluster_rank() : 0;  // 0: the leader CTA of the pair (issues every MMA)
  const int cta0 = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;  // schedule index: the pair walks pair tiles
  const int ncta = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;

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
      mbar_init(&acc_empty[b], PAIR ? 2 * NUM_EPI_WARPS : NUM_EPI_WARPS);  // pair: both CTAs' epilogues (leader's)
    }
    for (int i = 0; i < TQ; ++i) {
      mbar_init(&tq_full[i], 1);                   // the producer publishes the slot's tile
      mbar_init(&tq_empty[i], 1 + NUM_EPI_WARPS);  // the MMA issuer and every epilogue warp have read it
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // both CTAs' barriers initialised before any cross-CTA arrive / TMA
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // everything above overlapped the previous kernel (PDL); from here on we read its outputs -- except under a
  // dynamic schedule with independent leading tiles, where only the producer waits, before the first tile that
  // reads them (nothing else in the CTA reads memory that kernel wrote: MMA operands arrive through the producer)
  if (p.trace && blockIdx.x < TRACE_CTAS && threadIdx.x == 0) g_trace_cta[blockIdx.x * 2] = gtimer();
  const bool dyn = !PAIR && p.dyn;
  const bool lazy_wait = dyn && p.n_pre > 0;
  if (!lazy_wait) pdl_wait();
  pdl_launch();
  // tile sequence: static round robin, or (dyn) the producer claims tiles from the counter and publishes
  // each in the queue slot i % TQ; consumers read slot i and release it
  auto claim = [&](int i) -> int {  // producer lane only
    const int sl = i % TQ;
    mbar_wait(&tq_empty[sl], ((uint32_t)(i / TQ) & 1u) ^ 1u);
    int t = (int)atomicAdd(a.sched, 1u);
    if (t > T) t = T;
    tq[sl] = t;
    mbar_arrive(&tq_full[sl]);
    return t;
  };
  auto fetch = [&](int i, bool warp_release) -> int {  // MMA lane (warp_release false) / epilogue warp
    const int sl = i % TQ;
    mbar_wait(&tq_full[sl], (uint32_t)(i / TQ) & 1u);
    const int t = *reinterpret_cast<volatile int*>(&tq[sl]);
    if (warp_release) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&tq_empty[sl]);
    } else {
      mbar_arrive(&tq_empty[sl]);
    }
    return t;
  };
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) g_trace[TRACE_CTAS * TRACE_TILES * 4 - 1] = (unsigned long long)T;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: a continuous stream of k-blocks over this CTA's tiles
      int kg = 0, tile_p = 0;
      bool waited = !lazy_wait;
      for (int t = dyn ? claim(0) : cta0; t < T; t = dyn ? claim(tile_p + 1) : t + ncta, ++tile_p) {
        if (!waited && t >= p.n_pre) {
          pdl_wait();
          waited = true;
          if (p.trace && blockIdx.x < TRACE_CTAS) g_trace_cta[blockIdx.x * 2 + 1] = gtimer();
        }
        trace(tile_p, 0);
        if (p.trace && blockIdx.x < TRACE_CTAS && tile_p < TRACE_TILES) g_trace_tile[blockIdx.x * TRACE_TILES + tile_p] = t;
        const TileInfo ti = decode_tile(p, t, BN, crank);
        const int kps = group_kps(a.g[ti.grp], a.k_per_split);
        const int k_begin = ti.split * kps;
        const int k_end = min(a.K, k_begin + kps);
        const int nkb = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;
        for (int kb = 0; kb < nkb; ++kb, ++kg) {
          const int s = kg % NS;
          const uint32_t ph = (uint32_t)(kg / NS) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* sA = smem + s * STAGE;
          uint8_t* sB = sA + A_BYTES;
          const int k = k_begin + kb * BK;
          if constexpr (PAIR) {
            // both CTAs' loads complete on the leader's full[s] (it expects the pair's bytes)
            if (crank == 0) mbar_expect_tx(&full[s], 2 * STAGE);
            tma_load_2d_pair(sA, &p.ta[ti.grp], &full[s], k, ti.m0);
            tma_load_2d_pair(sB, &p.tb[ti.grp], &full[s], k, ti.n0 + crank * (BN / 2));
            continue;
          }
          mbar_expect_tx(&full[s], STAGE);
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
      // the grid completes only after the kernel it was launched behind: later kernels rely on that
      if (!waited) pdl_wait();
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {
      // ---------------- MMA issuer: accumulator buffer (tile_i & 1), freed by the epilogue warps
      //                  (pair: the leader issues the pair's M = 256 MMAs; commits reach both CTAs)
      int kg = 0, tile_i = 0;
      for (int t = dyn ? fetch(0, false) : cta0; t < T; t = dyn ? fetch(tile_i + 1, false) : t + ncta, ++tile_i) {
        const TileInfo ti = decode_tile(p, t, BN, crank);
        const int kps = group_kps(a.g[ti.grp], a.k_per_split);
        const int k_begin = ti.split * kps;
        const int k_end = min(a.K, k_begin + kps);
        const int nkb = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;
        const int b = tile_i % NBUF;
        mbar_wait(&acc_empty[b], (((uint32_t)(tile_i / NBUF)) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)b * BUF_COLS;
        const bool bcol = S::BIASCOL && ti.n0 == 0 && a.g[ti.grp].colsum_out != nullptr;
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
            if constexpr (PAIR) umma_bf16_pair(acc, ad, bd, IDESC, (kb | kk) != 0 ? 1u : 0u);
            else umma_bf16(acc, ad, bd, IDESC, (kb | kk) != 0 ? 1u : 0u);
          }
          if constexpr (S::BIASCOL) {
            if (bcol) {
              const uint32_t so = smem_u32(ones_s);
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint64_t ad = AMN ? desc_mnmajor(sA, kk) : desc_kmajor(sA, kk);
                umma_bf16(acc + S::ACC_COLS, ad, desc_kmajor(so, kk), IDESC1, (kb | kk) != 0 ? 1u : 0u);
              }
            }
          }
          if constexpr (PAIR) umma_commit_pair(&empty[s]);  // frees the stage in both CTAs once read
          else umma_commit(&empty[s]);  // frees the smem stage once these MMAs have read it
        }
        if constexpr (PAIR) umma_commit_pair(&acc_full[b]);
        else umma_commit(&acc_full[b]);  // accumulator complete (immediately if the split is empty)
        trace(tile_i, 1);
      }
    }
  } else {
    // ---------------- epilogue: warp % 4 selects the TMEM lane quarter (32 rows); the WPQ warps of
    //                  a quarter split the columns (heads: one warp takes the whole row)
    const int e = warp - 2;
    const int q = warp & 3;
    const int hh = e >> 2;
    const bool active = S::SPLIT || hh == 0;
    const int c_lo = S::SPLIT ? hh * S::CPW : 0;  // first 16-column chunk of this warp
    const int r = q * 32 + lane;                  // tile row of this thread
    float* bias_s = bias_w[S::BIAS ? e : 0];
    float* dot_s = dotw_w[S::RELU ? e : 0];
    int tile_i = 0;
    int st_count = 0;   // TMA store blocks issued by this warp
    int dot_tiles = 0;  // fused row-dot tiles seen (dotpart buffer parity)
    const uint32_t acc_empty0 = PAIR ? mapa_shared(smem_u32(acc_empty), 0) : 0u;  // the leader's acc_empty[0]
    for (int t = dyn ? fetch(0, true) : cta0; t < T; t = dyn ? fetch(tile_i + 1, true) : t + ncta, ++tile_i) {
      const TileInfo ti = decode_tile(p, t, BN, crank);
      const GemmGroup& g = a.g[ti.grp];
      const int m = ti.m0 + r;
      const int n0 = ti.n0;
      const int ncol0 = n0 + c_lo * 16;  // first output column of this warp
      const int kps = group_kps(g, a.k_per_split);
      const int k_begin = ti.split * kps;
      const bool has_acc = min(a.K, k_begin + kps) > k_begin;
      const bool has_dot = S::RELU && g.dot_out != nullptr;
      const bool mask_out = S::RELU && g.mask_out != nullptr;
      // this warp's slice of the bias / row-dot weights (the previous tile's reads of the slice
      // are ordered by the __syncwarp that precedes every acc_empty arrival)
      if constexpr (S::BIAS) {
#pragma unroll
        for (int c = lane; c < S::SLICE; c += 32) {
          const int n = ncol0 + c;
          bias_s[c] = n < g.N ? g.bias[n] : 0.f;
          if constexpr (S::RELU) dot_s[c] = (has_dot && n < g.N) ? g.dot_w[n] : 0.f;
        }
      }
      // packed ReLU mask words of this row (dgrad), prefetched before the accumulator wait
      uint32_t mw[S::NB];
#pragma unroll
      for (int i = 0; i < S::NB; ++i) mw[i] = 0u;
      if constexpr (S::MASKB) {
        if (active && m < g.M) {
          const uint32_t* src = static_cast<const uint32_t*>(g.aux) + (int64_t)m * g.ldaux + ncol0 / 32;
#pragma unroll
          for (int i = 0; i < S::NB; ++i)
            if (ncol0 + 32 * i < g.N) mw[i] = __ldg(src + i);
        }
      }
      __syncwarp();
      const int b = tile_i % NBUF;
      mbar_wait(&acc_full[b], ((uint32_t)(tile_i / NBUF)) & 1u);
      tc_fence_after();
      if (e == 0 && lane == 0) trace(tile_i, 2);
      const uint32_t trow = tmem + (uint32_t)b * BUF_COLS + ((uint32_t)(q * 32) << 16);
      if constexpr (S::HEAD) {
        // the WPQ warps of a lane quarter share each row: warp hh takes the Philox blocks of 4 actions
        // hh, hh + WPQ, ...; the SAC log-pi parts are summed in warp order
        float hrow[BN];
#pragma unroll
        for (int c = 0; c < BN / 16; ++c) {
          float v[16];
          if (has_acc) tmem_ld16(trow + c * 16, v);
          else
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.f;
#pragma unroll
          for (int j = 0; j < 16; ++j) hrow[c * 16 + j] = v[j] + bias_s[c * 16 + j];
        }
        tc_fence_before();
        const bool live = m < g.M;
        if (a.epi == EPI_SAC_HEAD) {
          const float lp = live ? sac_head_blocks<__nv_bfloat16>(a.head, g.row0 + m, hrow, hrow + a.head.m, hh, WPQ) : 0.f;
          const int pb = tile_i & 1;
          headpart[pb][hh][r] = lp;
          named_bar(2 + q, WPQ * 32);
          if (hh == 0 && live) {
            float tot = 0.f;
#pragma unroll
            for (int k = 0; k < WPQ; ++k) tot += headpart[pb][k][r];
            sac_head_logp(a.head, g.row0 + m, tot);
          }
        } else if (live) {
          td3_head_blocks<__nv_bfloat16>(a.head, g.row0 + m, hrow, hh, WPQ);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[b]);
      } else {
        float dot2[2] = {0.f, 0.f};  // row-dot partials of the even / odd columns
        uint8_t* wstage = stage_s + e * 4096;
#pragma unroll
        for (int ib = 0; ib < S::NB; ++ib) {
          const int c = c_lo + ib * S::CPB;           // first chunk of this store block
          if (!active || n0 + c * 16 >= g.N) break;  // warp-uniform
          uint8_t* blk = wstage + (st_count & 1) * 2048;
          if (p.tma_out && st_count >= 2) {
            if (lane == 0) bulk_wait_read1();  // the block issued two stores ago has left this slot
            __syncwarp();
          }
          float v[S::CPB][16];
          if (has_acc) {
            if constexpr (S::CPB == 2 && S::CPW >= 2) {
              tmem_ld32(trow + c * 16, v[0], v[1]);
            } else {
              tmem_ld16(trow + c * 16, v[0]);
#pragma unroll
              for (int cc = 1; cc < S::CPB; ++cc)
#pragma unroll
                for (int j = 0; j < 16; ++j) v[cc][j] = 0.f;  // past the tile (BN = 16)
            }
          } else {
#pragma unroll
            for (int cc = 0; cc < S::CPB; ++cc)
#pragma unroll
              for (int j = 0; j < 16; ++j) v[cc][j] = 0.f;
          }
          uint32_t word = 0u;
#pragma unroll
          for (int cc = 0; cc < S::CPB; ++cc) {
            const int cl = ib * S::CPB + cc;  // chunk within this warp's slice
            if (cl >= S::CPW) break;          // past the tile (BN = 16): stays zero
            if constexpr (S::RELU) {
              // columns past N: zero-filled B rows and zero bias -> pre = 0 -> bit 0, value 0.  Column
              // pairs in packed fp32 (FADD2 / FFMA2); the row dot keeps even / odd column partials.
#pragma unroll
              for (int j = 0; j < 16; j += 2) {
                const float2 b2 = *reinterpret_cast<const float2*>(bias_s + cl * 16 + j);
                const float2 w2 = *reinterpret_cast<const float2*>(dot_s + cl * 16 + j);
                float p0, p1;
                add2(p0, p1, v[cc][j], v[cc][j + 1], b2.x, b2.y);
                word |= mask_pair(p0, p1, 16 * cc + j);
                v[cc][j] = fmaxf(p0, 0.f);
                v[cc][j + 1] = fmaxf(p1, 0.f);
                fma2(dot2[0], dot2[1], v[cc][j], v[cc][j + 1], w2.x, w2.y);
              }
              continue;
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if constexpr (S::MASKB) {
                v[cc][j] = (mw[ib] >> (16 * cc + j)) & 1u ? v[cc][j] : 0.f;
              } else if constexpr (S::BIAS) {
                v[cc][j] += bias_s[cl * 16 + j];
              }
            }
          }
          if constexpr (S::RELU) mw[ib] = word;
          if (p.tma_out) {
#pragma unroll
            for (int cc = 0; cc < S::CPB; ++cc) stage16<S::OBF>(blk, lane, cc * (S::OBF ? 2 : 4), v[cc]);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&p.tc[ti.grp], blk, n0 + c * 16, ti.m0 + q * 32, ti.split);
              bulk_commit();
            }
            ++st_count;
          } else {
#pragma unroll
            for (int cc = 0; cc < S::CPB; ++cc)
              if (n0 + (c + cc) * 16 < g.N) direct16<S::OBF>(g, ti.split, m, n0 + (c + cc) * 16, v[cc]);
          }
        }
        if constexpr (S::BIASCOL) {
          // row sums of A (every one of the 16 columns holds the same sum)
          if (hh == 0 && ti.n0 == 0 && g.colsum_out != nullptr) {
            float v[16];
            if (has_acc) tmem_ld16(trow + S::ACC_COLS, v);
            else v[0] = 0.f;
            if (m < g.M) g.colsum_out[(int64_t)ti.split * g.colsum_stride + m] = v[0];
          }
        }
        if (e == 0 && lane == 0) trace(tile_i, 3);
        // accumulator buffer drained by this warp
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_cluster(acc_empty0 + (uint32_t)b * 8u);
          else mbar_arrive(&acc_empty[b]);
        }
        if constexpr (S::RELU) {
          if (has_dot) {
            // the WPQ warps of this lane quarter combine their row-dot slices in a fixed order
            // (dotpart double-buffered by tile parity; the quarter barrier orders reuse)
            const float dot = dot2[0] + dot2[1];
            float tot = dot;
            if constexpr (S::SPLIT) {
              const int pb = dot_tiles & 1;
              dotpart[pb][hh][r] = dot;
              named_bar(2 + q, WPQ * 32);
              tot = 0.f;
#pragma unroll
              for (int k = 0; k < WPQ; ++k) tot += dotpart[pb][k][r];
            }
            ++dot_tiles;
            if (hh == 0 && m < g.M) g.dot_out[(int64_t)(n0 / BN) * g.dot_pstride + m] = tot + (n0 == 0 ? g.dot_b[0] : 0.f);
          }
          if (mask_out && active && m < g.M) {
            const int w_hi = min(S::NB, (g.N - ncol0 + 31) / 32);
            uint32_t* dst = g.mask_out + (int64_t)m * g.mask_ld + ncol0 / 32;
            if (S::NB == 4 && w_hi == 4 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
              *reinterpret_cast<uint4*>(dst) = make_uint4(mw[0], mw[S::NB > 1 ? 1 : 0], mw[S::NB > 2 ? 2 : 0], mw[S::NB > 3 ? 3 : 0]);
            } else if (S::NB == 2 && w_hi == 2 && (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
              *reinterpret_cast<uint2*>(dst) = make_uint2(mw[0], mw[S::NB > 1 ? 1 : 0]);
            } else {
#pragma unroll
              for (int i = 0; i < S::NB; ++i)
                if (i < w_hi) dst[i] = mw[i];
            }
          }
        }
      }
    }
  }
  if (warp >= 2 && lane == 0) bulk_wait_all();  // every TMA store of this warp has completed
  tc_fence_before();
  if constexpr (PAIR) {
    cluster_sync();  // no CTA leaves while its peer may still arrive on its barriers or read its operands
    if (warp == 1) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
    }
  } else {
    __syncthreads();
    if (warp == 1) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
    }
    // dynamic schedule: every CTA claimed its last tile (>= T) before arriving here; the last CTA to arrive
    // resets the counters for the next launch (which starts only after this grid completes)
    if (dyn && threadIdx.x == 0) {
      if (atomicAdd(a.sched + 1, 1u) == gridDim.x - 1) {
        a.sched[0] = 0u;
        a.sched[1] = 0u;
      }
    }
  }
}

// ------------------------------------------------------------------ host side
// tile tracing: 0 off; 1 every launch records (the last one wins); k >= 2 only the (k-2)-th launch from now
int g_trace_mode = 0;
long g_trace_count = 0;

// dynamic shared memory besides the pipeline stages: alignment slack, barriers + TMEM slot,
// per-warp TMA store staging, the all-ones operand
template <int WPQ>
constexpr int smem_extras() { return 1024 + 1024 + 4 * WPQ * 4096 + 2048; }
// static shared memory of one instantiation (per-warp bias / row-dot slices, row-dot partials)
template <int BN, int EK, int WPQ>
constexpr int smem_static() {
  using S = EpiShape<BN, EK, WPQ>;
  return (S::BIAS ? 4 * WPQ * S::SLICE * 4 : 16) + (S::RELU ? 4 * WPQ * S::SLICE * 4 : 16) +
         (S::RELU ? 2 * WPQ * BM * 4 : 4) + 64;
}

template <int BN, bool AMN, bool BMN, int EK, bool PAIR, int WPQ>
cudaError_t launch(TcParams& p, cudaStream_t st) {
  constexpr int NTHREADS = gemm_threads(WPQ);
  constexpr int STAGE = A_BYTES + (PAIR ? BN * BK : BN * BK * 2);
  constexpr int AVAIL = 227 * 1024 - smem_static<BN, EK, WPQ>() - smem_extras<WPQ>();
  constexpr int MAX_ST = std::min(STAGES, AVAIL / STAGE);
  static_assert(MAX_ST >= 1, "shared memory budget");
  constexpr int SMEM_MAX = MAX_ST * STAGE + smem_extras<WPQ>();
  auto kern = tc_gemm_kernel<BN, AMN, BMN, EK, PAIR, WPQ>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once(attr, kern, SMEM_MAX); e != cudaSuccess) return e;
  // persistent schedule: tiles of every group, one CTA per SM (or more when TMEM and smem allow)
  int T = 0;
  p.pair = PAIR ? 1 : 0;
  for (int i = 0; i < p.a.n_groups; ++i) {
    const GemmGroup& g = p.a.g[i];
    p.tile0[i] = T;
    p.mtiles[i] = g.M > 0 && g.N > 0 ? (int)cdiv(g.M, PAIR ? 2 * BM : BM) : 0;  // pair: 256-row pair tiles
    p.ntiles[i] = g.M > 0 && g.N > 0 ? (int)cdiv(g.N, BN) : 1;
    if (p.mtiles[i] == 0) p.mtiles[i] = 1, p.ntiles[i] = 0;
    T += p.mtiles[i] * p.ntiles[i] * group_splits(g, p.a.splits);
  }
  p.tile0[p.a.n_groups] = T;
  p.total_tiles = T;
  p.dyn = !PAIR && p.a.sched != nullptr ? 1 : 0;
  p.n_pre = p.dyn ? p.tile0[std::max(0, std::min(p.a.n_pre_groups, p.a.n_groups))] : 0;
  if (T == 0) return cudaSuccess;
  constexpr int TMEM_COLS = EpiShape<BN, EK, WPQ>::TMEM_COLS;
  static int occ = [&] {
    int o = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, NTHREADS, STAGE + smem_extras<WPQ>());
    return std::max(1, o);
  }();
  const int per_sm = std::max(1, std::min(512 / TMEM_COLS, occ));
  const int budget = 227 * 1024 / per_sm - smem_static<BN, EK, WPQ>();
  int kspan = 0;  // longest contraction of one tile
  for (int i = 0; i < p.a.n_groups; ++i)
    kspan = std::max(kspan, group_splits(p.a.g[i], p.a.splits) > 1 ? group_kps(p.a.g[i], p.a.k_per_split) : p.a.K);
  const int want = (int)std::min<int64_t>(STAGES, std::max<int64_t>(1, cdiv(kspan, BK)));
  p.stages = std::max(1, std::min(std::min(want, MAX_ST), (budget - smem_extras<WPQ>()) / STAGE));
  const int smem = p.stages * STAGE + smem_extras<WPQ>();
  p.trace = g_trace_mode == 1 || (g_trace_mode >= 2 && g_trace_count == g_trace_mode - 2);
  ++g_trace_count;
  if constexpr (PAIR) {
    // one 2-CTA cluster per TPC: as many pairs as can be co-resident, each walking pair tiles
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    static int max_clusters = [&] {
      cudaLaunchConfig_t c = cfg;
      c.gridDim = dim3(2 * (num_sms() / 2));
      c.numAttrs = 1;  // cluster shape only
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &c) != cudaSuccess || n < 1) {
        cudaGetLastError();
        n = num_sms() / 2 - 4;  // conservative: leave room for TPCs with one usable SM
      }
      return n;
    }();
    cfg.gridDim = dim3(2 * std::min(T, max_clusters));
    return cudaLaunchKernelEx(&cfg, kern, p);
  }
  const int grid = std::min(T, num_sms() * per_sm);
  return launch_pdl(kern, dim3(grid), dim3(NTHREADS), (size_t)smem, st, p);
}

// CTA-pair kernel for a K-major forward GEMM (BN = 256).  Measured on B200: no faster than the
// single-CTA kernel on the HUM / TD3 hidden layers (HUM critic forward 588 -> 652 us, TD3 2627 -> 2611 us, with 4 or
// 8 pipeline stages alike), so the hidden-layer GEMMs are not bound by operand delivery and the pair kernel is
// off by default; SPZ_TC_PAIR=1 selects it wherever legal (parity- and unit-tested).
bool want_pair(const GemmArgs& a, int bn) {
  if (a.a_mn || a.b_mn || bn != 256) return false;
  if (a.epi != EPI_BIAS_RELU && a.epi != EPI_BIAS_F32 && a.epi != EPI_F32) return false;
  const char* fe = std::getenv("SPZ_TC_PAIR");
  return fe && std::atoi(fe) == 1;
}

// epilogue kinds instantiated per operand layout: forward (K-major A and B), dgrad (MN-major B),
// wgrad (both MN-major)
template <bool AMN, bool BMN>
constexpr bool ek_ok(int epi, int bn) {
  if (!AMN && !BMN)
    return epi == EPI_BIAS_RELU || epi == EPI_BIAS_F32 || epi == EPI_F32 ||
           ((epi == EPI_SAC_HEAD || epi == EPI_TD3_HEAD) && bn <= 64);
  if (!AMN && BMN) return epi == EPI_MASK_BITS || epi == EPI_F32;
  if (AMN && BMN) return epi == EPI_F32 || epi == EPI_WGRAD_BIAS;
  return false;
}

template <int BN, bool AMN, bool BMN, int W>
cudaError_t launch_ek_w(TcParams& p, cudaStream_t st) {
  if constexpr (!AMN && !BMN && BN == 256) {
    if (p.pair) {
      switch (p.a.epi) {
        case EPI_BIAS_RELU: return launch<BN, AMN, BMN, EPI_BIAS_RELU, true, W>(p, st);
        case EPI_BIAS_F32: return launch<BN, AMN, BMN, EPI_BIAS_F32, true, W>(p, st);
        case EPI_F32: return launch<BN, AMN, BMN, EPI_F32, true, W>(p, st);
        default: return cudaErrorInvalidValue;
      }
    }
  }
  if constexpr (!AMN && !BMN) {
    switch (p.a.epi) {
      case EPI_BIAS_RELU: return launch<BN, AMN, BMN, EPI_BIAS_RELU, false, W>(p, st);
      case EPI_BIAS_F32: return launch<BN, AMN, BMN, EPI_BIAS_F32, false, W>(p, st);
      case EPI_F32: return launch<BN, AMN, BMN, EPI_F32, false, W>(p, st);
      case EPI_SAC_HEAD:
      case EPI_TD3_HEAD:
        if constexpr (BN <= 64) return launch<BN, AMN, BMN, EPI_SAC_HEAD, false, W>(p, st);
        break;
      default: break;
    }
  } else if constexpr (!AMN && BMN) {
    if (p.a.epi == EPI_MASK_BITS) return launch<BN, AMN, BMN, EPI_MASK_BITS, false, W>(p, st);
    if (p.a.epi == EPI_F32) return launch<BN, AMN, BMN, EPI_F32, false, W>(p, st);
  } else {
    if (p.a.epi == EPI_F32) return launch<BN, AMN, BMN, EPI_F32, false, W>(p, st);
    if (p.a.epi == EPI_WGRAD_BIAS) return launch<BN, AMN, BMN, EPI_WGRAD_BIAS, false, W>(p, st);
  }
  return cudaErrorInvalidValue;
}

template <int BN, bool AMN, bool BMN>
cudaError_t launch_ek(TcParams& p, cudaStream_t st) {
  if constexpr (BN >= 128)
    if (p.wpq == 4) return launch_ek_w<BN, AMN, BMN, 4>(p, st);
  return launch_ek_w<BN, AMN, BMN, 2>(p, st);
}

template <bool AMN, bool BMN>
cudaError_t launch_bn(TcParams& p, int bn, cudaStream_t st) {
  switch (bn) {
    case 16: if constexpr (!BMN) return launch_ek<16, AMN, BMN>(p, st); break;
    case 32: if constexpr (!BMN) return launch_ek<32, AMN, BMN>(p, st); break;
    case 64: return launch_ek<64, AMN, BMN>(p, st);
    case 128: return launch_ek<128, AMN, BMN>(p, st);
    default: return launch_ek<256, AMN, BMN>(p, st);
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
  if (on) {
    static std::vector<int> neg(TRACE_CTAS * TRACE_TILES, -1);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_tile, neg.data(), neg.size() * sizeof(int));
    static std::vector<unsigned long long> z2(TRACE_CTAS * 2, 0ull);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_cta, z2.data(), z2.size() * sizeof(unsigned long long));
  }
  if (e != cudaSuccess || !out) return e;
  // n > stamps: the tile indices follow (as 64-bit values)
  const int ns = TRACE_CTAS * TRACE_TILES * 4;
  e = cudaMemcpyFromSymbol(out, g_trace, std::min(n, ns) * sizeof(unsigned long long));
  if (e != cudaSuccess || n <= ns) return e;
  std::vector<int> ti(TRACE_CTAS * TRACE_TILES);
  e = cudaMemcpyFromSymbol(ti.data(), g_trace_tile, ti.size() * sizeof(int));
  for (int i = 0; i < (int)ti.size() && ns + i < n; ++i) out[ns + i] = (unsigned long long)(long long)ti[i];
  const int nc = ns + (int)ti.size();
  if (e != cudaSuccess || n <= nc) return e;
  return cudaMemcpyFromSymbol(out + nc, g_trace_cta, std::min(n - nc, TRACE_CTAS * 2) * sizeof(unsigned long long));
}

bool tc_gemm_supported(const GemmArgs& a) {
  if (a.N < 1 || a.K < 1 || a.n_groups < 1 || a.n_groups > MAX_GROUPS) return false;
  if (a.splits > 1 && (a.k_per_split % BK)) return false;
  for (int i = 0; i < a.n_groups; ++i)
    if (a.g[i].splits > 0 && (a.g[i].splits < 1 || (a.g[i].splits > 1 && (a.g[i].k_per_split % BK)) ||
                              (int64_t)a.g[i].splits * a.g[i].k_per_split < a.K))
      return false;
  const int bn = pick_bn(a.N, a.b_mn);
  const bool ek = a.a_mn ? (a.b_mn && ek_ok<true, true>(a.epi, bn))
                         : (a.b_mn ? ek_ok<false, true>(a.epi, bn) : ek_ok<false, false>(a.epi, bn));
  if (!ek) return false;  // layout / epilogue combination not instantiated
  for (int i = 0; i < a.n_groups; ++i) {
    const GemmGroup& g = a.g[i];
    if ((g.lda & 7) || (g.ldb & 7)) return false;
    if ((reinterpret_cast<uintptr_t>(g.A) & 15) || (reinterpret_cast<uintptr_t>(g.B) & 15)) return false;
    if (g.dot_out && g.N > bn && g.dot_pstride == 0) return false;  // wide rows need per-tile partials
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
  const bool f32out = a.epi == EPI_F32 || a.epi == EPI_BIAS_F32 || a.epi == EPI_WGRAD_BIAS;
  p.out_bytes = f32out ? 4 : 2;
  p.tma_out = (a.epi == EPI_BIAS_RELU || a.epi == EPI_MASK_BITS || f32out) ? 1 : 0;
  for (int i = 0; i < a.n_groups && p.tma_out; ++i) {
    const GemmGroup& g = a.g[i];
    if (g.M < 1 || g.N < 1) continue;
    if (!g.C || !make_map_out(&p.tc[i], g.C, p.out_bytes, g.N, g.M, group_splits(g, a.splits), g.ldc, g.split_stride)) p.tma_out = 0;
  }
  const int bn = pick_bn(a.N, a.b_mn);
  p.pair = want_pair(a, bn) ? 1 : 0;
  {  // 4 epilogue warps per lane quarter under two tiles per SM, else 2 (SPZ_TC_WPQ=2 / 4 forces; diagnostics)
    int64_t tiles = 0;
    for (int i = 0; i < a.n_groups; ++i) tiles += cdiv(a.g[i].M, BM) * cdiv(a.g[i].N, bn) * group_splits(a.g[i], a.splits);
    // (4 warps only at BN >= 128: a warp's column slice must fill its 64-byte store blocks, EpiShape)
    p.wpq = tiles < 2 * num_sms() && bn >= 128 ? 4 : 2;
    if (const char* w = std::getenv("SPZ_TC_WPQ")) p.wpq = std::atoi(w) == 4 && bn >= 128 ? 4 : 2;
  }
  int maxM = 0;
  for (int i = 0; i < a.n_groups; ++i) {
    const GemmGroup& g = a.g[i];
    maxM = g.M > maxM ? g.M : maxM;
    if (g.M < 1 || g.N < 1) continue;
    bool ok;
    if (!a.a_mn) ok = make_map(&p.ta[i], g.A, a.K, g.M, g.lda, BK, BM);      // A [M x K]
    else ok = make_map(&p.ta[i], g.A, g.M, a.K, g.lda, 64, BK);             // A stored [K x M]
    if (ok) {
      if (!a.b_mn) ok = make_map(&p.tb[i], g.B, a.K, g.N, g.ldb, BK, p.pair ? bn / 2 : bn);  // B [N x K] (pair: half)
      else ok = make_map(&p.tb[i], g.B, g.N, a.K, g.ldb, 64, BK);           // B stored [K x N]
    }
    if (!ok) return cudaErrorInvalidValue;
  }
  if (maxM == 0) return cudaSuccess;
  if (!a.a_mn && !a.b_mn) return launch_bn<false, false>(p, bn, st);
  if (!a.a_mn && a.b_mn) return launch_bn<false, true>(p, bn, st);
  return launch_bn<true, true>(p, bn, st);
}

}  // namespace spz
