// tc_actor_bwd.cu -- fused actor backward (see tc_actor_bwd.cuh).
//
// Warp roles (one CTA per SM, persistent over 128-row blocks):
//   warp 0      TMA producer: every operand the MMA consumes, in consumption order, through a 4-deep
//               stage ring (S1: dZ1 tile + W0 action-column tile per 64-deep k-block; S2: the head
//               weights; S3: one 64-row slab of W_l per k-block)
//   warp 1      TMEM allocator (512 columns) + MMA issuer; each stage waits for the epilogue that
//               produced its A operand (epi_done)
//   warps 2..9  epilogue: TMEM lane quarter (warp % 4) x column half; E1 on the first warp of each
//               quarter, E2/E3 on all eight
// TMEM: S1 -> columns [0, 64), S2 -> [256, 256 + h), S3 -> [0, h).
#include "tc_actor_bwd.cuh"

#include <algorithm>
#include <cstring>

#include "tc_common.cuh"

namespace spz {

namespace {

constexpr int ABM = 128, ABK = 64, AB_STAGES = 4;
// epilogue warps: AB_WPQ per TMEM lane quarter, each owning H / AB_WPQ columns of the masked gradients
#ifndef SPZ_AB_WPQ
#define SPZ_AB_WPQ 4
#endif
template <int H>
constexpr int ab_wpq() { return H >= 128 ? SPZ_AB_WPQ : 2; }  // (a warp keeps whole 32-column mask words)
template <int H>
constexpr int ab_threads() { return 64 + 4 * ab_wpq<H>() * 32; }
constexpr uint32_t AB_TMEM_COLS = 512, S2_COL = 256;

struct ActorBwdParams {
  int Bl, o, m, h, L, nout, td3, ncrit, ldh, mask_ld, stages, tiles;
  const uint32_t* mask[MLP_MAXL];
  void* dH;
  const float *u, *a, *eps, *sig, *l;
  const float* log_alpha;
  float invB, lo, hi;
  CUtensorMap tdz1[2];               // dZ1 [Bl x h], box 64 x 128
  CUtensorMap tw0[2];                // W0 [h x (o + m)], box 64 x 64 (MN-major B, from column o)
  CUtensorMap twa[MLP_MAXL + 1];     // W_l [out x in], box 64 x 64 (MN-major B)
  CUtensorMap tdza[MLP_MAXL];        // dZ_l [Bl x h] stores, box 64 x 128
};

__device__ __forceinline__ void tma_store_2d_ab(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// bf16 bits of x at column c of row r in a 128-row x 64-column K-major SW128 tile
__device__ __forceinline__ void st_bf16_sw128(uint8_t* tile, int r, int c, float x) {
  const __nv_bfloat16 b = __float2bfloat16_rn(x);
  *reinterpret_cast<__nv_bfloat16*>(tile + r * 128 + ((((c >> 3) ^ (r & 7))) << 4) + (c & 7) * 2) = b;
}

// Masked gradient epilogue of one warp: 32-column blocks [c_lo, c_lo + NB * 32) of row r ->
// acc * mask bit -> bf16 into the hidden buffer H (K-major SW128 slabs of 64 columns).
template <int NB>
__device__ __forceinline__ void mask_epi(uint32_t trow, int c_lo, int r, uint8_t* Hs, const uint32_t (&mw)[NB]) {
#pragma unroll
  for (int ib = 0; ib < NB; ++ib) {
    const int c0 = c_lo + ib * 32;
    float v[2][16];
    tmem_ld32(trow + c0, v[0], v[1]);
    const uint32_t w = mw[ib];
    uint32_t pk[16];
#pragma unroll
    for (int cc = 0; cc < 2; ++cc)
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const int b = cc * 16 + j;
        const float x0 = (w >> b) & 1u ? v[cc][j] : 0.f;
        const float x1 = (w >> (b + 1)) & 1u ? v[cc][j + 1] : 0.f;
        pk[cc * 8 + j / 2] = pack_bf16(x0, x1);
      }
    uint8_t* rowp = Hs + (c0 / 64) * 16384 + r * 128;
    const int u0 = (c0 % 64) / 8;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      *reinterpret_cast<uint4*>(rowp + (((u0 + k) ^ (r & 7)) << 4)) = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
  }
}

template <int H>
__global__ void __launch_bounds__(ab_threads<H>(), 1) tc_actor_bwd_kernel(const __grid_constant__ ActorBwdParams p) {
  constexpr int SLABS = H / 64;
  constexpr int STAGE = (16384 + 8192) > SLABS * 8192 ? (16384 + 8192) : SLABS * 8192;
  constexpr int AB_WPQ = ab_wpq<H>(), AB_EPI_WARPS = 4 * AB_WPQ;
  constexpr int NB = H / AB_WPQ / 32;  // 32-column blocks per epilogue warp
  constexpr uint32_t IDESC1 = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(64 >> 3) << 17) |
                              ((uint32_t)(ABM >> 4) << 24);
  constexpr uint32_t IDESCH = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(H >> 3) << 17) |
                              ((uint32_t)(ABM >> 4) << 24);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NS = p.stages;
  uint8_t* Dh = smem + NS * STAGE;   // dH tile [128 x 64] bf16, SW128
  uint8_t* Hs = Dh + 16384;          // hidden gradient buffer, SLABS x [128 x 64]
  uint64_t* full = reinterpret_cast<uint64_t*>(Hs + SLABS * 16384);
  uint64_t* empty = full + AB_STAGES;
  uint64_t* acc_full = empty + AB_STAGES;
  uint64_t* epi_done = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(epi_done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = p.tiles, L = p.L;
  const int nkh = H / ABK;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < p.ncrit; ++i) {
      tma_prefetch(&p.tdz1[i]);
      tma_prefetch(&p.tw0[i]);
    }
    for (int l = 1; l <= L; ++l) tma_prefetch(&p.twa[l]);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(epi_done, AB_EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(AB_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: S1, S2, S3 operands of every tile in consumption order
      int kg = 0;
      auto stage_begin = [&](uint32_t bytes) -> uint8_t* {
        const int s = kg % NS;
        mbar_wait(&empty[s], ((uint32_t)(kg / NS) & 1u) ^ 1u);
        mbar_expect_tx(&full[s], bytes);
        return smem + s * STAGE;
      };
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int m0 = t * ABM;
        for (int ci = 0; ci < p.ncrit; ++ci)
          for (int kb = 0; kb < nkh; ++kb, ++kg) {
            uint8_t* st = stage_begin(16384 + 8192);
            uint64_t* bar = &full[kg % NS];
            tma_load_2d(st, &p.tdz1[ci], bar, kb * ABK, m0);
            tma_load_2d(st + 16384, &p.tw0[ci], bar, p.o & ~7, kb * ABK);  // 16-byte aligned box start
          }
        {
          uint8_t* st = stage_begin(SLABS * 8192);
          uint64_t* bar = &full[kg % NS];
#pragma unroll
          for (int c = 0; c < SLABS; ++c) tma_load_2d(st + c * 8192, &p.twa[L], bar, c * 64, 0);
          ++kg;
        }
        for (int l = L - 1; l >= 1; --l)
          for (int kb = 0; kb < nkh; ++kb, ++kg) {
            uint8_t* st = stage_begin(SLABS * 8192);
            uint64_t* bar = &full[kg % NS];
#pragma unroll
            for (int c = 0; c < SLABS; ++c) tma_load_2d(st + c * 8192, &p.twa[l], bar, c * 64, kb * ABK);
          }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      int kg = 0, ep = 0;
      bool first = true;
      const uint32_t sDh = smem_u32(Dh), sH = smem_u32(Hs);
      auto wait_epi = [&]() {
        if (!first) {
          mbar_wait(epi_done, (uint32_t)ep & 1u);
          ++ep;
          tc_fence_after();
        }
        first = false;
      };
      auto take = [&]() -> uint32_t {
        const int s = kg % NS;
        mbar_wait(&full[s], (uint32_t)(kg / NS) & 1u);
        tc_fence_after();
        return smem_u32(smem + s * STAGE);
      };
      const int kh = (p.nout + 15) / 16;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        // S1: g_a, both critics into one accumulator
        wait_epi();  // the previous tile's last epilogue has drained TMEM [0, h)
        for (int ci = 0; ci < p.ncrit; ++ci)
          for (int kb = 0; kb < nkh; ++kb, ++kg) {
            const uint32_t sA = take(), sB = sA + 16384;
#pragma unroll
            for (int kk = 0; kk < ABK / 16; ++kk)
              umma_bf16(tmem, desc_kmajor(sA, kk), desc_mnmajor(sB, kk), IDESC1, (ci | kb | kk) != 0 ? 1u : 0u);
            umma_commit(&empty[kg % NS]);
          }
        umma_commit(acc_full);
        // S2: dA_L = dH W_head
        wait_epi();
        {
          const uint32_t sB = take();
          for (int kk = 0; kk < kh; ++kk)
            umma_bf16(tmem + S2_COL, desc_kmajor(sDh, kk), desc_mnmajor(sB, kk), IDESCH, kk != 0 ? 1u : 0u);
          umma_commit(&empty[kg % NS]);
          ++kg;
        }
        umma_commit(acc_full);
        // S3: down the hidden stack
        for (int l = L - 1; l >= 1; --l) {
          wait_epi();
          for (int kb = 0; kb < nkh; ++kb, ++kg) {
            const uint32_t sB = take();
#pragma unroll
            for (int kk = 0; kk < ABK / 16; ++kk)
              umma_bf16(tmem, desc_kmajor(sH + kb * 16384, kk), desc_mnmajor(sB, kk), IDESCH, (kb | kk) != 0 ? 1u : 0u);
            umma_commit(&empty[kg % NS]);
          }
          umma_commit(acc_full);
        }
      }
    }
  } else {
    // ---------------- epilogue
    const int e = warp - 2, q = warp & 3, hh = e >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int ac = 0;
    auto wait_acc = [&]() {
      mbar_wait(acc_full, (uint32_t)ac & 1u);
      ++ac;
      tc_fence_after();
    };
    auto done = [&]() {
      tc_fence_before();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(epi_done);
    };
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      const int m0 = t * ABM;
      const int j = m0 + r;
      const bool live = j < p.Bl;
      // ---- E1: head backward (eq. H) -> dH (HBM) and the S2 A operand (SMEM).  The row's head cache
      //      (first 8 actions) and alpha are loaded before the accumulator wait.
      constexpr int PF = 8;
      float pa[PF], pl[PF], ps[PF], pe[PF];
      float g_lp = 0.f;
      if (hh == 0 && live) {
#pragma unroll
        for (int i = 0; i < PF; ++i) {
          const int64_t ci = (int64_t)(i < p.m ? i : 0) * p.Bl + j;  // action-major [m x Bl]
          pa[i] = __ldg(p.a + ci);
          pl[i] = p.td3 ? 0.f : __ldg(p.l + ci);
          ps[i] = p.td3 ? 0.f : __ldg(p.sig + ci);
          pe[i] = p.td3 ? 0.f : __ldg(p.eps + ci);
        }
        g_lp = p.td3 ? 0.f : expf(__ldg(p.log_alpha)) * p.invB;
      }
      wait_acc();
      if (hh == 0) {
        // the W0 tile starts at column o & ~7: action i is accumulator column (o & 7) + i
        float ga[48];
        const int off = p.o & 7;
        tmem_ld16(tmem + lane_off, *reinterpret_cast<float(*)[16]>(ga));
        if (off + p.m > 16) tmem_ld16(tmem + lane_off + 16, *reinterpret_cast<float(*)[16]>(ga + 16));
        if (off + p.m > 32) tmem_ld16(tmem + lane_off + 32, *reinterpret_cast<float(*)[16]>(ga + 32));
#pragma unroll
        for (int k = 0; k < 8; ++k) *reinterpret_cast<uint4*>(Dh + r * 128 + ((k ^ (r & 7)) << 4)) = make_uint4(0, 0, 0, 0);
        if (live) {
          __nv_bfloat16* dh = static_cast<__nv_bfloat16*>(p.dH) + (int64_t)j * p.ldh;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (i >= p.m) break;
            const int64_t ci = (int64_t)i * p.Bl + j;
            const float a = i < PF ? pa[i < PF ? i : 0] : __ldg(p.a + ci);
            const float gu = ga[off + i] * (1.f - a * a) + 2.f * a * g_lp;
            st_bf16_sw128(Dh, r, i, gu);
            dh[i] = __float2bfloat16_rn(gu);
            if (!p.td3) {
              const float l = i < PF ? pl[i < PF ? i : 0] : __ldg(p.l + ci);
              const float sg = i < PF ? ps[i < PF ? i : 0] : __ldg(p.sig + ci);
              const float ep = i < PF ? pe[i < PF ? i : 0] : __ldg(p.eps + ci);
              const float gl = (l >= p.lo && l <= p.hi) ? (gu * sg * ep - g_lp) : 0.f;
              st_bf16_sw128(Dh, r, p.m + i, gl);
              dh[p.m + i] = __float2bfloat16_rn(gl);
            }
          }
        }
      }
      done();
      // ---- E2 / E3: masked gradients down the stack; E2 reads S2's accumulator
      for (int l = L - 1; l >= 0; --l) {
        // this warp's mask words of the row, loaded before the accumulator wait
        uint32_t mw[NB];
        const uint32_t* mrow = p.mask[l] + (int64_t)(live ? j : 0) * p.mask_ld + hh * (H / AB_WPQ) / 32;
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) mw[ib] = live ? __ldg(mrow + ib) : 0u;
        wait_acc();
        // H must be free of the TMA stores issued from it by the previous epilogue
        if (e == 0 && lane == 0) bulk_wait_read_all();
        named_bar(1, AB_EPI_WARPS * 32);
        const uint32_t trow = tmem + lane_off + (l == L - 1 ? S2_COL : 0u);
        mask_epi<NB>(trow, hh * (H / AB_WPQ), r, Hs, mw);
        tc_fence_before();
        fence_async_smem();
        named_bar(1, AB_EPI_WARPS * 32);
        if (e == 0 && lane == 0) {
#pragma unroll
          for (int sl = 0; sl < SLABS; ++sl) tma_store_2d_ab(&p.tdza[l], Hs + sl * 16384, sl * 64, m0);
          bulk_commit();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(epi_done);
      }
    }
    if (e == 0 && lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(AB_TMEM_COLS) : "memory");
  }
}

// bf16 2-D map [outer x inner] (pitch ld elements), box box_inner x box_outer, 128 B swizzle
bool map_ab(CUtensorMap* m, const void* ptr, int inner, int outer, int ld, int box_inner, int box_outer) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld % 8)) return false;
  return make_map(m, ptr, (uint64_t)inner, (uint64_t)outer, (uint64_t)ld, (uint32_t)box_inner, (uint32_t)box_outer);
}

template <int H>
cudaError_t launch_ab(ActorBwdParams& p, cudaStream_t st) {
  constexpr int SLABS = H / 64;
  constexpr int STAGE = (16384 + 8192) > SLABS * 8192 ? (16384 + 8192) : SLABS * 8192;
  const int fixed = 1024 + 16384 + SLABS * 16384 + 1024;
  const int ns = std::min(AB_STAGES, (227 * 1024 - 8 * 1024 - fixed) / STAGE);
  if (ns < 2) return cudaErrorInvalidValue;
  auto kern = tc_actor_bwd_kernel<H>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once(attr, kern, 227 * 1024 - 8 * 1024); e != cudaSuccess) return e;
  p.stages = ns;
  const int grid = std::min(p.tiles, num_sms());
  return launch_pdl(kern, dim3(grid), dim3(ab_threads<H>()), (size_t)(ns * STAGE + fixed), st, p);
}

}  // namespace

bool tc_actor_bwd_supported(const ActorBwdArgs& a) {
  if (!get_encode()) return false;
  if (a.h != 64 && a.h != 128 && a.h != 256) return false;
  if (a.L < 1 || a.L > MLP_MAXL || a.m < 1 || a.m > 32 || a.nout > 64) return false;
  if (a.ncrit < 1 || a.ncrit > 2 || a.mask_ld * 32 < a.h) return false;
  // the stages of a row block run back to back in one CTA: worth it while every block has its own SM
  // (WLK); larger batches keep the separate launches, whose persistent tiles pipeline
  if (cdiv(a.Bl, ABM) > num_sms()) return false;
  for (int i = 0; i < a.ncrit; ++i)
    if (!a.dZ1[i] || !a.W0c[i] || (a.ldw0c % 8)) return false;
  for (int l = 0; l < a.L; ++l)
    if (!a.mask[l] || !a.dZa[l]) return false;
  return a.dH != nullptr;
}

cudaError_t tc_actor_bwd(const ActorBwdArgs& a, cudaStream_t st) {
  ActorBwdParams p;
  std::memset(&p, 0, sizeof(p));
  p.Bl = a.Bl;
  p.o = a.o;
  p.m = a.m;
  p.h = a.h;
  p.L = a.L;
  p.nout = a.nout;
  p.td3 = a.td3;
  p.ncrit = a.ncrit;
  p.ldh = a.ldh;
  p.mask_ld = a.mask_ld;
  p.dH = a.dH;
  p.u = a.u;
  p.a = a.a;
  p.eps = a.eps;
  p.sig = a.sig;
  p.l = a.l;
  p.log_alpha = a.log_alpha;
  p.invB = a.invB;
  p.lo = a.lo;
  p.hi = a.hi;
  p.tiles = (int)cdiv(a.Bl, ABM);
  if (p.tiles == 0) return cudaSuccess;
  for (int i = 0; i < a.ncrit; ++i) {
    if (!map_ab(&p.tdz1[i], a.dZ1[i], a.h, a.Bl, a.h, 64, ABM)) return cudaErrorInvalidValue;
    // W0 [h x (o + m)]: columns past o + m read as zero
    if (!map_ab(&p.tw0[i], a.W0c[i], a.o + a.m, a.h, a.ldw0c, 64, 64)) return cudaErrorInvalidValue;
  }
  for (int l = 1; l <= a.L; ++l) {
    const int out = l == a.L ? a.nout : a.h;
    if (!map_ab(&p.twa[l], a.Wa[l], a.h, out, a.ldwa[l], 64, 64)) return cudaErrorInvalidValue;
  }
  for (int l = 0; l < a.L; ++l) {
    p.mask[l] = a.mask[l];
    if (!map_ab(&p.tdza[l], a.dZa[l], a.h, a.Bl, a.h, 64, ABM)) return cudaErrorInvalidValue;
  }
  switch (a.h) {
    case 64: return launch_ab<64>(p, st);
    case 128: return launch_ab<128>(p, st);
    default: return launch_ab<256>(p, st);
  }
}

}  // namespace spz
