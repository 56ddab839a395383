// tc_gemm_tf32.cu -- FP32-precision GEMM on the 5th-generation tensor cores as 3xTF32 (SURVEY.md §8(a)
// a3: "GEMM bf16 or 3xTF32 with fp32 accumulate"; §8(c) reading 15), behind the GemmArgs contract.
//
// Every fp32 operand x is split into two tf32 values, hi = rna_tf32(x) and lo = rna_tf32(x - hi), and
//     D = A_hi B_hi + A_hi B_lo + A_lo B_hi          (lo * lo dropped, ~2^-22 relative)
// Both parts are exact tf32 values, so the result does not depend on whether the tensor core truncates
// or rounds its fp32 inputs.  The tensor core's fp32 accumulation is biased toward zero (measured:
// tools/tf32_accuracy.py, mean error -2.4e-9 K relative, i.e. 1.6e-4 at K = 65536 vs 3e-9 for fp32 FMA),
// so the contraction is cut into KC-deep chunks: each chunk starts a fresh TMEM accumulator, and the
// epilogue adds the chunk sums into fp32 registers with round-to-nearest adds.
//
// One CTA computes 128 x BN output tiles (persistent over the tiles of every group) from 32-deep K
// slabs (128-byte fp32 rows, 128 B swizzle) staged by TMA:
//   warp 0      TMA producer (one lane): 3-stage ring (full / empty mbarriers)
//   warp 1      TMEM allocator + MMA issuer: per 8-deep k step three tcgen05.mma.kind::tf32
//   warps 2..5  splitters: stage -> (hi in place, lo in the stage's twin), then `conv` mbarrier
//   warps 6..13 epilogue: TMEM lane quarter (warp % 4) x column half; chunk sums -> registers, then the
//               fp32 epilogue kinds (bias + ReLU, bias, ReLU-mask from the stored activation, split-K partials)
// The chunk accumulator is double-buffered in TMEM, so the next chunk's MMAs overlap the drain.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "tc_gemm.cuh"
#include "tc_common.cuh"

namespace spz {

namespace {

constexpr int TBM = 128, TBK = 32, TSTAGES = 3;
constexpr int KC_BLOCKS = 2;  // k-blocks per TMEM accumulation chunk (KC = 64)
constexpr int T_NTHREADS = 448;
constexpr int A32_BYTES = TBM * TBK * 4;  // 16 KB

struct Tf32Params {
  GemmArgs a;
  int stages, total_tiles;
  int tile0[MAX_GROUPS + 1];
  int mtiles[MAX_GROUPS], ntiles[MAX_GROUPS];
  CUtensorMap ta[MAX_GROUPS];
  CUtensorMap tb[MAX_GROUPS];
};

struct Tile32 {
  int grp, m0, n0, split;
};
__device__ __forceinline__ Tile32 decode32(const Tf32Params& p, int t, int bn) {
  int g = 0;
  while (g + 1 < p.a.n_groups && t >= p.tile0[g + 1]) ++g;
  const int r = t - p.tile0[g];
  const int mt = r % p.mtiles[g];
  const int rest = r / p.mtiles[g];
  const int nt = rest % p.ntiles[g];
  return {g, mt * TBM, nt * bn, rest / p.ntiles[g]};
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}
// MN-major tf32 operands take only the SWIZZLE_128B_BASE32B smem layout (descriptor layout type 1; TMA
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B: 32-byte units of a 128-byte row XOR-ed with row % 4): 32-element
// (128 B) MN chunks of TBK K-rows, chunks 4 KB apart (LBO); 4-row K groups 512 B apart (SBO); one 8-deep
// k step = 8 rows = +1024 B.  K-major: plain SW128, 128 B rows, 8-row atoms 1024 B apart, +32 B per step.
__device__ __forceinline__ uint64_t desc_mn32(uint32_t base, int kk) {
  const uint64_t d = umma_desc(base + kk * 1024, 4096, 512);
  return (d & ~((uint64_t)7 << 61)) | ((uint64_t)1 << 61);
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t d;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(d) : "f"(x));
  return __uint_as_float(d);
}

template <int BN, bool AMN, bool BMN, int EK>
__global__ void __launch_bounds__(T_NTHREADS, 1) tc_gemm_tf32_kernel(const __grid_constant__ Tf32Params p) {
  constexpr int B_BYTES = BN * TBK * 4;
  constexpr int HALF = A32_BYTES + B_BYTES;  // hi (in place) or lo copy of one stage
  constexpr int STAGE = 2 * HALF;
  constexpr uint32_t ACC_COLS = BN < 32 ? 32 : BN;
  constexpr uint32_t TMEM_COLS = 2 * ACC_COLS <= 32 ? 32 : 2 * ACC_COLS <= 64 ? 64 : 2 * ACC_COLS <= 128 ? 128 : 256;
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) | ((BMN ? 1u : 0u) << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TBM >> 4) << 24);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NS = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * STAGE);
  uint64_t* conv = full + TSTAGES;
  uint64_t* empty = conv + TSTAGES;
  uint64_t* acc_full = empty + TSTAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

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
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);
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
  pdl_wait();
  pdl_launch();

  auto nkb_of = [&](const Tile32& ti) {
    const int k_begin = ti.split * a.k_per_split;
    const int k_end = min(a.K, k_begin + a.k_per_split);
    return k_end > k_begin ? (k_end - k_begin + TBK - 1) / TBK : 0;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int kg = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const Tile32 ti = decode32(p, t, BN);
        const int nkb = nkb_of(ti);
        for (int kb = 0; kb < nkb; ++kb, ++kg) {
          const int s = kg % NS;
          mbar_wait(&empty[s], (((uint32_t)(kg / NS)) & 1u) ^ 1u);
          uint8_t* sA = smem + s * STAGE;
          uint8_t* sB = sA + A32_BYTES;
          mbar_expect_tx(&full[s], HALF);
          const int k = ti.split * a.k_per_split + kb * TBK;
          if (!AMN) {
            tma_load_2d(sA, &p.ta[ti.grp], &full[s], k, ti.m0);
          } else {
#pragma unroll
            for (int i = 0; i < TBM / 32; ++i) tma_load_2d(sA + i * 4096, &p.ta[ti.grp], &full[s], ti.m0 + 32 * i, k);
          }
          if (!BMN) {
            tma_load_2d(sB, &p.tb[ti.grp], &full[s], k, ti.n0);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 32; ++i) tma_load_2d(sB + i * 4096, &p.tb[ti.grp], &full[s], ti.n0 + 32 * i, k);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      int kg = 0, ci = 0;  // k-blocks and chunks issued by this CTA
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const Tile32 ti = decode32(p, t, BN);
        const int nkb = nkb_of(ti);
        const int nch = nkb > 0 ? (nkb + KC_BLOCKS - 1) / KC_BLOCKS : 1;
        for (int c = 0; c < nch; ++c, ++ci) {
        const int b = ci & 1;
        mbar_wait(&acc_empty[b], (((uint32_t)(ci >> 1)) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)b * ACC_COLS;
        const int kb_end = min(nkb, (c + 1) * KC_BLOCKS);
        for (int kb = c * KC_BLOCKS; kb < kb_end; ++kb, ++kg) {
          const int s = kg % NS;
          mbar_wait(&conv[s], ((uint32_t)(kg / NS)) & 1u);
          tc_fence_after();
          const uint32_t hA = smem_u32(smem + s * STAGE), hB = hA + A32_BYTES;
          const uint32_t lA = hA + HALF, lB = hB + HALF;
#pragma unroll
          for (int kk = 0; kk < TBK / 8; ++kk) {
            const uint64_t ah = AMN ? desc_mn32(hA, kk) : desc_kmajor(hA, kk);
            const uint64_t al = AMN ? desc_mn32(lA, kk) : desc_kmajor(lA, kk);
            const uint64_t bh = BMN ? desc_mn32(hB, kk) : desc_kmajor(hB, kk);
            const uint64_t bl = BMN ? desc_mn32(lB, kk) : desc_kmajor(lB, kk);
            // small cross terms first, then the dominant hi * hi product
            umma_tf32(acc, al, bh, IDESC, (kb != c * KC_BLOCKS || kk != 0) ? 1u : 0u);
            umma_tf32(acc, ah, bl, IDESC, 1u);
            umma_tf32(acc, ah, bh, IDESC, 1u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[b]);  // chunk sum complete (immediately if the split is empty)
        }
      }
    }
  } else if (warp < 6) {
    // ---------------- splitters: x -> (hi in place, lo in the twin half); every stage the MMA consumes
    const int tid = threadIdx.x - 64;
    int kg = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      const Tile32 ti = decode32(p, t, BN);
      const int nkb = nkb_of(ti);
      for (int kb = 0; kb < nkb; ++kb, ++kg) {
        const int s = kg % NS;
        mbar_wait(&full[s], ((uint32_t)(kg / NS)) & 1u);
        float4* hv = reinterpret_cast<float4*>(smem + s * STAGE);
        float4* lv = reinterpret_cast<float4*>(smem + s * STAGE + HALF);
#pragma unroll 4
        for (int i = tid; i < HALF / 16; i += 128) {
          const float4 x = hv[i];
          const float4 h = make_float4(rna_tf32(x.x), rna_tf32(x.y), rna_tf32(x.z), rna_tf32(x.w));
          hv[i] = h;
          lv[i] = make_float4(rna_tf32(x.x - h.x), rna_tf32(x.y - h.y), rna_tf32(x.z - h.z), rna_tf32(x.w - h.w));
        }
        fence_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
    }
  } else {
    // ---------------- epilogue: 32 rows (TMEM lane quarter warp % 4) x CW columns (half hh of the tile)
    constexpr int CW = BN / 2 < 16 ? 16 : BN / 2;
    const int e = warp - 6, q = warp & 3, hh = e >> 2;
    const bool active = hh * CW < BN;
    const int r = q * 32 + lane;
    int ci = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      const Tile32 ti = decode32(p, t, BN);
      const GemmGroup& g = a.g[ti.grp];
      const int nkb = nkb_of(ti);
      const int nch = nkb > 0 ? (nkb + KC_BLOCKS - 1) / KC_BLOCKS : 1;
      float accr[CW];
#pragma unroll
      for (int j = 0; j < CW; ++j) accr[j] = 0.f;
      for (int c = 0; c < nch; ++c, ++ci) {
        const int b = ci & 1;
        mbar_wait(&acc_full[b], ((uint32_t)(ci >> 1)) & 1u);
        tc_fence_after();
        const uint32_t trow = tmem + (uint32_t)b * ACC_COLS + (uint32_t)(hh * CW) + ((uint32_t)(q * 32) << 16);
        if (active && nkb > 0) {
#pragma unroll
          for (int cc = 0; cc < CW / 16; ++cc) {
            float v[16];
            tmem_ld16(trow + cc * 16, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) accr[cc * 16 + j] += v[j];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[b]);
      }
      const int m = ti.m0 + r;
      if (!active || m >= g.M) continue;
#pragma unroll
      for (int cc = 0; cc < CW / 16; ++cc) {
        const int n = ti.n0 + hh * CW + cc * 16;
        if (n >= g.N) continue;
        float v[16];
        const int64_t off = (int64_t)m * g.ldc + n;
        float* C = static_cast<float*>(g.C) + off;
        if constexpr (EK == EPI_F32) C += (int64_t)ti.split * g.split_stride;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          v[j] = accr[cc * 16 + j];
          if constexpr (EK == EPI_BIAS_RELU) {
            v[j] = n + j < g.N ? fmaxf(v[j] + __ldg(g.bias + n + j), 0.f) : 0.f;
          } else if constexpr (EK == EPI_BIAS_F32) {
            v[j] = n + j < g.N ? v[j] + __ldg(g.bias + n + j) : 0.f;
          } else if constexpr (EK == EPI_MASK) {
            const float* aux = static_cast<const float*>(g.aux) + (int64_t)m * g.ldaux + n;
            v[j] = (n + j < g.N && __ldg(aux + j) > 0.f) ? v[j] : 0.f;
          }
        }
        if (n + 16 <= g.N && (reinterpret_cast<uintptr_t>(C) & 15) == 0) {
#pragma unroll
          for (int j = 0; j < 4; ++j) reinterpret_cast<float4*>(C)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        } else {
          for (int j = 0; j < 16 && n + j < g.N; ++j) C[j] = v[j];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

constexpr int t_extras() { return 1024 + 1024; }

template <int BN, bool AMN, bool BMN, int EK>
cudaError_t launch32(Tf32Params& p, cudaStream_t st) {
  constexpr int STAGE = 2 * (A32_BYTES + BN * TBK * 4);
  constexpr int MAX_ST = std::min(TSTAGES, (227 * 1024 - t_extras()) / STAGE);
  static_assert(MAX_ST >= 2, "shared memory budget");
  auto kern = tc_gemm_tf32_kernel<BN, AMN, BMN, EK>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once(attr, kern, MAX_ST * STAGE + t_extras()); e != cudaSuccess) return e;
  int T = 0;
  for (int i = 0; i < p.a.n_groups; ++i) {
    const GemmGroup& g = p.a.g[i];
    p.tile0[i] = T;
    p.mtiles[i] = g.M > 0 && g.N > 0 ? (int)cdiv(g.M, TBM) : 0;
    p.ntiles[i] = g.M > 0 && g.N > 0 ? (int)cdiv(g.N, BN) : 1;
    if (p.mtiles[i] == 0) p.mtiles[i] = 1, p.ntiles[i] = 0;
    T += p.mtiles[i] * p.ntiles[i] * p.a.splits;
  }
  p.tile0[p.a.n_groups] = T;
  p.total_tiles = T;
  if (T == 0) return cudaSuccess;
  const int kspan = p.a.splits > 1 ? p.a.k_per_split : p.a.K;
  p.stages = std::max(2, std::min<int>(MAX_ST, (int)cdiv(kspan, TBK)));
  const int grid = std::min(T, num_sms());
  return launch_pdl(kern, dim3(grid), dim3(T_NTHREADS), (size_t)(p.stages * STAGE + t_extras()), st, p);
}

template <int BN, bool AMN, bool BMN>
cudaError_t launch32_ek(Tf32Params& p, cudaStream_t st) {
  if constexpr (!AMN && !BMN) {
    switch (p.a.epi) {
      case EPI_BIAS_RELU: return launch32<BN, AMN, BMN, EPI_BIAS_RELU>(p, st);
      case EPI_BIAS_F32: return launch32<BN, AMN, BMN, EPI_BIAS_F32>(p, st);
      case EPI_F32: return launch32<BN, AMN, BMN, EPI_F32>(p, st);
      default: break;
    }
  } else if constexpr (!AMN && BMN) {
    if (p.a.epi == EPI_MASK) return launch32<BN, AMN, BMN, EPI_MASK>(p, st);
    if (p.a.epi == EPI_F32) return launch32<BN, AMN, BMN, EPI_F32>(p, st);
  } else {
    if (p.a.epi == EPI_F32) return launch32<BN, AMN, BMN, EPI_F32>(p, st);
  }
  return cudaErrorInvalidValue;
}

template <bool AMN, bool BMN>
cudaError_t launch32_bn(Tf32Params& p, int bn, cudaStream_t st) {
  switch (bn) {
    case 16: if constexpr (!BMN) return launch32_ek<16, AMN, BMN>(p, st); break;
    case 32: return launch32_ek<32, AMN, BMN>(p, st);
    case 64: return launch32_ek<64, AMN, BMN>(p, st);
    default: return launch32_ek<128, AMN, BMN>(p, st);
  }
  return cudaErrorInvalidValue;
}

int pick_bn32(int N, bool bmn) {
  if (N > 64) return 128;
  if (N > 32) return 64;
  if (N > 16 || bmn) return 32;  // MN-major B loads 32-element chunks
  return 16;
}

template <bool AMN, bool BMN>
constexpr bool ek32_ok(int epi) {
  if (!AMN && !BMN) return epi == EPI_BIAS_RELU || epi == EPI_BIAS_F32 || epi == EPI_F32;
  if (!AMN && BMN) return epi == EPI_MASK || epi == EPI_F32;
  if (AMN && BMN) return epi == EPI_F32;
  return false;
}

// 2-D fp32 tensor map, 128-byte rows (box inner = 32 elements): K-major operands SW128, MN-major ones
// SW128 with 32-byte atoms (the only MN-major tf32 layout the MMA reads)
bool make_map32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                uint32_t box_outer, bool mn_major) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

bool tc_gemm_tf32_supported(const GemmArgs& a) {
  if (a.N < 1 || a.K < 1 || a.n_groups < 1 || a.n_groups > MAX_GROUPS) return false;
  if (a.splits > 1 && (a.k_per_split % TBK)) return false;
  for (int i = 0; i < a.n_groups; ++i)
    if (a.g[i].splits > 0) return false;  // per-group split-K: bf16 kernel only
  if (a.a_mn && !a.b_mn) return false;
  const bool ek = a.a_mn ? ek32_ok<true, true>(a.epi) : (a.b_mn ? ek32_ok<false, true>(a.epi) : ek32_ok<false, false>(a.epi));
  if (!ek) return false;
  for (int i = 0; i < a.n_groups; ++i) {
    const GemmGroup& g = a.g[i];
    if ((g.lda & 3) || (g.ldb & 3)) return false;  // 16-byte TMA row pitch
    if ((reinterpret_cast<uintptr_t>(g.A) & 15) || (reinterpret_cast<uintptr_t>(g.B) & 15)) return false;
    if (g.dot_out || g.mask_out || g.colsum_out) return false;  // fused bf16-path extras
  }
  return get_encode();
}

cudaError_t tc_gemm_tf32x3(const GemmArgs& a, cudaStream_t st) {
  Tf32Params p;
  std::memset(&p, 0, sizeof(p));
  p.a = a;
  const int bn = pick_bn32(a.N, a.b_mn);
  int maxM = 0;
  for (int i = 0; i < a.n_groups; ++i) {
    const GemmGroup& g = a.g[i];
    maxM = g.M > maxM ? g.M : maxM;
    if (g.M < 1 || g.N < 1) continue;
    bool ok;
    if (!a.a_mn) ok = make_map32(&p.ta[i], g.A, a.K, g.M, g.lda, TBK, TBM, false);  // A [M x K]
    else ok = make_map32(&p.ta[i], g.A, g.M, a.K, g.lda, 32, TBK, true);           // A stored [K x M]
    if (ok) {
      if (!a.b_mn) ok = make_map32(&p.tb[i], g.B, a.K, g.N, g.ldb, TBK, bn, false);  // B [N x K]
      else ok = make_map32(&p.tb[i], g.B, g.N, a.K, g.ldb, 32, TBK, true);          // B stored [K x N]
    }
    if (!ok) return cudaErrorInvalidValue;
  }
  if (maxM == 0) return cudaSuccess;
  if (!a.a_mn && !a.b_mn) return launch32_bn<false, false>(p, bn, st);
  if (!a.a_mn && a.b_mn) return launch32_bn<false, true>(p, bn, st);
  return launch32_bn<true, true>(p, bn, st);
}

}  // namespace spz
