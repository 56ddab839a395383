// gemm.cuh -- the GEMM contract used by every dense layer of the update.
//
// For each group g:  C[m, n] = epi( sum_k A(m, k) * B(n, k) ),  m < g.M, n < g.N, k < K.
//   A K-major : A(m,k) = A[m * lda + k]    (activations, row = batch row)
//   A MN-major: A(m,k) = A[k * lda + m]    (wgrad: dZ stored [batch x out])
//   B K-major : B(n,k) = B[n * ldb + k]    (forward: W stored [out x in])
//   B MN-major: B(n,k) = B[k * ldb + n]    (dgrad: W stored [out x in], contraction over out;
//                                            wgrad: activations stored [batch x in])
// Split-K (wgrad, contraction over the batch) writes split s's partial sum to
// C + s * split_stride; the fused Adam kernel sums splits in a fixed order, so the
// result is deterministic (reading #16).
// Up to MAX_GROUPS groups per launch (twin critics, online + target critics, all wgrads of a
// network) share K, operand majorness and the epilogue kind; pointers, M, N and row
// pitches are per group.  The grid covers the largest group; other CTAs exit early.
#pragma once

#include "heads.cuh"

namespace spz {

enum EpiKind : int {
  EPI_BIAS_RELU = 0,  // C (T) = relu(acc + bias[n]); optional fused row dot -> dot_out  -- hidden layer forward
  EPI_BIAS_F32 = 1,   // C (f32) = acc + bias[n]                                           -- linear head forward
  EPI_MASK = 2,       // C (T) = acc * (aux[m, n] > 0)                                     -- dgrad through ReLU
  EPI_F32 = 3,        // C (f32) = acc                                                     -- wgrad partials / input dgrad
  EPI_SAC_HEAD = 4,   // acc + bias -> squashed-Gaussian head (heads.cuh), nothing stored in C
  EPI_TD3_HEAD = 5,   // acc + bias -> tanh head with target smoothing (heads.cuh)
  EPI_MASK_BITS = 6,  // C (T) = acc * bit(aux[m, n / 32], n % 32)                        -- dgrad, packed ReLU mask
  EPI_WGRAD_BIAS = 7, // C (f32) = acc, and colsum_out[split][m] = sum_k A(m, k)               -- wgrad + bias grad
                      // (tcgen05 only: one extra MMA against an all-ones operand on the n-tile 0 tiles)
};

struct GemmGroup {
  const void* A;
  const void* B;
  void* C;
  const float* bias;
  const void* aux;
  const float* dot_w;  // EPI_BIAS_RELU: if set, dot_out[m] = sum_n relu(z[m, n]) dot_w[n] + dot_b[0]
  const float* dot_b;
  float* dot_out;
  int64_t dot_pstride;  // N wider than one tile: tile n0 / BN writes its partial row dot at dot_out + (n0 / BN) *
                        // dot_pstride (tile 0 adds dot_b); the consumer sums the partials in tile order
  uint32_t* mask_out;  // EPI_BIAS_RELU: if set, bit n % 32 of mask_out[m * mask_ld + n / 32] = (z[m, n] > 0)
  int64_t split_stride;  // elements between split partials in C
  float* colsum_out;     // EPI_WGRAD_BIAS: per-split row sums of A (bias gradient partials), may be null
  int64_t colsum_stride; // elements between split partials in colsum_out
  int M, N;
  int lda, ldb, ldc, ldaux;
  int row0;     // head epilogues: local actor-pass row of this group's row 0
  int mask_ld;  // words per row of mask_out
  int splits, k_per_split;  // tcgen05 kernel: this group's split-K (0: the launch's GemmArgs values)
};
__host__ __device__ __forceinline__ int group_splits(const GemmGroup& g, int launch_splits) {
  return g.splits > 0 ? g.splits : launch_splits;
}
__host__ __device__ __forceinline__ int group_kps(const GemmGroup& g, int launch_kps) {
  return g.splits > 0 ? g.k_per_split : launch_kps;
}

constexpr int MAX_GROUPS = 12;

struct GemmArgs {
  int N, K;  // N: max over groups (grid width)
  int a_mn, b_mn;  // 0 = K-major, 1 = MN-major
  int epi;
  int splits;       // split-K count (>= 1)
  int k_per_split;  // contraction rows per split (multiple of the K tile)
  int n_groups;
  GemmGroup g[MAX_GROUPS];
  HeadEpi head;
  // tcgen05 kernel only: dynamic tile schedule.  sched != null: CTAs take tiles in linear order from an atomic
  // counter (sched[0]; sched[1] counts finished CTAs, the last one resets both to 0 for the next launch), and
  // the tiles of groups [0, n_pre_groups) are computed before the grid-dependency wait -- their inputs must not
  // be written by the kernel this one is launched behind (PDL).  CTAs that start while that kernel still holds
  // part of the GPU take the independent tiles first.
  unsigned* sched;
  int n_pre_groups;
};

// Apply the epilogue to one accumulator element (SIMT backend; no fused heads / dots).
template <typename T>
__device__ __forceinline__ void epi_store(const GemmArgs& a, const GemmGroup& g, int split, int m, int n, float acc) {
  const int64_t off = (int64_t)m * g.ldc + n;
  switch (a.epi) {
    case EPI_BIAS_RELU: {
      const float z = acc + g.bias[n];
      static_cast<T*>(g.C)[off] = from_f<T>(z > 0.f ? z : 0.f);
      break;
    }
    case EPI_BIAS_F32:
      static_cast<float*>(g.C)[off] = acc + g.bias[n];
      break;
    case EPI_MASK: {
      const float msk = to_f(static_cast<const T*>(g.aux)[(int64_t)m * g.ldaux + n]);
      static_cast<T*>(g.C)[off] = from_f<T>(msk > 0.f ? acc : 0.f);
      break;
    }
    default:
      static_cast<float*>(g.C)[off + (int64_t)split * g.split_stride] = acc;
      break;
  }
}

// Portable fp32 SIMT GEMM (FP32 precision path).  Defined in gemm_simt.cu.
template <typename T>
cudaError_t gemm_simt(const GemmArgs& a, cudaStream_t st);

}  // namespace spz
