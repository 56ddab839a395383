// gemm_simt.cu -- fp32 SIMT GEMM with the shared epilogues (FP32 precision path).
//
// 64x64 output tile per 256-thread CTA, 4x4 micro-tile per thread, K staged in
// 16-deep shared-memory slabs.  Exact fp32 FMA accumulation in a fixed order, so
// the FP32 path is bit-reproducible run to run.
#include "gemm.cuh"

namespace spz {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <typename T>
__global__ void __launch_bounds__(NT) gemm_simt_kernel(const __grid_constant__ GemmArgs a) {
  pdl_wait();
  pdl_launch();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int gz = blockIdx.z;
  const int grp = gz / a.splits, split = gz % a.splits;
  const GemmGroup& g = a.g[grp];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= g.M || n0 >= g.N) return;
  const int k_begin = split * a.k_per_split;
  const int k_end = min(a.K, k_begin + a.k_per_split);
  const T* A = static_cast<const T*>(g.A);
  const T* B = static_cast<const T*>(g.B);
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  float acc[4][4] = {};
  for (int k0 = k_begin; k0 < k_end; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * NT;  // 0..1023
      int mm, kk;
      if (a.a_mn) { kk = e / BM; mm = e % BM; } else { mm = e / BK; kk = e % BK; }
      const int gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < g.M && gk < k_end) v = to_f(a.a_mn ? A[(int64_t)gk * g.lda + gm] : A[(int64_t)gm * g.lda + gk]);
      As[kk][mm] = v;
      int nn;
      if (a.b_mn) { kk = e / BN; nn = e % BN; } else { nn = e / BK; kk = e % BK; }
      const int gn = n0 + nn;
      const int gk2 = k0 + kk;
      float w = 0.f;
      if (gn < g.N && gk2 < k_end) w = to_f(a.b_mn ? B[(int64_t)gk2 * g.ldb + gn] : B[(int64_t)gn * g.ldb + gk2]);
      Bs[kk][nn] = w;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < g.N) epi_store<T>(a, g, split, m, n, acc[i][j]);
    }
  }
}
}  // namespace

template <typename T>
cudaError_t gemm_simt(const GemmArgs& a, cudaStream_t st) {
  int maxM = 0;
  for (int i = 0; i < a.n_groups; ++i) maxM = a.g[i].M > maxM ? a.g[i].M : maxM;
  if (maxM == 0 || a.N == 0) return cudaSuccess;
  dim3 grid((unsigned)cdiv(a.N, BN), (unsigned)cdiv(maxM, BM), (unsigned)(a.n_groups * a.splits));
  return launch_pdl(gemm_simt_kernel<T>, grid, dim3(NT), 0, st, a);
}

template cudaError_t gemm_simt<float>(const GemmArgs&, cudaStream_t);
template cudaError_t gemm_simt<__nv_bfloat16>(const GemmArgs&, cudaStream_t);

}  // namespace spz
