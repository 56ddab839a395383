// api.cu -- error reporting, device checks and small C-ABI entry points.
#include <cstring>
#include <string>

#include "internal.h"
#include "tc_gemm.cuh"
#include <cstdlib>
#include "tc_mlp.cuh"

namespace spz {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

spz_status fail(spz_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

spz_status check_device(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(SPZ_ECUDA, std::string("no CUDA device available (") + cudaGetErrorString(e) + "); spz has no CPU fallback");
  }
  if (device < 0 || device >= n) return fail(SPZ_EINVAL, "device ordinal " + std::to_string(device) + " out of range");
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return fail(SPZ_ECUDA, "cudaGetDeviceProperties failed");
  if (p.major != 10 || p.minor != 0)
    return fail(SPZ_ECUDA, "device " + std::to_string(device) + " is sm_" + std::to_string(p.major) + std::to_string(p.minor) +
                               "; this library is built for sm_100a only");
  return SPZ_OK;
}

}  // namespace spz

extern "C" {

const char* spz_last_error(void) { return spz::g_last_error.c_str(); }

const char* spz_version(void) { return "spz 0.1 (sm_100a)"; }

spz_status spz_diag_gemm_bf16(int32_t device, int32_t tensor_cores, int64_t M, int64_t N, int64_t K, const void* A,
                              int64_t lda, int32_t a_mn, const void* B, int64_t ldb, int32_t b_mn, float* C, int64_t ldc,
                              int32_t splits, int64_t k_per_split) {
  spz_status st = spz::check_device(device);
  if (st != SPZ_OK) return st;
  if (M < 1 || N < 1 || K < 1 || !A || !B || !C || splits < 1) return spz::fail(SPZ_EINVAL, "spz_diag_gemm_bf16: bad argument");
  spz::DeviceGuard dg(device);
  spz::GemmArgs a{};
  a.N = (int)N;
  a.K = (int)K;
  a.a_mn = a_mn;
  a.b_mn = b_mn;
  a.epi = spz::EPI_F32;
  a.splits = splits;
  a.k_per_split = splits > 1 ? (int)k_per_split : (int)K;
  a.n_groups = 1;
  a.g[0].lda = (int)lda;
  a.g[0].ldb = (int)ldb;
  a.g[0].ldc = (int)ldc;
  a.g[0].N = (int)N;
  a.g[0].split_stride = M * ldc;
  a.g[0].A = A;
  a.g[0].B = B;
  a.g[0].C = C;
  a.g[0].M = (int)M;
  // SPZ_DIAG_GEMM_DYN=<n_pre_groups>: the dynamic tile schedule (tcgen05 only); its counters must be back at 0
  static unsigned* sched = nullptr;
  const char* dyn = std::getenv("SPZ_DIAG_GEMM_DYN");
  if (dyn && tensor_cores) {
    if (!sched && (cudaMalloc(&sched, 2 * sizeof(unsigned)) != cudaSuccess || cudaMemset(sched, 0, 2 * sizeof(unsigned)) != cudaSuccess))
      return spz::fail(SPZ_ECUDA, "spz_diag_gemm_bf16: schedule counters");
    a.sched = sched;
    a.n_pre_groups = std::atoi(dyn);
  }
  cudaError_t e;
  if (tensor_cores) {
    if (!spz::tc_gemm_supported(a)) return spz::fail(SPZ_EUNSUPPORTED, "spz_diag_gemm_bf16: problem not supported by the tcgen05 kernel");
    e = spz::tc_gemm_bf16(a, 0);
  } else {
    e = spz::gemm_simt<__nv_bfloat16>(a, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return spz::fail(SPZ_ECUDA, std::string("spz_diag_gemm_bf16: ") + cudaGetErrorString(e));
  if (a.sched) {
    unsigned h[2] = {1u, 1u};
    if (cudaMemcpy(h, a.sched, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess || h[0] || h[1])
      return spz::fail(SPZ_ESTATE, "spz_diag_gemm_bf16: dynamic schedule counters not reset");
  }
  return SPZ_OK;
}

spz_status spz_diag_gemm_f32(int32_t device, int32_t tensor_cores, int64_t M, int64_t N, int64_t K, const float* A,
                             int64_t lda, int32_t a_mn, const float* B, int64_t ldb, int32_t b_mn, float* C, int64_t ldc,
                             int32_t splits, int64_t k_per_split) {
  spz_status st = spz::check_device(device);
  if (st != SPZ_OK) return st;
  if (M < 1 || N < 1 || K < 1 || !A || !B || !C || splits < 1) return spz::fail(SPZ_EINVAL, "spz_diag_gemm_f32: bad argument");
  spz::DeviceGuard dg(device);
  spz::GemmArgs a{};
  a.N = (int)N;
  a.K = (int)K;
  a.a_mn = a_mn;
  a.b_mn = b_mn;
  a.epi = spz::EPI_F32;
  a.splits = splits;
  a.k_per_split = splits > 1 ? (int)k_per_split : (int)K;
  a.n_groups = 1;
  a.g[0].lda = (int)lda;
  a.g[0].ldb = (int)ldb;
  a.g[0].ldc = (int)ldc;
  a.g[0].N = (int)N;
  a.g[0].split_stride = M * ldc;
  a.g[0].A = A;
  a.g[0].B = B;
  a.g[0].C = C;
  a.g[0].M = (int)M;
  cudaError_t e;
  if (tensor_cores) {
    if (!spz::tc_gemm_tf32_supported(a)) return spz::fail(SPZ_EUNSUPPORTED, "spz_diag_gemm_f32: problem not supported by the 3xTF32 kernel");
    e = spz::tc_gemm_tf32x3(a, 0);
  } else {
    e = spz::gemm_simt<float>(a, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return spz::fail(SPZ_ECUDA, std::string("spz_diag_gemm_f32: ") + cudaGetErrorString(e));
  return SPZ_OK;
}

spz_status spz_diag_tc_trace(int32_t device, int32_t on, uint64_t* host_out, int32_t n) {
  spz_status st = spz::check_device(device);
  if (st != SPZ_OK) return st;
  spz::DeviceGuard dg(device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess)
    e = on >= 100 ? spz::mlp_trace(on - 100, reinterpret_cast<unsigned long long*>(host_out), n)
                  : spz::tc_trace(on, reinterpret_cast<unsigned long long*>(host_out), n);
  if (e != cudaSuccess) return spz::fail(SPZ_ECUDA, std::string("spz_diag_tc_trace: ") + cudaGetErrorString(e));
  return SPZ_OK;
}

}  // extern "C"
