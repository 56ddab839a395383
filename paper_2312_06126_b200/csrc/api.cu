// api.cu -- error reporting, device checks and small C-ABI entry points.
#include <cstring>
#include <string>

#include "internal.h"
#include "tc_gemm.cuh"

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

spz_status spz_nccl_unique_id(uint8_t out[128]) {
  (void)out;
  return spz::fail(SPZ_EUNSUPPORTED, "spz_nccl_unique_id: NCCL support not built yet");
}

}  // extern "C"
