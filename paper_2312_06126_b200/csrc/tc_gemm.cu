// tc_gemm.cu -- placeholder until the tcgen05 kernel lands: every problem goes to SIMT.
#include "tc_gemm.cuh"

namespace spz {
bool tc_gemm_supported(const GemmArgs&) { return false; }
cudaError_t tc_gemm_bf16(const GemmArgs&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace spz
