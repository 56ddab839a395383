// tc_gemm.cuh -- tcgen05 / TMEM / TMA bf16 GEMM (sm_100a) behind the GemmArgs contract.
#pragma once

#include "gemm.cuh"

namespace spz {

// True if the tensor-core kernel handles this problem (layouts, alignment, sizes).
bool tc_gemm_supported(const GemmArgs& a);
// True if the tcgen05 path can run at all (driver entry point for tensor maps resolved).
bool tc_gemm_available();
// Diagnostics: enable/disable per-tile timestamps and copy them out (see tc_gemm.cu).
cudaError_t tc_trace(int on, unsigned long long* out, int n);
// Launch it (bf16 operands, fp32 accumulation in TMEM, shared epilogues).
cudaError_t tc_gemm_bf16(const GemmArgs& a, cudaStream_t st);
// FP32 precision on the tensor cores: 3xTF32 (tc_gemm_tf32.cu); fp32 operands, fp32 epilogue kinds.
bool tc_gemm_tf32_supported(const GemmArgs& a);
cudaError_t tc_gemm_tf32x3(const GemmArgs& a, cudaStream_t st);

}  // namespace spz
