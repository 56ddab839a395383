"""Diagnostics: error of the 3xTF32 tcgen05 GEMM and the fp32 SIMT GEMM against float64, for growing K
(mean and max of |C - C64| / sum|a||b| and the signed mean, which exposes a biased accumulator)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2312_06126_b200 import spz

for K in (256, 1024, 8192, 65536):
    M, N = 256, 256
    g = torch.Generator(device="cuda").manual_seed(K)
    A = torch.randn(M, K, generator=g, device="cuda") + 0.5  # positive mean: long same-sign sums
    B = torch.randn(N, K, generator=g, device="cuda") + 0.5
    ref = A.double() @ B.double().t()
    sc = A.double().abs() @ B.double().abs().t()
    for tc in (True, False):
        C = torch.empty(M, N, device="cuda")
        spz.spz_diag_gemm_f32(M, N, K, A, K, 0, B, K, 0, C, N, tensor_cores=tc)
        e = (C.double() - ref) / sc
        print(f"K={K:6d} {'3xtf32' if tc else 'simt  '} max {e.abs().max().item():.2e} mean|e| {e.abs().mean().item():.2e} "
              f"mean e {e.mean().item():+.2e}  (2^-24 = 6.0e-08)")
