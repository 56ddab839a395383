"""tcgen05 GEMM kernel unit tests: every operand layout, tile width and split-K path of the
dense layers, against a float32 matmul of the same bf16 operands (test-only torch)."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_06126_b200 import spz  # noqa: E402


def _mk(rows, cols, ld, gen):
    x = torch.zeros(rows, ld, dtype=torch.bfloat16, device="cuda")
    x[:, :cols] = torch.randn(rows, cols, generator=gen, device="cuda").to(torch.bfloat16)
    return x


def _ref(A, a_mn, B, b_mn, M, N, K):
    Af = A.float()
    Bf = B.float()
    Am = Af[:K, :M].t() if a_mn else Af[:M, :K]
    Bm = Bf[:K, :N] if b_mn else Bf[:N, :K].t()
    return Am @ Bm


CASES = [
    # (M, N, K, a_mn, b_mn)  -- forward (K-major x K-major)
    (16384, 256, 256, 0, 0), (1000, 256, 22, 0, 0), (300, 12, 256, 0, 0), (257, 512, 64, 0, 0), (130, 33, 100, 0, 0),
    (128, 1, 256, 0, 0), (4096, 1024, 1024, 0, 0),
    # dgrad (K-major x MN-major)
    (16384, 256, 256, 0, 1), (1000, 28, 256, 0, 1), (777, 256, 12, 0, 1), (200, 300, 96, 0, 1),
    # wgrad (MN-major x MN-major): M = out features, N = in features, K = batch
    (256, 256, 8192, 1, 1), (256, 28, 1000, 1, 1), (12, 256, 1000, 1, 1), (512, 44, 333, 1, 1),
]


@pytest.mark.parametrize("M,N,K,a_mn,b_mn", CASES)
def test_tc_gemm_matches_fp32_matmul(M, N, K, a_mn, b_mn):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    lda = ((M if a_mn else K) + 7) // 8 * 8
    ldb = ((N if b_mn else K) + 7) // 8 * 8
    A = _mk(K, M, lda, g) if a_mn else _mk(M, K, lda, g)
    B = _mk(K, N, ldb, g) if b_mn else _mk(N, K, ldb, g)
    ldc = N
    C = torch.full((M, ldc), float("nan"), device="cuda")
    spz.spz_diag_gemm_bf16(M, N, K, A, lda, a_mn, B, ldb, b_mn, C, ldc)
    ref = _ref(A, a_mn, B, b_mn, M, N, K)
    err = (C - ref).abs().max().item() / max(ref.abs().max().item(), 1e-6)
    assert err < 2e-6 * K ** 0.5, err  # same bf16 products, fp32 accumulation: only summation order differs


@pytest.mark.parametrize("K,splits,kps", [(8192, 32, 256), (1000, 3, 384), (65536, 8, 8192)])
def test_tc_gemm_split_k_partials(K, splits, kps):
    M, N = 256, 256
    g = torch.Generator(device="cuda").manual_seed(K)
    A = _mk(K, M, M, g)
    B = _mk(K, N, N, g)
    C = torch.full((splits, M, N), float("nan"), device="cuda")
    spz.spz_diag_gemm_bf16(M, N, K, A, M, 1, B, N, 1, C, N, splits=splits, k_per_split=kps)
    ref = _ref(A, 1, B, 1, M, N, K)
    err = (C.sum(0) - ref).abs().max().item() / ref.abs().max().item()
    assert err < 2e-6 * K ** 0.5
    for s in range(splits):
        lo, hi = s * kps, min(K, (s + 1) * kps)
        part = _ref(A[lo:hi] if lo < K else A[:0], 1, B[lo:hi] if lo < K else B[:0], 1, M, N, max(hi - lo, 0)) if hi > lo else torch.zeros(M, N, device="cuda")
        assert (C[s] - part).abs().max().item() <= 2e-6 * K ** 0.5 * max(ref.abs().max().item(), 1.0)


def test_simt_and_tc_agree():
    M, N, K = 1000, 256, 256
    g = torch.Generator(device="cuda").manual_seed(1)
    A = _mk(M, K, K, g)
    B = _mk(N, K, K, g)
    C1 = torch.empty(M, N, device="cuda")
    C2 = torch.empty(M, N, device="cuda")
    spz.spz_diag_gemm_bf16(M, N, K, A, K, 0, B, K, 0, C1, N, tensor_cores=True)
    spz.spz_diag_gemm_bf16(M, N, K, A, K, 0, B, K, 0, C2, N, tensor_cores=False)
    assert (C1 - C2).abs().max().item() < 1e-4 * C2.abs().max().item()


# ----------------------------------------------------------------------------- 3xTF32 (FP32 precision path)

def _mk32(rows, cols, ld, gen):
    x = torch.zeros(rows, ld, dtype=torch.float32, device="cuda")
    x[:, :cols] = torch.randn(rows, cols, generator=gen, device="cuda")
    return x


CASES32 = [
    (16384, 256, 256, 0, 0), (1000, 256, 28, 0, 0), (300, 12, 256, 0, 0), (257, 512, 64, 0, 0), (130, 33, 100, 0, 0),
    (128, 1, 256, 0, 0), (2048, 1024, 1024, 0, 0),
    (16384, 256, 256, 0, 1), (1000, 28, 256, 0, 1), (777, 256, 12, 0, 1), (200, 300, 96, 0, 1),
    (256, 256, 8192, 1, 1), (256, 28, 1000, 1, 1), (12, 256, 1000, 1, 1), (512, 44, 333, 1, 1),
]


@pytest.mark.parametrize("M,N,K,a_mn,b_mn", CASES32)
def test_tf32x3_gemm_matches_fp64(M, N, K, a_mn, b_mn):
    """3xTF32 keeps ~fp32 accuracy: error vs a float64 matmul of the same fp32 operands within a small
    multiple of fp32 rounding (plain tf32 would be ~2^-11 relative: 500x larger)."""
    g = torch.Generator(device="cuda").manual_seed(M * 5 + N * 11 + K)
    lda = ((M if a_mn else K) + 3) // 4 * 4
    ldb = ((N if b_mn else K) + 3) // 4 * 4
    A = _mk32(K, M, lda, g) if a_mn else _mk32(M, K, lda, g)
    B = _mk32(K, N, ldb, g) if b_mn else _mk32(N, K, ldb, g)
    C = torch.full((M, N), float("nan"), device="cuda")
    spz.spz_diag_gemm_f32(M, N, K, A, lda, a_mn, B, ldb, b_mn, C, N)
    Ad, Bd = A.double(), B.double()
    Am = Ad[:K, :M].t() if a_mn else Ad[:M, :K]
    Bm = Bd[:K, :N] if b_mn else Bd[:N, :K].t()
    ref = Am @ Bm
    scale = (Am.abs() @ Bm.abs())  # the fp32 error bound of each dot product scales with sum |a||b|
    err = ((C.double() - ref).abs() / scale.clamp_min(1e-30)).max().item()
    assert err < 3e-7 * K ** 0.5 + 1e-6, err  # fp32-accumulation scale; plain tf32 is ~5e-4


def test_tf32x3_split_k_partials():
    M, N, K, splits, kps = 256, 256, 1000, 3, 384
    g = torch.Generator(device="cuda").manual_seed(7)
    A = _mk32(K, M, M, g)
    B = _mk32(K, N, N, g)
    C = torch.full((splits, M, N), float("nan"), device="cuda")
    spz.spz_diag_gemm_f32(M, N, K, A, M, 1, B, N, 1, C, N, splits=splits, k_per_split=kps)
    for s in range(splits):
        lo, hi = s * kps, min(K, (s + 1) * kps)
        ref = A[lo:hi].double().t() @ B[lo:hi].double()
        scale = A[lo:hi].double().abs().t() @ B[lo:hi].double().abs()
        assert ((C[s].double() - ref).abs() / scale).max().item() < 2e-6


def test_tf32x3_and_simt_agree():
    M, N, K = 1000, 256, 256
    g = torch.Generator(device="cuda").manual_seed(3)
    A = _mk32(M, K, K, g)
    B = _mk32(N, K, K, g)
    C1 = torch.empty(M, N, device="cuda")
    C2 = torch.empty(M, N, device="cuda")
    spz.spz_diag_gemm_f32(M, N, K, A, K, 0, B, K, 0, C1, N, tensor_cores=True)
    spz.spz_diag_gemm_f32(M, N, K, A, K, 0, B, K, 0, C2, N, tensor_cores=False)
    assert (C1 - C2).abs().max().item() < 1e-5 * C2.abs().max().item()


PAIR_CASES = [
    # (M, N, K): forward K-major GEMMs on the CTA-pair kernel (cta_group::2, 256-row pair tiles): one pair tile,
    # a half-empty last pair (3 row blocks), ragged M / N / K, several tiles per pair, the HUM / TD3 layer shapes
    (256, 256, 64), (384, 256, 256), (1000, 300, 100), (4096, 512, 512), (49152, 256, 256), (20000, 1024, 1024),
]


@pytest.mark.parametrize("M,N,K", PAIR_CASES)
def test_tc_gemm_cta_pair_matches_fp32_matmul(M, N, K, monkeypatch):
    monkeypatch.setenv("SPZ_TC_PAIR", "1")
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    lda, ldb = (K + 7) // 8 * 8, (K + 7) // 8 * 8
    A = _mk(M, K, lda, g)
    B = _mk(N, K, ldb, g)
    C = torch.full((M, N), float("nan"), device="cuda")
    spz.spz_diag_gemm_bf16(M, N, K, A, lda, 0, B, ldb, 0, C, N)
    ref = _ref(A, 0, B, 0, M, N, K)
    err = (C - ref).abs().max().item() / max(ref.abs().max().item(), 1e-6)
    assert err < 2e-6 * K ** 0.5, err


@pytest.mark.parametrize("n_pre", [0, 1])
@pytest.mark.parametrize("M,N,K,splits,kps", [(256, 256, 8192, 32, 256), (512, 44, 3000, 3, 1024), (16384, 256, 256, 1, 256)])
def test_tc_gemm_dynamic_schedule(M, N, K, splits, kps, n_pre, monkeypatch):
    """Dynamic tile schedule (atomic tile counter, tiles handed to the MMA / epilogue warps through the shared
    queue; n_pre = 1: the group's tiles run before the grid-dependency wait): the same result as the static
    schedule, bit for bit, and the counters are back at zero after every launch (checked inside the call)."""
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a_mn = b_mn = 1 if splits > 1 or K > 1000 else 0
    lda = ((M if a_mn else K) + 7) // 8 * 8
    ldb = ((N if b_mn else K) + 7) // 8 * 8
    A = _mk(K, M, lda, g) if a_mn else _mk(M, K, lda, g)
    B = _mk(K, N, ldb, g) if b_mn else _mk(N, K, ldb, g)
    C0 = torch.full((splits, M, N), float("nan"), device="cuda")
    spz.spz_diag_gemm_bf16(M, N, K, A, lda, a_mn, B, ldb, b_mn, C0, N, splits=splits, k_per_split=kps)
    monkeypatch.setenv("SPZ_DIAG_GEMM_DYN", str(n_pre))
    for _ in range(3):  # repeated launches: the last CTA of each resets the counters
        C = torch.full((splits, M, N), float("nan"), device="cuda")
        spz.spz_diag_gemm_bf16(M, N, K, A, lda, a_mn, B, ldb, b_mn, C, N, splits=splits, k_per_split=kps)
        assert torch.equal(C, C0)
