"""Diagnosis: per-tile timeline of the persistent tcgen05 GEMM (test infrastructure)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_06126_b200 import spz

def run(M, N, K, a_mn, b_mn, label):
    lda = ((M if a_mn else K) + 7)//8*8; ldb = ((N if b_mn else K) + 7)//8*8
    A = torch.randn((K, lda) if a_mn else (M, lda), device="cuda").bfloat16()
    B = torch.randn((K, ldb) if b_mn else (N, ldb), device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda")
    for _ in range(3): spz.spz_diag_gemm_bf16(M, N, K, A, lda, a_mn, B, ldb, b_mn, C, N)
    spz.spz_diag_tc_trace(True)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); spz.spz_diag_gemm_bf16(M, N, K, A, lda, a_mn, B, ldb, b_mn, C, N); e.record(); torch.cuda.synchronize()
    tr = spz.spz_diag_tc_trace(False, read=True).astype(np.int64)
    t0 = tr[tr > 0].min()
    print(f"== {label}: M={M} N={N} K={K} event-time {s.elapsed_time(e)*1000:.1f} us")
    for c in (0, 1, 74, 147):
        row = []
        for i in range(8):
            if tr[c, i, 0] == 0: break
            row.append("[" + " ".join(f"{(x - t0)/1000:6.2f}" if x else "   -  " for x in tr[c, i]) + "]")
        print(f"cta {c:3d}: " + " ".join(row))
    prod = tr[:, :, 0]; mma = tr[:, :, 1]; acc = tr[:, :, 2]; done = tr[:, :, 3]
    ok = (prod > 0) & (done > 0)
    print("mean mainloop (prod start -> mma done) %.2f us; mean epilogue (acc -> done) %.2f us; last done %.2f us" % (
        ((mma - prod)[ok]).mean() / 1000, ((done - acc)[ok]).mean() / 1000, (done[ok].max() - t0) / 1000))

run(49152, 256, 256, 0, 0, "critic-fwd-like (K-major, 384 tiles)")
run(49152, 256, 32, 0, 0, "layer-0-like K=32")
run(16384, 256, 256, 0, 1, "dgrad-like")
