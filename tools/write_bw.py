"""Measured HBM bandwidth of a write-only stream (torch fill_ over 268 MB, the HUM dZ_L size) and of a copy,
for the roofline of the write-bound kernels (critic_dz_kernel, the gather's operand stores)."""
import torch

x = torch.empty(268 * 2**20 // 2, dtype=torch.bfloat16, device="cuda")
y = torch.empty_like(x)
for name, fn, mult in [("fill (write only)", lambda: x.fill_(1.0), 1), ("copy (read + write)", lambda: y.copy_(x), 2)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{name}: {x.numel() * 2 * mult / best / 1e6:.0f} GB/s ({best * 1e3:.1f} us for {x.numel() * 2 / 2**20:.0f} MiB)")
