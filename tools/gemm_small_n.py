"""Merged-GEMM throughput for tall, narrow shapes (FSRCNN 1x1 layers): time and HBM GB/s of X + T."""
import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_02025_b200 import ollie as O
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
for M, N, K in ((4194304, 16, 56), (4194304, 64, 16), (4194304, 576, 64), (1048576, 16, 64), (262144, 16, 64)):
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    ldT = (N + 3) // 4 * 4
    T = torch.empty(M, ldT, device="cuda")
    us = t(lambda: O.merged_gemm(M, N, K, O.BF16, a, b, T, ldT))
    byts = M * K * 2 + M * ldT * 4
    print(f"M={M} N={N} K={K}: {us:.1f} us, {byts / us / 1e3:.0f} GB/s")
