"""Graph-replay time of the unfused plan's two kernels (merged GEMM, OffsetAdd) on their own,
for the layers whose AUTO plan is unfused (warm L2, 10 back-to-back launches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.layers import DerivedConv

REPS = 10
def graph_time(fn):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(REPS): fn(s)
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    for _ in range(50): a @ a
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / REPS)
    return min(ts)

cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
for i, lay in enumerate(syn.CONFIGS[cfg]):
    if lay.transposed: continue
    x, w = syn.layer_inputs(lay, 1000 + i)
    conv = DerivedConv.from_layer(lay, plan=O.PLAN_UNFUSED).prepare(w.cuda())
    xd = x.cuda(); y = conv.new_output()
    sh = conv.shape
    M, K, N = sh.n * sh.h * sh.w, sh.c, sh.r * sh.s * sh.f
    ldT = (N + 3) // 4 * 4
    T = torch.empty(M * ldT, dtype=torch.float32, device="cuda")
    tg = graph_time(lambda s: O.merged_gemm(M, N, K, conv.code, xd, conv.w_prep, T, ldT, s.cuda_stream))
    to = graph_time(lambda s: O.offset_add(sh, False, T, ldT, conv.code, y, s.cuda_stream))
    tu = graph_time(lambda s: conv(xd, y, s.cuda_stream))
    fl = 2 * M * N * K
    print(f"{lay.name:20s} M={M} N={N} K={K}: gemm {tg:6.2f} us ({fl / tg / 1e6:6.1f} TF/s, T {M * ldT * 4 / 1e6:.1f} MB "
          f"-> {M * ldT * 4 / tg / 1e3:.0f} GB/s)  offset_add {to:6.2f} us  unfused total {tu:6.2f} us")
