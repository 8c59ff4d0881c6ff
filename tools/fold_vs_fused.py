"""Strided / wide layers as im2col ("tap folding") eOperator + 1x1 derived conv (a plain merged GEMM)
vs the fused phase plan: warm (10 calls in a graph) and L2-flushed (differential graph) times, and
parity of the folded path against the fused one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.stack import StackLayer

flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def graph_us(fn, reps=10, flush=False):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s)
    torch.cuda.synchronize()
    def build(with_call):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for k in range(reps):
                if flush:
                    flush_buf.fill_(k & 255)
                if with_call:
                    fn(s)
        return g
    def t(g):
        best = 1e30
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
        return best
    gc = build(True)
    tc = t(gc)
    if flush:
        tc -= t(build(False))
    return tc


cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet18_s2"
for li, lay in enumerate(syn.CONFIGS[cfg]):
    x, w = syn.layer_inputs(lay, 60 + li)
    xd, wd = x.cuda(), w.cuda()
    fused = StackLayer(lay, lay.c, lay.f, False, O.PLAN_AUTO, "cuda", fold=False)
    fused.prepare(wd)
    folded = StackLayer(lay, lay.c, lay.f, False, O.PLAN_AUTO, "cuda", fold=True)
    folded.prepare(wd)
    y0 = fused(xd); y1 = folded(xd); torch.cuda.synchronize()
    y0 = fused(xd); y1 = folded(xd); torch.cuda.synchronize()
    diff = (y0.float() - y1.float()).abs().max().item() / max(y0.float().abs().max().item(), 1e-30)
    tw0 = graph_us(lambda s: fused(xd, stream=s.cuda_stream))
    tw1 = graph_us(lambda s: folded(xd, stream=s.cuda_stream))
    tf0 = graph_us(lambda s: fused(xd, stream=s.cuda_stream), flush=True)
    tf1 = graph_us(lambda s: folded(xd, stream=s.cuda_stream), flush=True)
    print(f"{lay.name:24s} fused {tf0:6.1f}/{tw0:6.1f} us  fold+1x1 {tf1:6.1f}/{tw1:6.1f} us (flushed/warm)  rel diff {diff:.2e}"
          f"  [{fused.conv.resolved_plan()} | {folded.conv.resolved_plan()}]", flush=True)
