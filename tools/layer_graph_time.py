"""Per-layer steady-state time inside a CUDA graph: 10 back-to-back calls of the same layer (PDL
on, warm L2), for ours (AUTO after autotune) and cuDNN (graph-captured too, for a like-for-like)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
import ollie_synth as syn
from paper_2208_02025_b200.layers import DerivedConv

torch.backends.cudnn.benchmark = True
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("cfg", nargs="?", default="resnet18")
ap.add_argument("--pair", type=int, default=-1, help="-1 auto, 0 single-CTA plans, 1 CTA-pair plans")
ap.add_argument("--no-cudnn", action="store_true")
ap.add_argument("--ks", type=int, default=-1, help="-1 auto, else force the split-K factor")
ap.add_argument("--describe", action="store_true")
ap.add_argument("--plan", type=int, default=0, help="0 auto, 1 fused, 2 unfused, 3 gemm_red")
args = ap.parse_args()
cfg = args.cfg
REPS = 10
from paper_2208_02025_b200 import ollie as O
O._lib.ollie_debug_force_pair(args.pair)
O._lib.ollie_debug_force_ksplit(args.ks)


def graph_time(fn):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(REPS):
            fn(s)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / REPS)
    return min(ts)


tot_o = tot_c = 0.0
for i, lay in enumerate(syn.CONFIGS[cfg]):
    x, w = syn.layer_inputs(lay, 1000 + i)
    conv = DerivedConv.from_layer(lay, plan=args.plan).prepare(w.cuda())
    xd = x.cuda(); y = conv.new_output()
    conv(xd, y)
    t_o = graph_time(lambda s: conv(xd, y, s.cuda_stream))
    xc = xd.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
    wc = w.cuda().contiguous(memory_format=torch.channels_last)
    if lay.transposed:
        fc = lambda s: F.conv_transpose2d(xc, wc, stride=lay.stride, padding=lay.pad, output_padding=lay.output_padding)
    else:
        fc = lambda s: F.conv2d(xc, wc, stride=lay.stride, padding=lay.pad, dilation=lay.dilation)
    t_c = 0.0 if args.no_cudnn else graph_time(fc)
    tot_o += t_o; tot_c += t_c
    print(f"{lay.name:24s} ours {t_o:7.2f} us   cudnn(graph) {t_c:7.2f} us   {conv.resolved_plan()}")
    if args.describe:
        print("    ", O.plan_describe(conv.shape, conv.code, conv.plan, conv.transposed))
print(f"{'sum':24s} ours {tot_o:7.2f} us   cudnn(graph) {tot_c:7.2f} us")
