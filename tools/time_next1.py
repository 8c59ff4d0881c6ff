"""NEXT-1 measurement: CSRNet's dilated 3x3 (c = f = 512, 64x64, batch 16, d = 2) as the direct
fused form (tap offsets scaled by d) vs the derived dense form (space_to_batch -> dense conv ->
batch_to_space), each as CUDA-graph replay of 10 back-to-back calls; eOperator HBM GB/s and the
dense conv's TFLOP/s; cuDNN (graph) for reference."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

import ollie_synth as syn
from paper_2208_02025_b200 import DerivedConv, DilatedAsDense
from paper_2208_02025_b200 import ollie as O

import faulthandler
faulthandler.dump_traceback_later(90, exit=True)
torch.backends.cudnn.benchmark = True
REPS = 10


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


lay = syn.CONFIGS["csrnet"][0]
x, w = syn.layer_inputs(lay, 1000)
xd, wd = x.cuda(), w.cuda()
direct = DerivedConv.from_layer(lay).prepare(wd)
yd = direct.new_output()
direct(xd, yd)
der = DilatedAsDense.from_layer(lay).prepare(wd)
yv = der.new_output()
der(xd, yv)
torch.cuda.synchronize()
assert torch.equal(yd, yv) or (yd.float() - yv.float()).abs().max().item() <= 1e-2 * yd.float().abs().max().item()
t_direct = graph_time(lambda s: direct(xd, yd, s.cuda_stream))
t_der = graph_time(lambda s: der(xd, yv, s.cuda_stream))
t_s2b = graph_time(lambda s: O.eop_eval(der.s2b, [xd], der.xs, s.cuda_stream))
t_conv = graph_time(lambda s: der.conv(der.xs, der.ys, s.cuda_stream))
t_b2s = graph_time(lambda s: O.eop_eval(der.b2s, [der.ys], yv, s.cuda_stream))
xc = xd.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
wc = wd.contiguous(memory_format=torch.channels_last)
t_cudnn = graph_time(lambda s: F.conv2d(xc, wc, padding=lay.pad, dilation=lay.dilation))
flops = lay.useful_flops
eb = x.numel() * 2 * 2
out = {"layer": lay.name, "direct_us": t_direct, "derived_us": t_der, "s2b_us": t_s2b, "dense_conv_us": t_conv,
       "b2s_us": t_b2s, "cudnn_us": t_cudnn,
       "direct_tflops": flops / t_direct / 1e6, "derived_tflops": flops / t_der / 1e6,
       "dense_conv_tflops": flops / t_conv / 1e6, "s2b_gbs": eb / t_s2b / 1e3, "b2s_gbs": eb / t_b2s / 1e3,
       "plans": {"direct": O.plan_describe(direct.shape, direct.code, direct.plan, False),
                 "dense": O.plan_describe(der.conv.shape, der.conv.code, der.conv.plan, False)}}
print(json.dumps(out, indent=1))
