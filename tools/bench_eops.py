"""Measure the eOperator configs of SURVEY 8(d) (E-b ... E-f): GB/s = algorithmic (|in|+|out|) / time,
events around each launch, L2 flushed before each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2208_02025_b200 import eops, ollie as O

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty((), dtype=torch.int64, device="cuda")


def timeit(fn, reps=10):
    ts = []
    for k in range(reps):
        flush.fill_(k); torch.sum(flush.view(torch.int64), dim=0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


res = {}
peak = 6553.6
# E-b: NCHW -> NHWC (CSRNet input [16,512,64,64] bf16)
n, c, h, w = 16, 512, 64, 64
x = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16)
y = torch.empty(n, h, w, c, device="cuda", dtype=torch.bfloat16)
e = O.make_eop(eops.nchw_to_nhwc(n, c, h, w), [O.BF16], O.BF16)
t = timeit(lambda: O.eop_eval(e, [x], y))
assert torch.equal(y, x.permute(0, 2, 3, 1))
res["E-b nchw_to_nhwc 16x512x64x64 bf16"] = (2 * x.numel() * 2, t)
# E-c: channel pad 1 -> 16 (FSRCNN input [64,256,256,1] bf16) and 12 -> 16 (FSRCNN mid activations)
for cc in (1, 12):
    x = torch.randn(64, 256, 256, cc, device="cuda").to(torch.bfloat16)
    y = torch.empty(64, 256, 256, 16, device="cuda", dtype=torch.bfloat16)
    e = O.make_eop(eops.channel_pad(64, 256, 256, cc, 16), [O.BF16], O.BF16)
    t = timeit(lambda: O.eop_eval(e, [x], y))
    assert torch.equal(y[..., :cc], x) and not y[..., cc:].any()
    res[f"E-c channel_pad {cc}->16 64x256x256 bf16"] = (x.numel() * 2 + y.numel() * 2, t)
# E-d: weight DLT [512,512,3,3] bf16 (compile time, timed once)
shp = O.conv_shape(1, 512, 7, 7, 512, 3, 3, 1)
wt = torch.randn(512, 512, 3, 3, device="cuda").to(torch.bfloat16)
wp = torch.empty(9 * 512, 512, device="cuda", dtype=torch.bfloat16)
t = timeit(lambda: O.prepare_weight_conv2d(shp, O.BF16, wt, wp))
res["E-d weight DLT 512x512x3x3 bf16"] = (2 * wt.numel() * 2, t)
# E-e: OffsetAdd standalone (B-K2), R18 64x56^2 b16: T fp32 [50176, 576] -> Y bf16
shp = O.conv_shape(16, 64, 56, 56, 64, 3, 3, 1)
T = torch.randn(16 * 56 * 56, 576, device="cuda")
Y = torch.empty(16, 56, 56, 64, device="cuda", dtype=torch.bfloat16)
t = timeit(lambda: O.offset_add(shp, False, T, 576, O.BF16, Y))
inb = 16 * (56 * 3 - 2) * (56 * 3 - 2) * 64 * 4           # in-bounds (pixel, tap) reads
res["E-e OffsetAdd (standalone) R18 64x56 b16"] = (inb + Y.numel() * 2, t)
# E-f: selective add (ConvT), DCGAN 128->64 16->32 b16: T fp32 [4096, 1024] -> Y bf16
shp = O.conv_shape(16, 128, 16, 16, 64, 4, 4, 1, 2)
T = torch.randn(16 * 16 * 16, 1024, device="cuda")
Y = torch.empty(16, 32, 32, 64, device="cuda", dtype=torch.bfloat16)
t = timeit(lambda: O.offset_add(shp, True, T, 1024, O.BF16, Y))
res["E-f selective add DCGAN 128->64 b16"] = (16 * 16 * 16 * 1024 * 4 * (15 * 15) / (16 * 16) + Y.numel() * 2, t)
out = {}
for k, (b, t) in res.items():
    out[k] = {"us": t * 1e6, "GBs": b / t / 1e9, "frac_of_measured_hbm": b / t / 1e9 / peak, "bytes": b}
    print(f"{k:45s} {t*1e6:9.2f} us {b/t/1e9:8.1f} GB/s  {b/t/1e9/peak:.2f} of measured HBM")
print(json.dumps(out))
