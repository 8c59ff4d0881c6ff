"""HBM write / copy / read ceilings on this box next to the eOperator kernels (E-b, E-c, E-f):
each op launched 20x back to back between two CUDA events (outputs > L2 where it matters), the
mean per launch reported with its algorithmic bytes.  Used to pick the roofline denominator of
write-dominated eOperators (a channel pad writes 16x what it reads)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2208_02025_b200 import eops, ollie as O


def t_of(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


out = {}
big = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for mb in (134, 512, 1024):
    nb = mb << 20
    v = big[:nb]
    t = t_of(lambda: v.fill_(1))
    out[f"fill {mb} MB"] = {"us": t * 1e6, "GBs": nb / t / 1e9}
    t = t_of(lambda: v.zero_())
    out[f"zero {mb} MB"] = {"us": t * 1e6, "GBs": nb / t / 1e9}
    t = t_of(lambda: dst[:nb].copy_(v))
    out[f"copy {mb} MB (r+w)"] = {"us": t * 1e6, "GBs": 2 * nb / t / 1e9}
    s = torch.empty((), dtype=torch.int64, device="cuda")
    t = t_of(lambda: torch.sum(v.view(torch.int64), dim=0, out=s))
    out[f"read-sum {mb} MB"] = {"us": t * 1e6, "GBs": nb / t / 1e9}

for cc in (1, 12):
    x = torch.randn(64, 256, 256, cc, device="cuda").to(torch.bfloat16)
    y = torch.empty(64, 256, 256, 16, device="cuda", dtype=torch.bfloat16)
    e = O.make_eop(eops.channel_pad(64, 256, 256, cc, 16), [O.BF16], O.BF16)
    t = t_of(lambda: O.eop_eval(e, [x], y))
    b = x.numel() * 2 + y.numel() * 2
    out[f"E-c channel_pad {cc}->16"] = {"us": t * 1e6, "GBs": b / t / 1e9, "write_GBs": y.numel() * 2 / t / 1e9}
    assert torch.equal(y[..., :cc], x) and not y[..., cc:].any()
x = torch.randn(16, 512, 64, 64, device="cuda").to(torch.bfloat16)
y = torch.empty(16, 64, 64, 512, device="cuda", dtype=torch.bfloat16)
e = O.make_eop(eops.nchw_to_nhwc(16, 512, 64, 64), [O.BF16], O.BF16)
t = t_of(lambda: O.eop_eval(e, [x], y))
out["E-b nchw_to_nhwc"] = {"us": t * 1e6, "GBs": 2 * x.numel() * 2 / t / 1e9}
assert torch.equal(y, x.permute(0, 2, 3, 1))
shp = O.conv_shape(16, 128, 16, 16, 64, 4, 4, 1, 2)
T = torch.randn(16 * 16 * 16, 1024, device="cuda")
Y = torch.empty(16, 32, 32, 64, device="cuda", dtype=torch.bfloat16)
t = t_of(lambda: O.offset_add(shp, True, T, 1024, O.BF16, Y))
b = 16 * 16 * 16 * 1024 * 4 * (15 * 15) / (16 * 16) + Y.numel() * 2
out["E-f selective add DCGAN"] = {"us": t * 1e6, "GBs": b / t / 1e9}
for k, v in out.items():
    print(f"{k:32s} {v['us']:9.2f} us {v['GBs']:8.1f} GB/s")
print(json.dumps(out))
