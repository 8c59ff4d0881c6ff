"""Sweep fused-plan parameters (MT, FS, resident) per layer; print the fastest (events, L2 flushed)."""
import os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.layers import DerivedConv
cfg = sys.argv[1]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty((), dtype=torch.int64, device="cuda")
def timeit(conv, xd, y):
    ts = []
    for it in range(5):
        flush.fill_(it); torch.sum(flush.view(torch.int64), dim=0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); conv(xd, y); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts[1:])[1]
for li, lay in enumerate(syn.CONFIGS[cfg]):
    x, w = syn.layer_inputs(lay, 1)
    conv = DerivedConv.from_layer(lay).prepare(w.cuda())
    xd = x.cuda(); y = conv.new_output()
    O._lib.ollie_debug_force_plan(0, 0, -1)
    base = timeit(conv, xd, y)
    res = []
    for mt, fs, rs in itertools.product((1, 2, 3, 4), (16, 32, 64, 128, 256), (0, 1)):
        O._lib.ollie_debug_force_plan(mt, fs, rs)
        try:
            d = O.plan_describe(conv.shape, conv.code)
            t = timeit(conv, xd, y)
            res.append((t, mt, fs, rs, d))
        except Exception:
            pass
    O._lib.ollie_debug_force_plan(0, 0, -1)
    res.sort()
    print(f"{lay.name}: auto {base:.2f} us ; best:")
    for r in res[:3]:
        print(f"   {r[0]:8.2f} us MT={r[1]} FS={r[2]} res={r[3]} | {r[4]}")
