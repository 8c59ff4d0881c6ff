"""Row-streaming kernel timeline on a raw torch input (no pad eOperator before it)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200 import DerivedConv
c = int(sys.argv[1]) if len(sys.argv) > 1 else 16
lay = syn.Layer("map16", 64, c, 256, 256, 16, 3, 3, pad=1)
conv = DerivedConv.from_layer(lay, plan=O.PLAN_ROWSTREAM)
x, w = syn.layer_inputs(lay, 5)
conv.prepare(w.cuda())
xd = x.cuda()
y = conv.new_output()
for _ in range(3):
    conv(xd, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); conv(xd, y); e1.record(); torch.cuda.synchronize()
print("layer us", e0.elapsed_time(e1) * 1e3)
tr = torch.zeros(1024, dtype=torch.int64, device="cuda")
O._lib.ollie_debug_set_trace(O.ctypes.c_void_p(tr.data_ptr()))
conv(xd, y)
torch.cuda.synchronize()
O._lib.ollie_debug_set_trace(O.ctypes.c_void_p(0))
t = tr.cpu().tolist()
t0 = min(v for v in t if v > 0)
for k in range(12):
    f = lambda v: f"{(v - t0) / 1e3:9.2f}" if v > 0 else "        -"
    print(f"{k:3d} {f(t[k])} {f(t[64 + k])}   | {k:3d} {f(t[128 + k])} {f(t[192 + k])}")
print("epilogue warp 0: start, after afull wait, h0 loads issued, h0 loaded, h1 issued, h1 loaded, stores done, released")
for k in range(12):
    print(k, " ".join(f"{(t[256 + k * 8 + i] - t0) / 1e3:6.2f}" for i in range(8)))
