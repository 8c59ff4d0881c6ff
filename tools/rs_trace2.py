"""Row-streaming kernel timeline on a raw torch input (no pad eOperator before it)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200 import DerivedConv
arg = sys.argv[1] if len(sys.argv) > 1 else "16"
if ":" in arg:                                   # config:layer-index, e.g. fsrcnn:7
    cname, li = arg.split(":")
    lay = syn.CONFIGS[cname][int(li)]
else:
    lay = syn.Layer("map16", 64, int(arg), 256, 256, 16, 3, 3, pad=1)
PLAN = {"auto": O.PLAN_ROWSTREAM, "ysum": O.PLAN_ROWSTREAM_YSUM, "direct": O.PLAN_ROWSTREAM_DIRECT}[os.environ.get("RS_FORM", "auto")]
conv = DerivedConv.from_layer(lay, plan=PLAN)
print(conv.resolved_plan(), O.plan_describe(conv.shape, conv.code, PLAN, lay.transposed))
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
for k in range(24):
    f = lambda v: f"{(v - t0) / 1e3:9.2f}" if v > 0 else "        -"
    print(f"{k:3d} {f(t[k])} {f(t[64 + k])}   | {k:3d} {f(t[128 + k])} {f(t[192 + k])}")
if int(os.environ.get("OLLIE_RS_DBG", "0")) & 4:
    c = t[256:256 + 12]
    print("epilogue row 4 (warp 4) clock64 since start: afull waited; per h: ld issued, ld waited, summed, stored:",
          [v - c[0] if v > 0 else None for v in c])
if int(os.environ.get("OLLIE_RS_DBG", "0")) & 8:
    c = t[319:319 + 16]
    print("direct MMA groups of row 5 (clock64 cycles since the waits):", [v - c[0] if v > 0 else None for v in c])
