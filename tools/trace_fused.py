"""Debug: per-CTA timeline of the fused kernel for one configured layer (clock64 deltas)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.layers import DerivedConv

cfg, li = sys.argv[1], int(sys.argv[2])
noflush = "noflush" in sys.argv[3:]
dbg = int([a for a in sys.argv[3:] if a.startswith("flags=")][0][6:]) if any(a.startswith("flags=") for a in sys.argv[3:]) else 0

lay = syn.CONFIGS[cfg][li]
from dataclasses import replace as _rep
from paper_2208_02025_b200.stack import padded_channels
lay = _rep(lay, c=padded_channels(lay.c, lay.dtype), f=padded_channels(lay.f, lay.dtype) if cfg == 'fsrcnn' and li < 7 else lay.f)
x, w = syn.layer_inputs(lay, 1)
auto = "auto" in sys.argv[3:]
kv = dict(a.split("=") for a in sys.argv[3:] if "=" in a and not a.startswith("flags="))
O._lib.ollie_debug_force_plan(int(kv.get("mt", 0)), int(kv.get("fs", 0)), int(kv.get("res", -1)))
O._lib.ollie_debug_force_pair(int(kv.get("pair", -1)))
O._lib.ollie_debug_force_ksplit(int(kv.get("ks", -1)))
conv = DerivedConv.from_layer(lay, plan=0 if auto else 1).prepare(w.cuda())
xd = x.cuda()
if auto:
    conv(xd)          # autotune; the trace then follows the tuned plan
tr = torch.zeros(148 * 32 * 4, dtype=torch.int64, device="cuda")
O._lib.ollie_debug_set_trace.argtypes = [ctypes.c_void_p]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    O._lib.ollie_debug_set_trace(tr.data_ptr() if it == 3 else None)
    if not noflush:
        flush.fill_(it)
    else:
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    conv(xd)
    e1.record()
    torch.cuda.synchronize()
    print("iter", it, "us", round(e0.elapsed_time(e1) * 1e3, 2))
O._lib.ollie_debug_set_trace(None)
print(lay.name, O.plan_describe(conv.shape, conv.code))
t = tr.view(-1, 32).cpu()
t = t[t[:, 30] != 0]
g0 = t[:, 30].min()
names = ["setup", "A0", "-", "tile0_mma", "-", "epi0", "epi_end", "end"]
for q in range(6):
    names += [f"s{q}_A", f"s{q}_B", f"s{q}_issued"]
names = names[:8] + names[8:]
print("CTAs", t.shape[0], "start spread (ns):", int((t[:, 30] - g0).max()))
for k, nm in enumerate(names):
    if nm == '-': continue
    if k >= 8 and (t[:, k] == 0).all(): continue
    col = t[:, k].double()
    print(f"{nm:10s} min {col.min():9.0f} med {col.median():9.0f} max {col.max():9.0f}")
