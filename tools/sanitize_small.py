"""Small configs through every ABI path, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O, eops
from paper_2208_02025_b200.layers import DerivedConv
from tests import eop_cases as ec

layers = [syn.Layer("c", 2, 64, 9, 11, 64, 3, 3, pad=1), syn.Layer("t", 2, 64, 3, 3, 48, 4, 4, pad=1, stride=2, transposed=True),
          syn.Layer("d", 1, 32, 12, 12, 40, 3, 3, pad=2, dilation=2), syn.Layer("k", 1, 8, 9, 7, 24, 5, 5, pad=2),
          syn.Layer("o", 2, 16, 5, 5, 8, 1, 1)]
for lay in layers:
    x, w = syn.layer_inputs(lay, 3)
    for plan in (O.PLAN_FUSED, O.PLAN_UNFUSED):
        try:
            conv = DerivedConv.from_layer(lay, plan=plan, autotune=False).prepare(w.cuda())
            conv(x.cuda())
        except O.OllieError as e:
            if e.status != O.E_UNSUPPORTED:
                raise
for spec, shapes in ((ec.transpose_nchw_to_nhwc(2, 33, 5, 7), [(2, 33, 5, 7)]),
                     (ec.channel_pad(2, 5, 6, 3, 8), [(2, 5, 6, 3)]),
                     (ec.fused_pad_then_offset_add(1, 4, 5, 2, 3, 3, 1, 3), [(1, 4, 5, 18)])):
    e = O.make_eop(spec, [O.FP32] * len(shapes), O.FP32)
    ins = [torch.randn(s, device="cuda") for s in shapes]
    out = torch.empty([hi - lo for lo, hi in spec["scopes"][0]["trav"]], device="cuda")
    O.eop_eval(e, ins, out)
torch.cuda.synchronize()
print("sanitize run ok")
