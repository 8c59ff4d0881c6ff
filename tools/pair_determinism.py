"""CTA-pair (cta_group::2) fused plans: 30 back-to-back runs of the same random inputs must give
bit-identical outputs (a shared-memory race would show up as run-to-run differences)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.layers import DerivedConv

O._lib.ollie_debug_force_pair(1)
bad = 0
for lay in (syn.Layer("p1", 2, 256, 14, 14, 128, 3, 3, pad=1), syn.Layer("p2", 16, 64, 56, 56, 64, 3, 3, pad=1),
            syn.Layer("p3", 2, 64, 4, 4, 128, 4, 4, pad=1, stride=2, transposed=True)):
    x, w = syn.layer_inputs(lay, 11)
    conv = DerivedConv.from_layer(lay, plan=O.PLAN_FUSED).prepare(w.cuda())
    xd = x.cuda()
    ref = conv(xd).clone()
    for _ in range(30):
        y = conv(xd)
        bad += int(not torch.equal(y, ref))
    torch.cuda.synchronize()
    print(lay.name, O.plan_describe(conv.shape, conv.code, O.PLAN_FUSED, lay.transposed)[-60:], "mismatching runs:", bad)
print("determinism", "OK" if bad == 0 else "FAILED")
