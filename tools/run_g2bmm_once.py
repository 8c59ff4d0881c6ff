"""One G2BMM call per form on the LongFormer config (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O

g = syn.G2_CONFIGS["longformer"][0]
a, b = syn.g2bmm_inputs(g, 1000)
a, b = a.cuda(), b.cuda()
for ldo in (2 * g.W + 1, 520):
    out = torch.empty(g.batch, g.L, ldo, dtype=torch.bfloat16, device="cuda")
    for form in (0, 1):
        O.g2bmm(g.batch, g.L, g.K, g.W, g.d, O.BF16, a, b, out, ldo, form)
torch.cuda.synchronize()
print("done")
