"""Launch the channel-pad eOp and the standalone OffsetAdd a few times (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2208_02025_b200 import eops, ollie as O
x = torch.randn(64, 256, 256, 12, device="cuda").to(torch.bfloat16)
y = torch.empty(64, 256, 256, 16, device="cuda", dtype=torch.bfloat16)
e = O.make_eop(eops.channel_pad(64, 256, 256, 12, 16), [O.BF16], O.BF16)
shp = O.conv_shape(16, 64, 56, 56, 64, 3, 3, 1)
T = torch.randn(16 * 56 * 56, 576, device="cuda")
Y = torch.empty(16, 56, 56, 64, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    O.eop_eval(e, [x], y)
    O.offset_add(shp, False, T, 576, O.BF16, Y)
torch.cuda.synchronize()
print("ok")
