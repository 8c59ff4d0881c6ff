import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.layers import DerivedConv
lay = syn.CONFIGS["resnet18"][3]
x, w = syn.layer_inputs(lay, 1)
conv = DerivedConv.from_layer(lay).prepare(w.cuda())
tr = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
O._lib.ollie_debug_set_trace.argtypes = [ctypes.c_void_p]
O._lib.ollie_debug_set_trace(tr.data_ptr())
xd = x.cuda()
for v in (3, 7, 11, 15):
    O._lib.ollie_debug_set_flags(1 | 2 | 4 | 8 | (v << 4))
    conv(xd); torch.cuda.synchronize()
    t = tr.view(-1, 32)[:128].cpu()
    d = float((t[:, 3] - t[:, 1]).double().median())
    print("variant", v, "(1=LDS offsets, 2=var accumulate, 4=A stage rotation, 8=commit per chunk): cycles/MMA", d / 288)
