"""Time each layer of a config through the C ABI (events, L2 flush before each), print plan."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.layers import DerivedConv
cfg = sys.argv[1]
flags = 0
plan = int(sys.argv[3]) if len(sys.argv) > 3 else 0

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty((), dtype=torch.int64, device="cuda")
for li, lay in enumerate(syn.CONFIGS[cfg]):
    x, w = syn.layer_inputs(lay, 1)
    try:
        conv = DerivedConv.from_layer(lay, plan=plan).prepare(w.cuda())
    except Exception as e:
        print(lay.name, "skip", e); continue
    xd = x.cuda()
    ts = []
    for it in range(6):
        flush.fill_(it); torch.sum(flush.view(torch.int64), dim=0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); conv(xd); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts = sorted(ts[1:])
    tf = lay.useful_flops / (ts[len(ts) // 2] * 1e-6) / 1e12
    print(f"{lay.name:26s} {ts[len(ts)//2]:8.2f} us  {tf:7.1f} TF/s  | {O.plan_describe(conv.shape, conv.code, plan, lay.transposed)}")
