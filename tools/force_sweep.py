"""Warm CUDA-graph time (10 back-to-back launches) of one layer under forced fused-plan families
(MT, FS, residency, CTA pairs, split-K), next to the autotuned plan -- checks the autotuner's pick."""
import itertools, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.layers import DerivedConv

cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
li = int(sys.argv[2]) if len(sys.argv) > 2 else 0
REPS = 10


def graph_time(fn):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(REPS):
            fn(s)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / REPS)
    return min(ts)


lay = syn.CONFIGS[cfg][li]
x, w = syn.layer_inputs(lay, 1000 + li)
xd, wd = x.cuda(), w.cuda()
auto = DerivedConv.from_layer(lay).prepare(wd)
y = auto.new_output()
auto(xd, y)
print(f"{lay.name} auto {graph_time(lambda s: auto(xd, y, s.cuda_stream)):.2f} us  {auto.resolved_plan()}")
res = []
G8S = tuple(int(v) for v in os.environ.get("G8S", "-1").split(","))
OCCS = tuple(int(v) for v in os.environ.get("OCCS", "0").split(","))   # CTAs per SM (0 = planner's choice)
for mt, fs, rs, pr, ks, g8, occ in itertools.product((1, 2, 4), (32, 64, 128, 256), (0, 1), (0, 1), (1, 2, 4), G8S, OCCS):
    O._lib.ollie_debug_force_grp8(g8)
    O._lib.ollie_debug_force_occ(occ)
    O._lib.ollie_debug_force_plan(mt, fs, rs)
    O._lib.ollie_debug_force_pair(pr)
    O._lib.ollie_debug_force_ksplit(ks)
    try:
        conv = DerivedConv.from_layer(lay, plan=O.PLAN_FUSED, autotune=False).prepare(wd)
        d = O.plan_describe(conv.shape, conv.code, O.PLAN_FUSED, conv.transposed)
        t = graph_time(lambda s: conv(xd, y, s.cuda_stream))
        res.append((t, d))
    except Exception:
        pass
O._lib.ollie_debug_force_plan(0, 0, -1)
O._lib.ollie_debug_force_pair(-1)
O._lib.ollie_debug_force_ksplit(-1)
O._lib.ollie_debug_force_grp8(-1)
O._lib.ollie_debug_force_occ(0)
res.sort()
for t, d in res[:int(os.environ.get("TOP", "6"))]:
    print(f"   {t:7.2f} us  {d}")
