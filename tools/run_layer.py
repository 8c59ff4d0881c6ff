"""Run one configured layer N times through the C ABI (for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.stack import DerivedStack

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="resnet18")
ap.add_argument("--layer", type=int, default=-1, help="-1: all layers of the config")
ap.add_argument("--plan", default="auto", choices=["auto", "fused", "unfused", "rowstream", "rs_ysum", "rs_direct"])
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
layers = syn.CONFIGS[a.config]
if a.layer >= 0:
    layers = [layers[a.layer]]
chained = a.config in ("fsrcnn", "dcgan") and a.layer < 0
plan = {"auto": O.PLAN_AUTO, "fused": O.PLAN_FUSED, "unfused": O.PLAN_UNFUSED, "rowstream": O.PLAN_ROWSTREAM, "rs_ysum": O.PLAN_ROWSTREAM_YSUM, "rs_direct": O.PLAN_ROWSTREAM_DIRECT}[a.plan]
st = DerivedStack(layers, chained)
for sl in st.layers:          # the requested plan where the layer admits it, else AUTO
    try:
        O.plan_describe(sl.conv.shape, sl.conv.code, plan, sl.conv.transposed)
        if plan != O.PLAN_AUTO:
            sl.conv.plan, sl.conv.autotune = plan, False
    except O.OllieError:
        pass
ws, xs = [], []
for i, l in enumerate(layers):
    x, w = syn.layer_inputs(l, 1000 + i)
    xs.append(x.cuda())
    ws.append(w.cuda())
st.prepare(ws)
st(xs[0] if chained else xs)       # first call autotunes every layer (not profiled)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()   # ncu --profile-from-start off: only the tuned launches
for _ in range(a.iters):
    st(xs[0] if chained else xs)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", [l.name for l in layers])
