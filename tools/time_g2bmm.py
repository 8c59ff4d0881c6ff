"""NEXT-4 measurement: G2BMM on the LongFormer config ([8, 10000, 64], W = 256, d = 4; reading R4),
derived form (residue-split tiles, the paper's optimized program) vs direct dilated form (the
original), CUDA-graph replay of 10 back-to-back calls (min of 5); HBM roofline from bytes
|A| + |B| + |out| against MEASURED_PEAKS.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O

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


peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = None
for k, v in peaks.items():
    if "hbm" in k.lower() or "copy" in k.lower() or "bandwidth" in k.lower():
        if isinstance(v, (int, float)):
            hbm = hbm or float(v)
res = {}
dbg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
O._lib.ollie_debug_g2bmm_flags(dbg)
for g in syn.G2_CONFIGS["longformer"] + [syn.G2("longformer_d1_w256", 8, 10000, 64, 256, 1),
                                         syn.G2("longformer_d2_w256", 8, 10000, 64, 256, 2)]:
    a, b = syn.g2bmm_inputs(g, 1000)
    a, b = a.cuda(), b.cuda()
    nw = 2 * g.W + 1
    for ldo in (nw, (nw + 7) // 8 * 8):
        out = torch.empty(g.batch, g.L, ldo, dtype=torch.bfloat16, device="cuda")
        nbytes = g.bytes + 2 * g.batch * g.L * (ldo - nw)
        for form, name in ((0, "derived"), (1, "direct")):
            if form == 1 and g.d > 4:
                continue
            t = graph_time(lambda s: O.g2bmm(g.batch, g.L, g.K, g.W, g.d, O.BF16, a, b, out, ldo, form=form,
                                             stream=s.cuda_stream))
            res[f"{g.name}/{name}/ldo{ldo}"] = {"us": t, "GBs": nbytes / t / 1e3, "TFLOPs": g.flops / t / 1e6,
                                                "frac_hbm": (nbytes / t / 1e3) / hbm if hbm else None, "bytes": nbytes}
print(json.dumps({"hbm_peak_GBs": hbm, "results": res}, indent=1))
