"""Per-layer device time of a config's chained/independent stack under several plans.

    python tools/plan_compare.py fsrcnn [plans...]      plans: auto fused unfused rowstream (default: all)

Each layer is captured alone in a CUDA graph of 10 back-to-back calls (warm) and timed with CUDA
events; 'flushed' replays one call after an L2 flush, averaged over 20 replays.  Parity is not
checked here (tests/ does that); the plan each layer resolved to is printed.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.stack import DerivedStack

cfg = sys.argv[1] if len(sys.argv) > 1 else "fsrcnn"
names = sys.argv[2:] or ["auto", "fused", "unfused", "rowstream"]
PLANS = {"auto": O.PLAN_AUTO, "fused": O.PLAN_FUSED, "unfused": O.PLAN_UNFUSED, "rowstream": O.PLAN_ROWSTREAM, "rs_ysum": O.PLAN_ROWSTREAM_YSUM, "rs_direct": O.PLAN_ROWSTREAM_DIRECT}
layers = syn.CONFIGS[cfg]
chained = cfg in ("fsrcnn", "dcgan")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty((), dtype=torch.int64, device="cuda")
stream = torch.cuda.Stream()


def graph(fn, reps):
    with torch.cuda.stream(stream):
        fn()
        fn()
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps):
            fn()
    return g


def timed(g, per, cold, reps):
    ts = []
    with torch.cuda.stream(stream):
        for k in range(reps):
            if cold:
                flush.fill_(k & 255)
                torch.sum(flush.view(torch.int64), dim=0, out=sink)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            ts.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) * 1e3 / per for a, b in ts)


xs, ws = [], []
for i, l in enumerate(layers):
    x, w = syn.layer_inputs(l, syn.config_seed(cfg, i))
    xs.append(x.cuda())
    ws.append(w.cuda())
for pn in names:
    plan = PLANS[pn]
    try:
        st = DerivedStack(layers, chained)
        for sl in st.layers:                 # the requested plan where the layer admits it, else AUTO
            try:
                O.plan_describe(sl.conv.shape, sl.conv.code, plan, sl.conv.transposed)
                if plan != O.PLAN_AUTO and (plan != O.PLAN_UNFUSED or sl.conv.ws_bytes >=
                                            O.workspace_bytes(sl.conv.shape, sl.conv.code, plan, sl.conv.transposed)):
                    sl.conv.plan, sl.conv.autotune = plan, False
            except O.OllieError:
                pass
        st.prepare(ws)
        st(xs[0] if chained else xs)          # autotune (AUTO)
        torch.cuda.synchronize()
    except Exception as e:                   # noqa: BLE001
        print(f"== {pn}: stack failed: {e!r}"[:200])
        continue
    print(f"== plan {pn}")
    src = xs[0] if chained else None
    tot_w = tot_f = 0.0
    for li, sl in enumerate(st.layers):
        inp = src if chained else xs[li]
        try:
            fn = (lambda sl, inp: (lambda: sl(inp, stream.cuda_stream)))(sl, inp)
            gw, gc = graph(fn, 10), graph(fn, 1)
            tw, tc = timed(gw, 10, False, 5), timed(gc, 1, True, 20)
            desc = O.plan_describe(sl.conv.shape, sl.conv.code, sl.conv.plan, sl.conv.transposed)
            print(f"  {sl.layer.name:28s} warm {tw:8.1f} us  flushed {tc:8.1f} us  {desc[:110]}")
            tot_w += tw
            tot_f += tc
        except Exception as e:               # noqa: BLE001
            print(f"  {sl.layer.name:28s} failed: {e!r}"[:160])
        src = sl.y
    print(f"  total warm {tot_w:.1f} us, flushed {tot_f:.1f} us")
