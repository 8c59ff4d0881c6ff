"""Per-layer in-kernel time and inter-kernel gaps INSIDE the bench's CUDA-graph replay: every
fused layer gets its own debug trace buffer (globaltimer at CTA entry; clock64 deltas inside)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.stack import DerivedStack

cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
layers = syn.CONFIGS[cfg]
chained = cfg in ("fsrcnn", "dcgan")
st = DerivedStack(layers, chained)
xs, ws = [], []
for i, l in enumerate(layers):
    x, w = syn.layer_inputs(l, 1000 + i)
    xs.append(x.cuda()); ws.append(w.cuda())
st.prepare(ws)
O._lib.ollie_debug_set_trace.argtypes = [ctypes.c_void_p]
bufs = [torch.zeros(4096 * 32, dtype=torch.int64, device="cuda") for _ in layers]
s = torch.cuda.Stream()
inputs = xs[0] if chained else xs
with torch.cuda.stream(s):
    for _ in range(3):
        st(inputs, stream=s.cuda_stream)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    x = inputs if chained else None
    for k, sl in enumerate(st.layers):
        O._lib.ollie_debug_set_trace(bufs[k].data_ptr())
        sl(x if chained else inputs[k], s.cuda_stream)
        x = sl.y
O._lib.ollie_debug_set_trace(None)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(5):
    flush.fill_(it); flush.view(torch.int64).sum()
    for b in bufs: b.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
step_us = e0.elapsed_time(e1) * 1e3
print(f"graph step {step_us:.1f} us")
# trace slots (fused_conv.cuh FC_TRACE): %globaltimer ns; 30 = CTA entry, 29 = epilogue warp past the
# final barrier (CTA exit), 0 = setup done, 1 = first A landed (MMA warp)
prev_end = None
for k, (sl, b) in enumerate(zip(st.layers, bufs)):
    t = b.view(-1, 32).cpu()
    t = t[t[:, 30] != 0].double()
    if t.shape[0] == 0:
        print(f"{sl.layer.name:24s} (unfused / not traced) plan: {O.plan_describe(sl.conv.shape, sl.conv.code, sl.conv.plan, sl.conv.transposed)[:40]}")
        prev_end = None
        continue
    start, end = t[:, 30].min().item(), t[:, 29].max().item()
    setup = ((t[:, 0] - t[:, 30]) / 1e3).median().item()
    a0 = ((t[:, 1] - t[:, 30]) / 1e3).median().item()
    gap = (start - prev_end) / 1e3 if prev_end else float("nan")
    print(f"{sl.layer.name:24s} start->end {(end - start) / 1e3:7.2f} us  gap-before {gap:6.2f} us  "
          f"setup {setup:5.2f} us  first-data {a0:5.2f} us  CTAs {t.shape[0]}")
    prev_end = end
