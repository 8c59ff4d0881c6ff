"""Per-launch CTA timeline of ONE fused layer replayed back to back inside a CUDA graph: every
launch gets its own trace buffer (globaltimer at CTA entry, clock64 deltas inside), so the span
of each launch (first CTA entry -> last CTA exit), the gaps between launches and the per-CTA
phases (setup, first data, last item issued, epilogue done) are separated from graph overheads.
usage: python tools/launch_trace.py [cfg] [layer_index] [reps]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.layers import DerivedConv

cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
li = int(sys.argv[2]) if len(sys.argv) > 2 else 0
REPS = int(sys.argv[3]) if len(sys.argv) > 3 else 6
MAXCTA = 4096
lay = syn.CONFIGS[cfg][li]
x, w = syn.layer_inputs(lay, 1000 + li)
DATA = os.environ.get("DATA", "")
if DATA == "zero":
    x.zero_(); w.zero_()
elif DATA == "big":
    x.uniform_(-2, 2); w.uniform_(-2, 2)
PLAN = int(os.environ.get("PLAN", "0"))   # 0 auto, 1 fused (no autotune)
FORCE = os.environ.get("FORCE", "")       # "mt,fs,resident,pair,ksplit": force the fused plan family (with PLAN=1)
if FORCE:
    mt, fs, res, pr, ks = (int(v) for v in FORCE.split(","))
    O._lib.ollie_debug_force_plan(mt, fs, res)
    O._lib.ollie_debug_force_pair(pr)
    O._lib.ollie_debug_force_ksplit(ks)
conv = DerivedConv.from_layer(lay, plan=PLAN).prepare(w.cuda())
xd = x.cuda(); y = conv.new_output()
conv(xd, y)
print(lay.name, O.plan_describe(conv.shape, conv.code, conv.plan, conv.transposed))
O._lib.ollie_debug_set_trace.argtypes = [ctypes.c_void_p]
bufs = [torch.zeros(MAXCTA * 32, dtype=torch.int64, device="cuda") for _ in range(REPS)]
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        conv(xd, y, s.cuda_stream)
torch.cuda.synchronize()
FLUSH = os.environ.get("FLUSH", "0") == "1"       # evict L2 (2x L2 write + read back) before every launch
if FLUSH:
    fbuf = torch.empty(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device="cuda")
    fsink = torch.empty((), dtype=torch.int64, device="cuda")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for k in range(REPS):
        if FLUSH:
            fbuf.fill_(k)
            torch.sum(fbuf.view(torch.int64), dim=0, out=fsink)
        O._lib.ollie_debug_set_trace(bufs[k].data_ptr())
        conv(xd, y, s.cuda_stream)
O._lib.ollie_debug_set_trace(None)
# ramp the SM clock first (an idle B200 sits at ~120 MHz and takes a while to boost)
_a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(200):
    _a @ _a
for it in range(3):
    for b in bufs: b.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print(f"graph: {e0.elapsed_time(e1) * 1e3 / REPS:.2f} us per launch ({REPS} launches)")
prev_end = None
NAMES = [(0, "setup"), (2, "pdl-wait"), (1, "A0"), (3, "item0-mma"), (5, "item0-epi"), (4, "mma-done"),
         (6, "epi-done"), (31, "exit")]
for k, b in enumerate(bufs):
    t = b.view(-1, 32).cpu()
    t = t[t[:, 30] != 0].double()
    if t.shape[0] == 0:
        print(f"launch {k}: not traced (unfused plan?)"); continue
    st = t[:, 30]
    start, end = st.min().item(), t[:, 31].max().item()
    gap = (start - prev_end) / 1e3 if prev_end is not None else float("nan")
    rel = lambda c: ((t[:, c] - st) / 1e3)
    parts = " ".join(f"{nm} {rel(c).median().item():5.2f}/{rel(c).max().item():5.2f}" for c, nm in NAMES)
    print(f"launch {k}: span {(end - start) / 1e3:6.2f} gap-before {gap:6.2f} CTAs {t.shape[0]} "
          f"entry-spread {(st.max().item() - start) / 1e3:5.2f} | med/max us: {parts}")
    prev_end = end
    steps = []
    for qi in range(6):
        if (t[:, 8 + 3 * qi] == 0).all(): break
        steps.append(f"q{qi}: A {rel(8 + 3 * qi).median().item():5.2f} B {rel(9 + 3 * qi).median().item():5.2f} "
                     f"issued {rel(10 + 3 * qi).median().item():5.2f}")
    print("   steps (med us):", " | ".join(steps))
    # producer side: when each of the first steps' weight boxes could be issued (its b_empty wait returned)
    bi = [f"q{qi}: {rel(26 + qi).median().item():5.2f}" for qi in range(2) if not (t[:, 26 + qi] == 0).all()]
    if bi:
        print("   producer, weights issued (med us):", " | ".join(bi))
    print(f"   barrier check: thread0 saw epilogue flag in {(t[:, 28] == 0xD0E).sum().item()}/{t.shape[0]} CTAs; "
          f"thread128 post-barrier med {rel(29).median().item():5.2f} vs thread0 {rel(31).median().item():5.2f}")

# clock check: replay the graph for ~1 s while nvidia-smi samples the SM clock
import subprocess, time
p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                      "--format=csv,noheader", "-lms", "100"], stdout=subprocess.PIPE, text=True)
t0 = time.time(); n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 1.5:
    g.replay(); n += 1
    if n % 50 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
p.terminate(); out = p.communicate()[0].strip().splitlines()
print(f"sustained: {e0.elapsed_time(e1) * 1e3 / (n * REPS):.2f} us per launch over {n * REPS} launches; smi: {out[2:8]}")
