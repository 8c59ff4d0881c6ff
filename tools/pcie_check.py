"""Pinned host <-> device copy bandwidth on this box (H2D, D2H, both at once), for the e2e bound."""
import torch
n = 12_794_880
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d():
    d_in.copy_(h_in, non_blocking=True)
def d2h():
    h_out.copy_(d_out, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms * 1e3:.1f} us for {n / 1e6:.1f} MB each way -> {n / ms / 1e6:.1f} GB/s per direction")

# the e2e pipeline's copy pattern without compute: per-layer H2D on one stream, the layer's D2H on
# the other once its H2D landed, 20 steps, two buffer sets
sizes = [6422528, 3211264, 1605632, 802816, 401408, 200704, 100352, 50176]
hi = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for n in sizes]
ho = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for n in sizes]
di = [[torch.empty(n, dtype=torch.uint8, device="cuda") for n in sizes] for _ in range(2)]
do = [[torch.empty(n, dtype=torch.uint8, device="cuda") for n in sizes] for _ in range(2)]
def pipe(steps=20, dep=True):
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    for k in range(steps):
        b = k % 2
        for i in range(len(sizes)):
            e = torch.cuda.Event()
            with torch.cuda.stream(s1):
                di[b][i].copy_(hi[i], non_blocking=True)
                e.record(s1)
            if dep:
                s2.wait_event(e)
            with torch.cuda.stream(s2):
                ho[i].copy_(do[b][i], non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for dep in (False, True):
    ms = t(lambda: pipe(20, dep), reps=3) / 20
    print(f"pipeline pattern dep={dep}: {ms * 1e3:.1f} us per step ({sum(sizes) / ms / 1e6:.1f} GB/s per direction)")
