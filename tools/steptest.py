import sys, os
sys.path.insert(0, os.getcwd())
import torch
import bench
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
dev = torch.device("cuda", 0)
wl = bench.Workload(torch, "csrnet", dev, O.PLAN_AUTO)
stream = torch.cuda.Stream()
flush = bench.Flusher(torch, dev)
with torch.cuda.stream(stream):
    wl.step(stream); wl.step(stream)
torch.cuda.synchronize()
sl = wl.stack.layers[0]
fn = lambda s: sl(wl.inputs[0], s.cuda_stream)
for _ in range(2):
    print("layer fn", bench.time_graph_flushed(torch, fn, stream, flush))
    print("wl.step ", bench.time_graph_flushed(torch, lambda s: wl.step(s), stream, flush))
