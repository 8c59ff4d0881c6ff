"""Run cuDNN's conv (torch, channels_last, cudnn.benchmark) on one BASELINE layer a few times -- for an
ncu capture of the library kernel next to ours (`ncu -k regex:'^(?!ollie)' ...`)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
import ollie_synth as syn

cfg = sys.argv[1] if len(sys.argv) > 1 else "csrnet"
li = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lay = syn.CONFIGS[cfg][li]
torch.backends.cudnn.benchmark = True
x, w = syn.layer_inputs(lay, 1)
xd = x.cuda().permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
wd = w.cuda().contiguous(memory_format=torch.channels_last)
fn = (lambda: F.conv_transpose2d(xd, wd, stride=lay.stride, padding=lay.pad, output_padding=lay.output_padding)) \
    if lay.transposed else (lambda: F.conv2d(xd, wd, stride=lay.stride, padding=lay.pad, dilation=lay.dilation))
for _ in range(5):
    fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", lay.name)
