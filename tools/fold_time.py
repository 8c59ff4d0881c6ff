import sys, os
sys.path.insert(0, os.getcwd())
import torch
import ollie_synth as syn
from paper_2208_02025_b200 import ollie as O
from paper_2208_02025_b200.stack import DerivedStack
lay = syn.CONFIGS["fsrcnn"][0]
st = DerivedStack([lay], False)
sl = st.layers[0]
x, w = syn.layer_inputs(lay, 3)
st.prepare([w.cuda()]); xd = x.cuda()
st([xd]); torch.cuda.synchronize()
def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n
print("fold eOp us", t(lambda: O.tap_fold(sl.fold_shape, sl.conv.code, xd, sl.kp, sl.x_fold)))
print("1x1 conv us", t(lambda: sl.conv(sl.x_fold, sl.y)), O.plan_describe(sl.conv.shape, sl.conv.code, sl.conv.plan, False))
for p in (O.PLAN_FUSED, O.PLAN_UNFUSED, O.PLAN_ROWSTREAM):
    try:
        print(p, "us", t(lambda: O.conv2d_derived(sl.conv.shape, sl.conv.code, sl.x_fold, sl.conv.w_prep, sl.y, sl.conv.ws, sl.conv.ws_bytes, p)))
    except Exception as e: print(p, e)
print("x_fold.zero_() us", t(lambda: sl.x_fold.zero_()), "bytes", sl.x_fold.numel() * 2)
big = torch.empty(sl.x_fold.numel(), dtype=torch.bfloat16, device="cuda")
print("fresh buffer zero_() us", t(lambda: big.zero_()))
print("fresh buffer fill_(1) us", t(lambda: big.fill_(1.0)))
src = torch.randn(sl.x_fold.numel() // 2, device="cuda")
print("copy 134MB->134MB us", t(lambda: big.view(torch.float32).copy_(src)))
