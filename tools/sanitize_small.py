"""Small configs through every ABI path, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ollie_synth as syn
STAGE = os.environ.get("SAN_STAGE", "all")
from paper_2208_02025_b200 import ollie as O, eops
from paper_2208_02025_b200.layers import DerivedConv
from tests import eop_cases as ec

layers = [syn.Layer("c", 2, 64, 9, 11, 64, 3, 3, pad=1), syn.Layer("t", 2, 64, 3, 3, 48, 4, 4, pad=1, stride=2, transposed=True),
          syn.Layer("d", 1, 32, 12, 12, 40, 3, 3, pad=2, dilation=2), syn.Layer("k", 1, 8, 9, 7, 24, 5, 5, pad=2),
          syn.Layer("o", 2, 16, 5, 5, 8, 1, 1)]
for lay in layers:
    x, w = syn.layer_inputs(lay, 3)
    for plan in (O.PLAN_FUSED, O.PLAN_UNFUSED):
        try:
            conv = DerivedConv.from_layer(lay, plan=plan, autotune=False).prepare(w.cuda())
            conv(x.cuda())
        except O.OllieError as e:
            if e.status != O.E_UNSUPPORTED:
                raise
# merged GEMM: TMA-store epilogue (BN % 32 == 0, M tail), narrow-N small-M tiles, row-store fallback
for M, N, K in ((777, 1024, 64), (49, 4608, 128), (300, 200, 136)):
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    ldT = (N + 3) // 4 * 4
    T = torch.empty(M, ldT, device="cuda")
    O.merged_gemm(M, N, K, O.BF16, a, b, T, ldT)
for spec, shapes in ((ec.transpose_nchw_to_nhwc(2, 33, 5, 7), [(2, 33, 5, 7)]),
                     (ec.channel_pad(2, 5, 6, 3, 8), [(2, 5, 6, 3)]),
                     (ec.fused_pad_then_offset_add(1, 4, 5, 2, 3, 3, 1, 3), [(1, 4, 5, 18)])):
    e = O.make_eop(spec, [O.FP32] * len(shapes), O.FP32)
    ins = [torch.randn(s, device="cuda") for s in shapes]
    out = torch.empty([hi - lo for lo, hi in spec["scopes"][0]["trav"]], device="cuda")
    O.eop_eval(e, ins, out)
# CTA pairs, split-K clusters, strided phases, the NEXT-3 epilogue
lay = syn.Layer("p", 2, 256, 14, 14, 128, 3, 3, pad=1)
x, w = syn.layer_inputs(lay, 4)
for pair, ks in (((1, -1),) if STAGE in ("all", "pair") else ()) + (((0, 2), (0, 4)) if STAGE != "pair" else ()):
    O._lib.ollie_debug_force_pair(pair)
    O._lib.ollie_debug_force_ksplit(ks)
    try:
        conv = DerivedConv.from_layer(lay, plan=O.PLAN_FUSED, autotune=False).prepare(w.cuda())
        conv(x.cuda(), bias=torch.randn(lay.f, device="cuda"), residual=torch.randn(lay.n, lay.oh, lay.ow, lay.f, device="cuda").bfloat16(), act=O.ACT_PRELU, alpha=torch.rand(lay.f, device="cuda"))
        torch.cuda.synchronize()
        print("ran pair", pair, "ks", ks, O.plan_describe(conv.shape, conv.code, O.PLAN_FUSED, False)[-40:], flush=True)
    except O.OllieError as e:
        if e.status != O.E_UNSUPPORTED:
            raise
        print("no plan for pair", pair, "ks", ks, flush=True)
O._lib.ollie_debug_force_pair(-1)
O._lib.ollie_debug_force_ksplit(-1)
lay = syn.Layer("s", 1, 64, 13, 11, 64, 3, 3, pad=1, stride=2)
x, w = syn.layer_inputs(lay, 5)
DerivedConv.from_layer(lay, plan=O.PLAN_FUSED, autotune=False).prepare(w.cuda())(x.cuda())
# multi-image tiles (ipt 2 / 3; ragged batch, split-K, strided phases, ConvT classes)
for lay, ipt, ks in ((syn.Layer("i7", 3, 64, 7, 7, 64, 3, 3, pad=1), 2, -1),
                     (syn.Layer("i7k", 3, 128, 7, 7, 64, 3, 3, pad=1), 2, 2),
                     (syn.Layer("is2", 3, 64, 10, 10, 64, 3, 3, pad=1, stride=2), 3, -1),
                     (syn.Layer("it", 3, 64, 4, 4, 32, 4, 4, pad=1, stride=2, transposed=True), 2, -1)):
    O._lib.ollie_debug_force_ipt(ipt)
    O._lib.ollie_debug_force_ksplit(ks)
    x, w = syn.layer_inputs(lay, 8)
    try:
        conv = DerivedConv.from_layer(lay, plan=O.PLAN_FUSED, autotune=False).prepare(w.cuda())
        conv(x.cuda())
        torch.cuda.synchronize()
        print("ran", lay.name, O.plan_describe(conv.shape, conv.code, O.PLAN_FUSED, lay.transposed)[-30:], flush=True)
    except O.OllieError as e:
        if e.status != O.E_UNSUPPORTED:
            raise
O._lib.ollie_debug_force_ipt(0)
O._lib.ollie_debug_force_ksplit(-1)
# NEXT-1 and NEXT-4
from paper_2208_02025_b200 import DilatedAsDense
lay = syn.Layer("dd", 1, 16, 10, 12, 16, 3, 3, pad=2, dilation=2)
x, w = syn.layer_inputs(lay, 6)
DilatedAsDense(1, 16, 10, 12, 16, 3, 3, 2, 2, plan=O.PLAN_FUSED).prepare(w.cuda())(x.cuda())
for form in (0, 1):
    g = syn.G2("g", 1, 300, 64, 20, 3)
    a, b = syn.g2bmm_inputs(g, 7)
    for ldo in (41, 48):
        out = torch.empty(1, 300, ldo, dtype=torch.bfloat16, device="cuda")
        O.g2bmm(1, 300, 64, 20, 3, O.BF16, a.cuda(), b.cuda(), out, ldo, form)
# round 2: row-streaming (ysum / direct, Conv2d and a sub-pixel ConvT; a 1x1 pad-1 layer whose bottom
# output row reads no input row), grp8 lanes, the tap-fold eOperator, the 2x2 selective-add fast path
for lay, plans in ((syn.Layer("rs3", 2, 16, 6, 20, 12, 3, 3, pad=1), (O.PLAN_ROWSTREAM_YSUM, O.PLAN_ROWSTREAM_DIRECT)),
                   (syn.Layer("rs1p", 3, 64, 5, 19, 8, 1, 1, pad=1), (O.PLAN_ROWSTREAM_YSUM, O.PLAN_ROWSTREAM_DIRECT)),
                   (syn.Layer("rst", 1, 64, 5, 9, 1, 9, 9, pad=4, stride=2, output_padding=1, transposed=True),
                    (O.PLAN_ROWSTREAM,))):
    x, w = syn.layer_inputs(lay, 9)
    for plan in plans:
        try:
            DerivedConv.from_layer(lay, plan=plan, autotune=False).prepare(w.cuda())(x.cuda())
            torch.cuda.synchronize()
            print("ran rowstream", lay.name, plan, flush=True)
        except O.OllieError as e:
            if e.status != O.E_UNSUPPORTED:
                raise
O._lib.ollie_debug_force_grp8(1)
lay = syn.Layer("g8", 2, 64, 10, 13, 64, 3, 3, pad=2, dilation=2)
x, w = syn.layer_inputs(lay, 10)
DerivedConv.from_layer(lay, plan=O.PLAN_FUSED, autotune=False).prepare(w.cuda())(x.cuda())
O._lib.ollie_debug_force_grp8(-1)
for (n, h, w_, c, r, s_, pad, st, kp) in ((2, 7, 16, 1, 5, 5, 2, 1, 32), (1, 6, 9, 3, 3, 3, 1, 2, 32)):
    shp = O.conv_shape(n, c, h, w_, 1, r, s_, pad, st)
    oh, ow = O.output_hw(shp, False)
    xx = torch.randn(n, h, w_, c, device="cuda").to(torch.bfloat16)
    out = torch.empty(n, oh, ow, kp, dtype=torch.bfloat16, device="cuda")
    O.tap_fold(shp, O.BF16, xx, kp, out)
shp = O.conv_shape(2, 32, 5, 6, 16, 4, 4, 1, 2)
T = torch.randn(2 * 5 * 6, 4 * 4 * 16, device="cuda")
Y = torch.empty(2, 10, 12, 16, device="cuda", dtype=torch.bfloat16)
O.offset_add(shp, True, T, 4 * 4 * 16, O.BF16, Y)
torch.cuda.synchronize()
print("sanitize run ok")
