"""GPU parity: every ABI call against the fp64 oracle on the same seeded inputs.

Bars (BASELINE north_star):
  integer mode (X, W in [-4, 4])  -> bit-exact (fp32 accumulation is exact, < 2^24)
  bf16 random                            -> max|err| <= 1e-2 * max|ref|
  TF32 random                            -> max|err| <= 2e-3 * max|ref|
  pure-indexing eOperators / weight DLT  -> bit-exact
"""
import numpy as np
import pytest
import torch

import oracle
import ollie_synth as syn
from tests import eop_cases as ec

pytestmark = pytest.mark.gpu

TOL = {"bf16": 1e-2, "tf32": 2e-3}


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


def _dev(t):
    return t.contiguous().cuda()


def _max_rel(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-30))


def _run_layer(O, lay, x, w, plan):
    from paper_2208_02025_b200 import DerivedConv
    conv = DerivedConv.from_layer(lay, plan=plan)
    conv.prepare(_dev(w))
    try:
        y = conv(_dev(x))
    except O.OllieError as e:
        if plan in (O.PLAN_FUSED, O.PLAN_GEMM_RED) and e.status == O.E_UNSUPPORTED:
            pytest.skip("no fused plan for this layer")
        raise
    torch.cuda.synchronize()
    return y.float().cpu().numpy()


def _oracle_layer(lay, x, w):
    if lay.transposed:
        return oracle.conv_transpose2d(x, w, lay.pad, lay.stride, lay.dilation, lay.output_padding)
    return oracle.conv2d(x, w, lay.pad, lay.stride, lay.dilation)


def _round_like(ref, dtype):
    """The GPU stores bf16 Y by RNE from the fp32 sum; compare the same decision."""
    if dtype == "bf16":
        return torch.from_numpy(ref).float().to(torch.bfloat16).float().numpy()
    return ref.astype(np.float32).astype(np.float64)


# --------------------------------------------------------------------- merged GEMM (a2)
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 200, 136), (49, 4608, 512), (1000, 48, 16),
                                   (2048, 576, 64), (5, 16, 8), (777, 1400, 8)])
def test_merged_gemm(O, dtype, M, N, K):
    if dtype == "bf16" and K % 8:
        pytest.skip("bf16 rows need K % 8 == 0")
    a = syn.integers((M, K), 7 + M, dtype)
    b = syn.integers((N, K), 8 + N, dtype)
    ldT = (N + 3) // 4 * 4
    T = torch.full((M, ldT), float("nan"), device="cuda")
    O.merged_gemm(M, N, K, O.BF16 if dtype == "bf16" else O.TF32, _dev(a), _dev(b), T, ldT)
    torch.cuda.synchronize()
    got = T[:, :N].cpu().numpy()
    assert np.array_equal(got, oracle.gemm_nt(a, b))          # integer mode: exact
    ar = syn.uniform((M, K), 9 + M, dtype)
    br = syn.uniform((N, K), 10 + N, dtype)
    O.merged_gemm(M, N, K, O.BF16 if dtype == "bf16" else O.TF32, _dev(ar), _dev(br), T, ldT)
    torch.cuda.synchronize()
    assert _max_rel(T[:, :N].cpu().numpy(), oracle.gemm_nt(ar, br)) <= TOL[dtype]


# --------------------------------------------------------------------- weight DLT (a0)
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("transposed", [False, True])
def test_weight_dlt_bit_exact(O, dtype, transposed):
    f, c, r, s = 37, 40, 3, 5
    shp = O.conv_shape(1, c, 8, 8, f, r, s, 1)
    w = syn.uniform((c, f, r, s) if transposed else (f, c, r, s), 3, dtype)
    wp = torch.empty(r * s * f, c, dtype=syn.torch_dtype(dtype), device="cuda")
    (O.prepare_weight_convtranspose2d if transposed else O.prepare_weight_conv2d)(
        shp, O.BF16 if dtype == "bf16" else O.TF32, _dev(w), wp)
    torch.cuda.synchronize()
    want = (oracle.weight_dlt_convt if transposed else oracle.weight_dlt_conv2d)(w)
    assert np.array_equal(wp.float().cpu().numpy().astype(np.float64), want)


# --------------------------------------------------------------------- OffsetAdd / selective add (a3/a4)
@pytest.mark.parametrize("ydt", ["bf16", "fp32"])
@pytest.mark.parametrize("n,h,w,f,r,s,pad,st,dil,tr,op", [
    (2, 7, 9, 64, 3, 3, 1, 1, 1, False, 0), (1, 8, 8, 3, 3, 3, 1, 1, 1, False, 0),
    (1, 9, 7, 4, 3, 3, 2, 1, 2, False, 0), (1, 11, 10, 8, 3, 3, 1, 2, 1, False, 0),
    (2, 5, 5, 1, 5, 5, 2, 1, 1, False, 0), (2, 3, 3, 12, 4, 4, 1, 2, 1, True, 0),
    (1, 6, 5, 1, 9, 9, 4, 2, 1, True, 1), (1, 4, 4, 3, 4, 4, 1, 2, 1, True, 0)])
def test_offset_add_standalone(O, ydt, n, h, w, f, r, s, pad, st, dil, tr, op):
    nt = r * s * f
    ldT = (nt + 3) // 4 * 4
    T = syn.integers((n * h * w, ldT), 5 + f, "tf32")
    shp = O.conv_shape(n, 1, h, w, f, r, s, pad, st, dil, op)
    oh, ow = O.output_hw(shp, tr)
    y = torch.empty(n, oh, ow, f, dtype=torch.bfloat16 if ydt == "bf16" else torch.float32, device="cuda")
    O.offset_add(shp, tr, _dev(T), ldT, O.BF16 if ydt == "bf16" else O.FP32, y)
    torch.cuda.synchronize()
    Td = T[:, :nt].double().numpy()
    want = (oracle.selective_add(Td, n, h, w, f, r, s, pad, st, dil, op) if tr
            else oracle.offset_add(Td, n, h, w, f, r, s, pad, st, dil))
    assert np.array_equal(y.float().cpu().numpy(), _round_like(want, "bf16" if ydt == "bf16" else "tf32"))


# --------------------------------------------------------------------- derived layers (a0-a4, unfused / auto)
SMALL = [
    syn.Layer("motivating", 1, 4, 8, 8, 4, 3, 3, pad=1, dtype="tf32"),              # c=4 fp32 = 16-byte rows
    syn.Layer("r18_64_tiny", 2, 64, 12, 13, 64, 3, 3, pad=1),
    syn.Layer("r18_s2", 1, 64, 14, 14, 128, 3, 3, pad=1, stride=2),
    syn.Layer("csr_dil", 1, 32, 16, 16, 40, 3, 3, pad=2, dilation=2),
    syn.Layer("one_by_one", 2, 56, 9, 9, 12, 1, 1, pad=0),
    syn.Layer("fsr_5x5", 1, 8, 17, 15, 56, 5, 5, pad=2),
    syn.Layer("f3", 1, 16, 8, 8, 3, 3, 3, pad=1),
    syn.Layer("convt_4x4", 2, 64, 3, 3, 48, 4, 4, pad=1, stride=2, transposed=True),
    syn.Layer("convt_9x9", 1, 56, 6, 5, 1, 9, 9, pad=4, stride=2, output_padding=1, transposed=True),
    syn.Layer("convt_tf32", 1, 32, 4, 4, 20, 4, 4, pad=1, stride=2, transposed=True, dtype="tf32"),
    syn.Layer("convt_1x1", 1, 16, 5, 5, 8, 1, 1, transposed=True),
    syn.Layer("r18_7x7_multi", 3, 512, 7, 7, 512, 3, 3, pad=1),
    syn.Layer("wide_cols", 1, 16, 5, 300, 24, 3, 3, pad=1),
    syn.Layer("tall_f_tail", 2, 40, 9, 11, 200, 3, 3, pad=0),
    syn.Layer("dil2_wide", 1, 64, 20, 70, 64, 3, 3, pad=2, dilation=2),
    syn.Layer("k5_c8", 2, 8, 19, 23, 56, 5, 5, pad=2),
    syn.Layer("tf32_fused", 2, 36, 13, 9, 40, 3, 3, pad=1, dtype="tf32"),
]


@pytest.mark.parametrize("plan", [0, 1, 2, 3])
@pytest.mark.parametrize("lay", SMALL, ids=[l.name for l in SMALL])
def test_derived_layer_integer_exact(O, lay, plan):
    x, w = syn.layer_inputs(lay, 100, exact_int=True)
    got = _run_layer(O, lay, x, w, plan)
    ref = _oracle_layer(lay, x, w)
    assert got.shape == ref.shape
    assert np.array_equal(got, _round_like(ref, lay.dtype))


@pytest.mark.parametrize("plan", [0, 1, 2, 3])
@pytest.mark.parametrize("lay", SMALL, ids=[l.name for l in SMALL])
def test_derived_layer_random_tolerance(O, lay, plan):
    x, w = syn.layer_inputs(lay, 200)
    got = _run_layer(O, lay, x, w, plan)
    assert _max_rel(got, _oracle_layer(lay, x, w)) <= TOL[lay.dtype]


# NEXT-2: strided Conv2d on the fused path (input-phase split, TMA element strides): zero-waste
STRIDED = [
    syn.Layer("s2_3x3_p1", 2, 64, 14, 14, 128, 3, 3, pad=1, stride=2),
    syn.Layer("s2_3x3_odd", 1, 64, 15, 13, 64, 3, 3, pad=1, stride=2),
    syn.Layer("s2_1x1_down", 2, 64, 14, 14, 128, 1, 1, pad=0, stride=2),
    syn.Layer("s2_5x5_p2", 1, 32, 17, 19, 48, 5, 5, pad=2, stride=2),
    syn.Layer("s3_3x3", 1, 64, 20, 23, 32, 3, 3, pad=1, stride=3),
    syn.Layer("s2_dil2", 1, 64, 16, 16, 64, 3, 3, pad=2, stride=2, dilation=2),
    syn.Layer("s2_planar_c16", 2, 16, 21, 18, 40, 3, 3, pad=1, stride=2),
    syn.Layer("s2_tf32", 1, 36, 12, 10, 24, 3, 3, pad=1, stride=2, dtype="tf32"),
    syn.Layer("s2_7x7_p3_c8", 1, 8, 32, 30, 64, 7, 7, pad=3, stride=2),
    syn.Layer("s2_big_c256", 2, 256, 14, 14, 512, 3, 3, pad=1, stride=2),
]


@pytest.mark.parametrize("lay", STRIDED, ids=[l.name for l in STRIDED])
def test_strided_fused_integer_exact(O, lay):
    x, w = syn.layer_inputs(lay, 400, exact_int=True)
    got = _run_layer(O, lay, x, w, O.PLAN_FUSED)
    ref = _oracle_layer(lay, x, w)
    assert got.shape == ref.shape
    assert np.array_equal(got, _round_like(ref, lay.dtype))


@pytest.mark.parametrize("lay", STRIDED, ids=[l.name for l in STRIDED])
def test_strided_fused_random_tolerance(O, lay):
    x, w = syn.layer_inputs(lay, 401)
    got = _run_layer(O, lay, x, w, O.PLAN_FUSED)
    assert _max_rel(got, _oracle_layer(lay, x, w)) <= TOL[lay.dtype]


def _configured():
    out = []
    for name in ("motivating", "resnet18", "resnet18_s2", "csrnet", "infogan", "infogan_tf32", "dcgan",
                 "paper_conv3x3"):
        for i, lay in enumerate(syn.CONFIGS[name]):
            out.append((name, i, lay))
    return out


@pytest.mark.parametrize("name,i,lay", _configured(), ids=[l.name for _, _, l in _configured()])
def test_configured_layers_full_size_sampled(O, name, i, lay):
    """Full BASELINE sizes, launch config of the bench; the oracle checks a sample of images."""
    if lay.c * (2 if lay.dtype == "bf16" else 4) % 16:
        pytest.skip("needs channel padding (covered by the FSRCNN stack test)")
    x, w = syn.layer_inputs(lay, syn.config_seed(name, i))
    got = _run_layer(O, lay, x, w, 0)
    budget = 2e9                                                   # oracle flop budget per test
    per_img = lay.useful_flops / lay.n
    k = max(1, min(lay.n, int(budget // per_img)))
    step = -(-lay.n // k)
    idx = list(range(0, lay.n, step))
    ref = _oracle_layer(lay, x[idx], w)
    assert _max_rel(got[idx], ref) <= TOL[lay.dtype]


# --------------------------------------------------------------------- eOperators (a5-a7)
def _eop_case(spec, arrays, out_dtype="fp32", in_dtype="fp32"):
    return spec, arrays, out_dtype, in_dtype


EOPS = {
    "transpose": lambda: (ec.transpose_nchw_to_nhwc(2, 37, 9, 11), [(2, 37, 9, 11)]),
    "layout_a_identity": lambda: (ec.layout_a(7, 9, 16), [(7, 9, 16)]),
    "channel_pad": lambda: (ec.channel_pad(2, 9, 10, 3, 8), [(2, 9, 10, 3)]),
    "offset_add": lambda: (ec.offset_add(2, 7, 6, 5, 3, 3, 1), [(2, 7, 6, 45)]),
    "offset_add_dil_stride": lambda: (ec.offset_add(1, 9, 8, 3, 3, 3, 2, 2, 2), [(1, 9, 8, 27)]),
    "selective_add": lambda: (ec.selective_add(2, 3, 4, 3, 4, 4, 1, 2), [(2, 3, 4, 4, 4, 3)]),
    "selective_add_9x9": lambda: (ec.selective_add(1, 4, 3, 1, 9, 9, 4, 2, 1), [(1, 4, 3, 9, 9, 1)]),
    "fused_pair": lambda: (ec.fused_pad_then_offset_add(1, 5, 6, 2, 3, 3, 1, 3), [(1, 5, 6, 18)]),
    "affine_mix": lambda: (ec.affine_mix(2, 3, 5, 6), [(2, 3, 5, 6), (5, 6)]),
    # fast paths: tiled transpose (inner output dim strided in the input) and affine gather
    "transpose_big": lambda: (ec.transpose_nchw_to_nhwc(2, 70, 33, 45), [(2, 70, 33, 45)]),
    # 16-byte transpose path (bf16, every dim a multiple of 8, partial 64 x 64 tiles)
    "transpose_v16": lambda: (ec.transpose_nchw_to_nhwc(2, 72, 16, 40), [(2, 72, 16, 40)]),
    "transpose_v16_partial": lambda: (ec.transpose_nchw_to_nhwc(1, 136, 24, 104), [(1, 136, 24, 104)]),
    # 64 x 128 tiles (c a multiple of 128), dt partial
    "transpose_v16_wide": lambda: (ec.transpose_nchw_to_nhwc(2, 256, 6, 24), [(2, 256, 6, 24)]),
    "transpose_v16_wide2": lambda: (ec.transpose_nchw_to_nhwc(1, 384, 3, 72), [(1, 384, 3, 72)]),
    "channel_pad_big": lambda: (ec.channel_pad(3, 17, 40, 12, 16), [(3, 17, 40, 12)]),
    "flip_pad": lambda: ({"inputs": [{"shape": [5, 37], "pad": [[2, 1], [0, 3]]}],
                          "scopes": [{"trav": [[0, 8], [0, 40]], "sum": [],
                                      "access": [{"tensor": 0, "index": [ec.idx(ec.I(0, -1), const=5),
                                                                         ec.idx(ec.I(1))]}],
                                      "body": [["acc", 0]]}]}, [(5, 37)]),
}


@pytest.mark.parametrize("dt", ["fp32", "bf16"])
@pytest.mark.parametrize("case", sorted(EOPS))
def test_eop_eval_vs_interpreter(O, case, dt):
    spec, shapes = EOPS[case]()
    arrays = [syn.integers(s, 40 + k, "bf16" if dt == "bf16" else "tf32") for k, s in enumerate(shapes)]
    code = O.BF16 if dt == "bf16" else O.FP32
    e = O.make_eop(spec, [code] * len(arrays), code)
    info = O.eop_analyze(e)
    assert info["is_identity"] == oracle.eop_is_identity(spec)
    want = oracle.eop_eval(spec, [a.double().numpy() for a in arrays])
    outs = torch.full(want.shape, -7.0, dtype=arrays[0].dtype, device="cuda")
    ins = [_dev(a) for a in arrays]
    O.eop_eval(e, ins, outs)
    torch.cuda.synchronize()
    got = outs.float().cpu().numpy().astype(np.float64)
    assert np.array_equal(got, _round_like(want, "bf16" if dt == "bf16" else "tf32"))


def test_eop_identity_aliased_launches_nothing(O):
    spec = ec.layout_a(4, 5, 8)
    e = O.make_eop(spec, [O.FP32], O.FP32)
    x = torch.arange(160, dtype=torch.float32, device="cuda")
    O.eop_eval(e, [x], x)          # aliased identity: no launch, unchanged
    assert torch.equal(x.cpu(), torch.arange(160, dtype=torch.float32))


def test_errors_are_statuses(O):
    shp = O.conv_shape(1, 12, 8, 8, 4, 3, 3, 1)         # c=12 bf16 -> 24-byte rows
    x = torch.zeros(1, 8, 8, 12, dtype=torch.bfloat16, device="cuda")
    wp = torch.zeros(36, 12, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(1, 8, 8, 4, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(O.OllieError) as ei:
        O.conv2d_derived(shp, O.BF16, x, wp, y, None, 0, O.PLAN_UNFUSED)
    assert ei.value.status == O.E_ALIGN
    shp = O.conv_shape(1, 16, 8, 8, 4, 3, 3, 1)
    x = torch.zeros(1, 8, 8, 16, dtype=torch.bfloat16, device="cuda")
    wp = torch.zeros(36, 16, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(O.OllieError) as ei:
        O.conv2d_derived(shp, O.BF16, x, wp, y, None, 0, O.PLAN_UNFUSED)
    assert ei.value.status == O.E_WORKSPACE
