"""GPU parity of the row-streaming plan (OLLIE_PLAN_ROWSTREAM, rowstream_conv.cuh): kernel rows
(and a ConvTranspose2d's output residue classes) on the MMA's N, kernel columns as A-row shifts, the
row OffsetAdd over the TMEM accumulators of consecutive input rows in the epilogue -- against the
fp64 oracle's direct Conv2d / scatter-form ConvTranspose2d.

Both forms of the kernel run every case they plan: "ysum" (kernel rows on N, the row OffsetAdd in
the epilogue) and "direct" (N = f, all r*s taps as A-row shifts, one accumulator per output row;
Conv2d only, which also takes the wide-f 1x1 / 3x3 layers of RS_DIRECT_LAYERS).

Integer mode is bit-exact; random data meets the bf16 / TF32 bars.  The shapes cover image
rows over several 128-pixel M-tiles (w up to 300, two TMA boxes per row), ragged widths, every
kernel-variant width (stride^2 * f = 4, 8, 12, 16), 32/64/128-byte pixel rows (c = 8..64 bf16,
8..16 fp32), batches whose row runs split images across CTAs, and a layer too wide for the plan
(UNSUPPORTED, not a wrong answer).
"""
import numpy as np
import pytest
import torch

import oracle
import ollie_synth as syn
from tests.test_gpu_parity import TOL, _dev, _max_rel, _oracle_layer, _round_like

pytestmark = pytest.mark.gpu

L = syn.Layer
RS_LAYERS = [
    L("rs_map_3x3_16", 2, 16, 9, 250, 16, 3, 3, pad=1),                     # FSRCNN map, 2 M-tiles, ragged
    L("rs_map_f12", 1, 16, 7, 37, 12, 3, 3, pad=1),                          # f = 12 (Fp 12), narrow rows
    L("rs_5x5_c8", 2, 8, 11, 100, 8, 5, 5, pad=2),                           # 16-byte pixels in 32-byte rows
    L("rs_c64_f4", 3, 64, 6, 129, 4, 3, 3, pad=1),                           # 128-byte rows, ragged w
    L("rs_nopad", 1, 32, 10, 140, 16, 3, 3, pad=0),                          # OW < W
    L("rs_bigpad", 1, 16, 5, 20, 8, 3, 3, pad=2),                            # OW > W, rows of zero taps
    L("rs_deconv_9x9", 2, 56, 13, 140, 1, 9, 9, pad=4, stride=2, output_padding=1, transposed=True),  # FSRCNN deconv
    L("rs_dcgan_64to3", 2, 64, 8, 8, 3, 4, 4, pad=1, stride=2, transposed=True),                      # DCGAN last layer
    L("rs_convt_f4", 1, 32, 6, 7, 4, 4, 4, pad=1, stride=2, transposed=True),                         # Fp 16, N 48
    L("rs_convt_3x3", 2, 16, 5, 9, 2, 3, 3, pad=1, stride=2, output_padding=1, transposed=True),       # Fp 8
    L("rs_convt_s1", 1, 16, 9, 33, 8, 3, 3, pad=1, stride=1, transposed=True),                        # sigma 1
    L("rs_tf32_conv", 2, 16, 6, 150, 8, 3, 3, pad=1, dtype="tf32"),          # 64-byte rows, fp32 Y
    L("rs_w300_f4", 1, 16, 5, 300, 4, 3, 3, pad=1),                         # 3 M-tiles, two TMA boxes per row
    L("rs_tf32_deconv", 1, 8, 7, 20, 1, 9, 9, pad=4, stride=2, output_padding=1, transposed=True, dtype="tf32"),
    L("rs_many_rows", 37, 16, 11, 16, 16, 3, 3, pad=1),                      # 407 rows: runs cross images
]
# shapes only the direct form (N = f, all r*s taps as A shifts) plans
RS_DIRECT_LAYERS = [
    L("rd_1x1_12to56", 2, 16, 7, 200, 56, 1, 1),                             # FSRCNN expand (c padded 12 -> 16)
    L("rd_1x1_56to12", 1, 56, 9, 150, 12, 1, 1),                             # FSRCNN shrink, 112-byte pixels
    L("rd_3x3_c64_f64", 1, 64, 6, 130, 64, 3, 3, pad=1),                     # 4 K steps, 36 MMAs per M-tile
    L("rd_f3_odd", 2, 32, 5, 40, 3, 3, 3, pad=1),                            # f = 3: scalar stores
    L("rd_5x5_f24", 1, 16, 9, 70, 24, 5, 5, pad=2),                          # NP 32, 25 taps
    L("rd_w400_f16", 1, 8, 4, 400, 16, 3, 3, pad=1),                         # 4 M-tiles, 2 TMA boxes
    L("rd_tf32_1x1", 2, 16, 5, 129, 40, 1, 1, dtype="tf32"),
    L("rd_pad0_top", 3, 16, 4, 20, 16, 3, 3, pad=0),                         # OH < H: runs skip rows
]
FORMS = ["ysum", "direct"]


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


def _plan(O, form):
    return {"ysum": O.PLAN_ROWSTREAM_YSUM, "direct": O.PLAN_ROWSTREAM_DIRECT, "auto": O.PLAN_ROWSTREAM}[form]


def _plannable(O, lay, form):
    from paper_2208_02025_b200 import DerivedConv
    try:
        return DerivedConv.from_layer(lay, plan=_plan(O, form)).resolved_plan() == "rowstream"
    except O.OllieError:
        return False


def _run(O, lay, x, w, form="auto", **epi):
    from paper_2208_02025_b200 import DerivedConv
    conv = DerivedConv.from_layer(lay, plan=_plan(O, form))
    assert conv.resolved_plan() == "rowstream"
    conv.prepare(_dev(w))
    y = torch.full(conv.out_shape(), float("nan"), dtype=syn.torch_dtype(lay.dtype), device="cuda")
    conv(_dev(x), y, None, **epi)
    torch.cuda.synchronize()
    return y.float().cpu().numpy()


ALL = RS_LAYERS + RS_DIRECT_LAYERS


@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("lay", ALL, ids=[l.name for l in ALL])
def test_rowstream_integer_exact(O, lay, form):
    if not _plannable(O, lay, form):
        pytest.skip(f"{form} form does not plan {lay.name}")
    x, w = syn.layer_inputs(lay, 300, exact_int=True)
    got = _run(O, lay, x, w, form)
    assert np.array_equal(got, _round_like(_oracle_layer(lay, x, w), lay.dtype))


@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("lay", ALL, ids=[l.name for l in ALL])
def test_rowstream_random(O, lay, form):
    if not _plannable(O, lay, form):
        pytest.skip(f"{form} form does not plan {lay.name}")
    x, w = syn.layer_inputs(lay, 301)
    got = _run(O, lay, x, w, form)
    assert _max_rel(got, _oracle_layer(lay, x, w)) <= TOL[lay.dtype]


def test_rowstream_direct_covers_every_conv_case(O):
    """Every stride-1 Conv2d case of the table plans in the direct form too (so both forms are
    exercised on them), and the direct-only table is plannable direct."""
    for lay in ALL:
        if not lay.transposed:
            assert _plannable(O, lay, "direct"), lay.name


@pytest.mark.parametrize("name,form", [("rs_map_3x3_16", "ysum"), ("rs_map_3x3_16", "direct"), ("rs_deconv_9x9", "ysum"),
                                       ("rs_dcgan_64to3", "ysum"), ("rd_1x1_12to56", "direct"), ("rd_f3_odd", "direct")])
@pytest.mark.parametrize("act", [1, 2])
def test_rowstream_epilogue_exact(O, name, form, act):
    lay = next(l for l in ALL if l.name == name)
    x, w = syn.layer_inputs(lay, 302, exact_int=True)
    g = torch.Generator().manual_seed(5)
    bias = torch.randint(-8, 9, (lay.f,), generator=g).float()
    res = torch.randint(-4, 5, (lay.n, lay.oh, lay.ow, lay.f), generator=g).to(syn.torch_dtype(lay.dtype))
    alpha = torch.full((lay.f,), 0.25)
    got = _run(O, lay, x, w, form, bias=_dev(bias), residual=_dev(res), act=act, alpha=_dev(alpha))
    ref = oracle.epilogue(_oracle_layer(lay, x, w), bias.numpy(), res, "relu" if act == 1 else "prelu", alpha.numpy())
    assert np.array_equal(got, _round_like(ref, lay.dtype))


def test_rowstream_unsupported_is_a_status(O):
    from paper_2208_02025_b200 import DerivedConv
    lay = L("too_wide", 1, 64, 8, 8, 96, 3, 3, pad=1)        # f = 96 > 64 (either form)
    conv = DerivedConv.from_layer(lay, plan=O.PLAN_ROWSTREAM)
    x, w = syn.layer_inputs(lay, 303, exact_int=True)
    conv.prepare(_dev(w))
    with pytest.raises(O.OllieError) as ei:
        conv(_dev(x))
    assert ei.value.status == O.E_UNSUPPORTED
