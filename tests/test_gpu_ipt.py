"""GPU parity of multi-image fused tiles (ipt > 1): small images share one 128-lane tile, the patch
rows interleaved [y][image][x] by a {c, w, n, h} tensor-map view, so every tap stays one row
offset.  Forced with the debug hook ollie_debug_force_ipt (alone, with split-K and with CTA pairs)
and compared with the fp64 oracle: integer mode bit-exact, random data within the bf16 / TF32
bars.  Batches that are not a multiple of ipt exercise the zero-filled missing images."""
import numpy as np
import pytest

import ollie_synth as syn
from tests.test_gpu_parity import TOL, _dev, _max_rel, _oracle_layer, _round_like

pytestmark = pytest.mark.gpu

LAYERS = [
    syn.Layer("r18_512x7_b4", 4, 512, 7, 7, 512, 3, 3, pad=1),
    syn.Layer("c64_7x7_b5_ragged", 5, 64, 7, 7, 64, 3, 3, pad=1),
    syn.Layer("c64_6x5_b3", 3, 64, 6, 5, 48, 3, 3, pad=1),
    syn.Layer("s2_14to7_b3", 3, 128, 14, 14, 128, 3, 3, pad=1, stride=2),
    syn.Layer("dil2_8x8_b2", 2, 64, 8, 8, 64, 3, 3, pad=2, dilation=2),
    syn.Layer("convt_4to8_b3", 3, 128, 4, 4, 64, 4, 4, pad=1, stride=2, transposed=True),
    syn.Layer("c32_5x5k_b2", 2, 32, 6, 6, 32, 5, 5, pad=2),
    syn.Layer("tf32_7x7_b3", 3, 64, 7, 7, 32, 3, 3, pad=1, dtype="tf32"),
]
MODES = [(2, -1, -1), (3, -1, -1), (2, 2, -1), (2, -1, 1)]   # (ipt, split-K, pair)


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


@pytest.fixture
def force(O):
    def f(ipt, ks, pair):
        O._lib.ollie_debug_force_ipt(ipt)
        O._lib.ollie_debug_force_ksplit(ks)
        O._lib.ollie_debug_force_pair(pair)
    yield f
    f(0, -1, -1)


def _run(O, lay, x, w):
    from paper_2208_02025_b200 import DerivedConv
    conv = DerivedConv.from_layer(lay, plan=O.PLAN_FUSED)
    conv.prepare(_dev(w))
    try:
        y = conv(_dev(x))
    except O.OllieError as e:
        if e.status == O.E_UNSUPPORTED:
            pytest.skip("no plan with this image count per tile")
        raise
    d = O.plan_describe(conv.shape, conv.code, O.PLAN_FUSED, conv.transposed)
    return y.float().cpu().numpy(), d


@pytest.mark.parametrize("mode", MODES, ids=lambda m: f"ipt{m[0]}_ks{m[1]}_pair{m[2]}")
@pytest.mark.parametrize("lay", LAYERS, ids=lambda l: l.name)
def test_ipt_exact(O, force, lay, mode):
    ipt, ks, pair = mode
    if lay.n < ipt:
        pytest.skip("batch smaller than ipt")
    force(ipt, ks, pair)
    x, w = syn.layer_inputs(lay, 31, exact_int=True)
    got, d = _run(O, lay, x, w)
    assert f"ipt={ipt}" in d, d
    assert np.array_equal(got, _round_like(_oracle_layer(lay, x, w), lay.dtype)), d


# up to 16 images per tile (GAN inputs of 2x2 / 4x4 pixels): ragged batches, ConvT classes, both lane
# layouts, bit-exact in integer mode
BIG = [
    syn.Layer("convt_2to4_b17", 17, 64, 2, 2, 48, 4, 4, pad=1, stride=2, transposed=True),
    syn.Layer("convt_4to8_b9", 9, 64, 4, 4, 32, 4, 4, pad=1, stride=2, transposed=True),
    syn.Layer("c3_2x2_b16", 16, 64, 2, 2, 64, 3, 3, pad=1),
    syn.Layer("s2_4to2_b11", 11, 64, 4, 4, 64, 3, 3, pad=1, stride=2),
]


@pytest.mark.parametrize("ipt", [5, 8, 16])
@pytest.mark.parametrize("lay", BIG, ids=lambda l: l.name)
def test_ipt_many_images_exact(O, force, lay, ipt):
    if lay.n < ipt:
        pytest.skip("batch smaller than ipt")
    force(ipt, -1, -1)
    x, w = syn.layer_inputs(lay, 33, exact_int=True)
    got, d = _run(O, lay, x, w)
    assert f"ipt={ipt}" in d, d
    assert np.array_equal(got, _round_like(_oracle_layer(lay, x, w), lay.dtype)), d


@pytest.mark.parametrize("lay", LAYERS[:3] + LAYERS[-1:], ids=lambda l: l.name)
def test_ipt_random(O, force, lay):
    force(2, -1, -1)
    x, w = syn.layer_inputs(lay, 32)
    got, d = _run(O, lay, x, w)
    ref = _oracle_layer(lay, x, w)
    assert _max_rel(got, ref) <= TOL[lay.dtype], d
