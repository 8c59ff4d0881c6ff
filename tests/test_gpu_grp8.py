"""GPU parity of the fused kernel's two lane layouts (FusedArgs::grp8): 128 consecutive patch rows
(halo columns idle) vs 16 groups of 8 rows at a stride of Xb patch rows (every lane an output,
XB <= 8).  The debug hook ollie_debug_force_grp8 restricts the planner to one layout, so every
SMALL / STRIDED layer of test_gpu_parity.py, CTA pairs, split-K and multi-image tiles run in both
and are compared with the fp64 oracle: bit-exact in integer mode, within the bars on random data."""
import numpy as np
import pytest
import torch

import ollie_synth as syn
from tests.test_gpu_parity import SMALL, STRIDED, TOL, _dev, _max_rel, _oracle_layer, _round_like

pytestmark = pytest.mark.gpu

EXTRA = [
    syn.Layer("csr_like_64", 2, 64, 32, 32, 64, 3, 3, pad=2, dilation=2),
    syn.Layer("w_not_mult8", 2, 64, 19, 13, 48, 3, 3, pad=1),
    syn.Layer("tiny_img_ipt", 6, 64, 5, 5, 64, 3, 3, pad=1),
    syn.Layer("convt_8x8", 3, 64, 8, 8, 32, 4, 4, pad=1, stride=2, transposed=True),
    syn.Layer("planar_c16_grp", 2, 16, 30, 27, 32, 3, 3, pad=1),
]
LAYERS = SMALL + STRIDED + EXTRA


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


@pytest.fixture(params=[0, 1], ids=["rows", "grp8"])
def layout(O, request):
    O._lib.ollie_debug_force_grp8(request.param)
    yield request.param
    O._lib.ollie_debug_force_grp8(-1)
    O._lib.ollie_debug_force_pair(-1)
    O._lib.ollie_debug_force_ksplit(-1)


def _run(O, lay, x, w, layout):
    from paper_2208_02025_b200 import DerivedConv
    conv = DerivedConv.from_layer(lay, plan=O.PLAN_FUSED)
    conv.prepare(_dev(w))
    try:
        y = conv(_dev(x))
    except O.OllieError as e:
        if e.status == O.E_UNSUPPORTED:
            pytest.skip("no fused plan in this lane layout")
        raise
    torch.cuda.synchronize()
    desc = O.plan_describe(conv.shape, conv.code, O.PLAN_FUSED, conv.transposed)
    assert f"grp8={layout}" in desc, desc
    return y.float().cpu().numpy()


@pytest.mark.parametrize("lay", LAYERS, ids=[l.name for l in LAYERS])
def test_layout_integer_exact(O, layout, lay):
    x, w = syn.layer_inputs(lay, 600, exact_int=True)
    got = _run(O, lay, x, w, layout)
    assert np.array_equal(got, _round_like(_oracle_layer(lay, x, w), lay.dtype))


@pytest.mark.parametrize("lay", LAYERS, ids=[l.name for l in LAYERS])
def test_layout_random_tolerance(O, layout, lay):
    x, w = syn.layer_inputs(lay, 601)
    got = _run(O, lay, x, w, layout)
    assert _max_rel(got, _oracle_layer(lay, x, w)) <= TOL[lay.dtype]


@pytest.mark.parametrize("mode", ["pair", "ks2", "ks4"])
@pytest.mark.parametrize("lay", EXTRA[:3] + [SMALL[11]], ids=[l.name for l in EXTRA[:3]] + [SMALL[11].name])
def test_layout_with_pairs_and_splitk(O, layout, lay, mode):
    if mode == "pair":
        O._lib.ollie_debug_force_pair(1)
    else:
        O._lib.ollie_debug_force_pair(0)
        O._lib.ollie_debug_force_ksplit(int(mode[2:]))
    x, w = syn.layer_inputs(lay, 602, exact_int=True)
    got = _run(O, lay, x, w, layout)
    assert np.array_equal(got, _round_like(_oracle_layer(lay, x, w), lay.dtype))
