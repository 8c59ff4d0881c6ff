"""GPU parity of the fused kernel's CTA-pair mode (cta_group::2, M = 256 MMAs issued by the
leader CTA of a 2-CTA cluster; each CTA holds its own input patch and half of every weight tile).

The debug hook ollie_debug_force_pair restricts the planner to pair plans (and
ollie_debug_force_plan to streamed / resident weights), so the same layers as
test_gpu_parity.py run through the pair path and are compared with the fp64 oracle:
bit-exact in integer mode, within the bf16 / TF32 bars on random data.
"""
import numpy as np
import pytest
import torch

import ollie_synth as syn
from tests.test_gpu_parity import SMALL, TOL, _dev, _max_rel, _oracle_layer, _round_like

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


@pytest.fixture
def pair_only(O):
    O._lib.ollie_debug_force_pair(1)
    yield
    O._lib.ollie_debug_force_pair(-1)
    O._lib.ollie_debug_force_plan(0, 0, -1)


def _run_pair(O, lay, x, w):
    from paper_2208_02025_b200 import DerivedConv
    conv = DerivedConv.from_layer(lay, plan=O.PLAN_FUSED)
    conv.prepare(_dev(w))
    try:
        y = conv(_dev(x))
    except O.OllieError as e:
        if e.status == O.E_UNSUPPORTED:
            pytest.skip("no pair plan for this layer")
        raise
    torch.cuda.synchronize()
    desc = O.plan_describe(conv.shape, conv.code, O.PLAN_FUSED, conv.transposed)
    assert "pair=1" in desc, desc
    return y.float().cpu().numpy()


@pytest.mark.parametrize("resident", [-1, 0, 1])
@pytest.mark.parametrize("lay", SMALL, ids=[l.name for l in SMALL])
def test_pair_integer_exact(O, pair_only, lay, resident):
    O._lib.ollie_debug_force_plan(0, 0, resident)
    x, w = syn.layer_inputs(lay, 100, exact_int=True)
    got = _run_pair(O, lay, x, w)
    assert np.array_equal(got, _round_like(_oracle_layer(lay, x, w), lay.dtype))


@pytest.mark.parametrize("lay", SMALL, ids=[l.name for l in SMALL])
def test_pair_random_tolerance(O, pair_only, lay):
    x, w = syn.layer_inputs(lay, 200)
    got = _run_pair(O, lay, x, w)
    assert _max_rel(got, _oracle_layer(lay, x, w)) <= TOL[lay.dtype]


# odd spatial-tile counts (the follower of the last pair has no tile) and multi-M-tile stacks
ODD = [
    syn.Layer("odd_tiles", 1, 64, 9, 9, 64, 3, 3, pad=1),
    syn.Layer("odd_mt", 3, 64, 23, 17, 96, 3, 3, pad=1),
    syn.Layer("convt_odd", 1, 64, 5, 3, 32, 4, 4, pad=1, stride=2, transposed=True),
]


@pytest.mark.parametrize("mt", [0, 1, 2])
@pytest.mark.parametrize("lay", ODD, ids=[l.name for l in ODD])
def test_pair_odd_and_stacked(O, pair_only, lay, mt):
    O._lib.ollie_debug_force_plan(mt, 0, -1)
    x, w = syn.layer_inputs(lay, 300, exact_int=True)
    got = _run_pair(O, lay, x, w)
    assert np.array_equal(got, _round_like(_oracle_layer(lay, x, w), lay.dtype))


@pytest.mark.parametrize("i", range(8))
def test_pair_resnet18_full_size_sampled(O, pair_only, i):
    lay = syn.CONFIGS["resnet18"][i]
    x, w = syn.layer_inputs(lay, syn.config_seed("resnet18", i))
    got = _run_pair(O, lay, x, w)
    idx = list(range(0, lay.n, max(1, lay.n // 4)))
    assert _max_rel(got[idx], _oracle_layer(lay, x[idx], w)) <= TOL[lay.dtype]
