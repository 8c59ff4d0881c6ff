"""GPU parity of NEXT-1: the dilated conv as space_to_batch -> dense derived conv ->
batch_to_space, all in libollie kernels, against the fp64 oracle's direct dilated convolution
(integer mode bit-exact; random within the bf16 / TF32 bars), incl. sizes that are not multiples
of the dilation (div / mod form of the eOperators) and CSRNet at full size (sampled images)."""
import numpy as np
import pytest
import torch

import oracle
import ollie_synth as syn
from tests.test_gpu_parity import TOL, _dev, _max_rel, _round_like

pytestmark = pytest.mark.gpu

LAYERS = [
    syn.Layer("d2_even", 2, 64, 16, 16, 64, 3, 3, pad=2, dilation=2),
    syn.Layer("d2_odd", 1, 32, 15, 13, 48, 3, 3, pad=2, dilation=2),
    syn.Layer("d3", 1, 64, 18, 21, 32, 3, 3, pad=3, dilation=3),
    syn.Layer("d2_5x5", 1, 16, 20, 20, 24, 5, 5, pad=4, dilation=2),
    syn.Layer("d2_tf32", 1, 36, 12, 12, 20, 3, 3, pad=2, dilation=2, dtype="tf32"),
]


def _run(lay, x, w, plan=0):
    from paper_2208_02025_b200 import DilatedAsDense
    m = DilatedAsDense.from_layer(lay, plan=plan).prepare(_dev(w))
    y = m(_dev(x))
    torch.cuda.synchronize()
    return y.float().cpu().numpy(), m


def _ref(lay, x, w):
    return oracle.conv2d(x, w, pad=lay.pad, dilation=lay.dilation)


@pytest.mark.parametrize("plan", [0, 1, 2, 3])
@pytest.mark.parametrize("lay", LAYERS, ids=[l.name for l in LAYERS])
def test_next1_integer_exact(lay, plan):
    x, w = syn.layer_inputs(lay, 600, exact_int=True)
    got, _ = _run(lay, x, w, plan)
    assert np.array_equal(got, _round_like(_ref(lay, x, w), lay.dtype))


@pytest.mark.parametrize("lay", LAYERS, ids=[l.name for l in LAYERS])
def test_next1_random_tolerance(lay):
    x, w = syn.layer_inputs(lay, 601)
    got, _ = _run(lay, x, w)
    assert _max_rel(got, _ref(lay, x, w)) <= TOL[lay.dtype]


def test_next1_csrnet_full_size_sampled():
    lay = syn.CONFIGS["csrnet"][0]
    x, w = syn.layer_inputs(lay, syn.config_seed("csrnet", 0))
    got, m = _run(lay, x, w)
    assert m.launches() in (3, 4)
    idx = [0, 9]
    assert _max_rel(got[idx], _ref(lay, x[idx], w)) <= TOL[lay.dtype]


def test_next1_matches_direct_dilated_form():
    """Both derived programs of the same layer agree with each other (bf16 RNE of the same exact
    integer sums)."""
    from paper_2208_02025_b200 import DerivedConv
    lay = LAYERS[0]
    x, w = syn.layer_inputs(lay, 602, exact_int=True)
    got, _ = _run(lay, x, w)
    direct = DerivedConv.from_layer(lay).prepare(_dev(w))(_dev(x))
    torch.cuda.synchronize()
    assert np.array_equal(got, direct.float().cpu().numpy())
