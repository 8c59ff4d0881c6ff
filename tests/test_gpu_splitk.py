"""GPU parity of split-K fused plans: a cluster of ksplit CTAs shares each output tile, every CTA
accumulates a contiguous range of (channel chunk, input phase) steps in its own TMEM, and the fp32
partials are reduced through distributed shared memory before the epilogue writes Y.  Forced
with the debug hook ollie_debug_force_ksplit; compared with the fp64 oracle (integer mode
bit-exact -- fp32 partial sums of integers are exact in any order -- and random within the
bf16 / TF32 bars)."""
import numpy as np
import pytest
import torch

import oracle
import ollie_synth as syn
from tests.test_gpu_parity import TOL, _dev, _max_rel, _oracle_layer, _round_like

pytestmark = pytest.mark.gpu

LAYERS = [
    syn.Layer("k4_256x14", 2, 256, 14, 14, 256, 3, 3, pad=1),
    syn.Layer("k8_512x7", 1, 512, 7, 7, 512, 3, 3, pad=1),
    syn.Layer("k2_f72_tail", 1, 128, 9, 11, 72, 3, 3, pad=1),
    syn.Layer("k2_c96_partial_chunk", 2, 96, 10, 9, 64, 3, 3, pad=1),
    syn.Layer("convt_classes", 2, 512, 4, 4, 256, 4, 4, pad=1, stride=2, transposed=True),
    syn.Layer("strided_phases", 2, 128, 14, 14, 256, 3, 3, pad=1, stride=2),
    syn.Layer("dilated", 1, 256, 16, 16, 128, 3, 3, pad=2, dilation=2),
    syn.Layer("tf32", 1, 64, 12, 10, 48, 3, 3, pad=1, dtype="tf32"),
]


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


@pytest.fixture
def force_ks(O):
    yield lambda ks: O._lib.ollie_debug_force_ksplit(ks)
    O._lib.ollie_debug_force_ksplit(-1)


def _run(O, lay, x, w, **epi):
    from paper_2208_02025_b200 import DerivedConv
    conv = DerivedConv.from_layer(lay, plan=O.PLAN_FUSED)
    conv.prepare(_dev(w))
    try:
        y = conv(_dev(x), **epi)
    except O.OllieError as e:
        if e.status == O.E_UNSUPPORTED:
            pytest.skip("no split-K plan for this layer")
        raise
    torch.cuda.synchronize()
    desc = O.plan_describe(conv.shape, conv.code, O.PLAN_FUSED, conv.transposed)
    return y.float().cpu().numpy(), desc


@pytest.mark.parametrize("ks", [2, 4])
@pytest.mark.parametrize("lay", LAYERS, ids=[l.name for l in LAYERS])
def test_splitk_integer_exact(O, force_ks, lay, ks):
    force_ks(ks)
    x, w = syn.layer_inputs(lay, 500, exact_int=True)
    got, desc = _run(O, lay, x, w)
    assert f"ksplit={ks}" in desc, desc
    assert np.array_equal(got, _round_like(_oracle_layer(lay, x, w), lay.dtype))


@pytest.mark.parametrize("ks", [2, 4])
@pytest.mark.parametrize("lay", LAYERS, ids=[l.name for l in LAYERS])
def test_splitk_random_tolerance(O, force_ks, lay, ks):
    force_ks(ks)
    x, w = syn.layer_inputs(lay, 501)
    got, desc = _run(O, lay, x, w)
    assert f"ksplit={ks}" in desc, desc
    assert _max_rel(got, _oracle_layer(lay, x, w)) <= TOL[lay.dtype]


def test_splitk_with_epilogue(O, force_ks):
    force_ks(4)
    lay = LAYERS[0]
    x, w = syn.layer_inputs(lay, 502, exact_int=True)
    g = torch.Generator().manual_seed(3)
    bias = torch.randint(-8, 9, (lay.f,), generator=g).float()
    res = torch.randint(-4, 5, (lay.n, lay.oh, lay.ow, lay.f), generator=g).to(torch.bfloat16)
    got, desc = _run(O, lay, x, w, bias=_dev(bias), residual=_dev(res), act=1)
    assert "ksplit=4" in desc
    want = oracle.epilogue(_oracle_layer(lay, x, w), bias.numpy(), res, "relu")
    assert np.array_equal(got, _round_like(want, lay.dtype))
