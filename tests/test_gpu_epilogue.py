"""GPU parity of the fused element-wise epilogue (NEXT-3): Y = act(conv + bias + residual)
computed inside the fused kernel, the OffsetAdd / selective-add kernels and the identity plan's
GEMM epilogue, against oracle.epilogue(oracle.conv*(...)).  Integer mode is bit-exact (integer
bias / residual, PReLU slope 0.25); random data meets the bf16 / TF32 bars."""
import numpy as np
import pytest
import torch

import oracle
import ollie_synth as syn
from tests.test_gpu_parity import SMALL, TOL, _dev, _max_rel, _oracle_layer, _round_like

pytestmark = pytest.mark.gpu

ACTS = {"none": 0, "relu": 1, "prelu": 2}


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


def _epi_inputs(lay, seed, exact):
    g = torch.Generator().manual_seed(seed)
    if exact:
        bias = torch.randint(-8, 9, (lay.f,), generator=g).float()
        res = torch.randint(-4, 5, (lay.n, lay.oh, lay.ow, lay.f), generator=g).float()
        alpha = torch.full((lay.f,), 0.25)
    else:
        bias = torch.randn(lay.f, generator=g)
        res = torch.rand((lay.n, lay.oh, lay.ow, lay.f), generator=g) * 2 - 1
        alpha = torch.rand(lay.f, generator=g) * 0.5
    res = res.to(syn.torch_dtype(lay.dtype))
    return bias, res, alpha


def _run(O, lay, x, w, plan, bias, res, act, alpha, in_place=False):
    from paper_2208_02025_b200 import DerivedConv
    conv = DerivedConv.from_layer(lay, plan=plan)
    conv.prepare(_dev(w))
    rd = _dev(res) if res is not None else None
    y = rd if in_place else None
    try:
        y = conv(_dev(x), y, None, bias=_dev(bias) if bias is not None else None, residual=rd,
                 act=ACTS[act], alpha=_dev(alpha))
    except O.OllieError as e:
        if plan in (O.PLAN_FUSED, O.PLAN_GEMM_RED) and e.status == O.E_UNSUPPORTED:
            pytest.skip("no fused plan for this layer")
        raise
    torch.cuda.synchronize()
    return y.float().cpu().numpy()


@pytest.mark.parametrize("act", ["none", "relu", "prelu"])
@pytest.mark.parametrize("plan", [0, 1, 2, 3])
@pytest.mark.parametrize("lay", SMALL, ids=[l.name for l in SMALL])
def test_epilogue_integer_exact(O, lay, plan, act):
    x, w = syn.layer_inputs(lay, 100, exact_int=True)
    bias, res, alpha = _epi_inputs(lay, 7, True)
    got = _run(O, lay, x, w, plan, bias, res, act, alpha)
    want = oracle.epilogue(_oracle_layer(lay, x, w), bias.numpy(), res, act, alpha.numpy())
    assert np.array_equal(got, _round_like(want, lay.dtype))


@pytest.mark.parametrize("plan", [0, 1, 2, 3])
@pytest.mark.parametrize("lay", SMALL, ids=[l.name for l in SMALL])
def test_epilogue_random_tolerance(O, lay, plan):
    x, w = syn.layer_inputs(lay, 200)
    bias, res, alpha = _epi_inputs(lay, 8, False)
    got = _run(O, lay, x, w, plan, bias, res, "prelu", alpha)
    want = oracle.epilogue(_oracle_layer(lay, x, w), bias.numpy(), res, "prelu", alpha.numpy())
    assert _max_rel(got, want) <= TOL[lay.dtype]


@pytest.mark.parametrize("plan", [0, 1, 2, 3])
def test_epilogue_bias_only_and_in_place_residual(O, plan):
    lay = syn.Layer("r18_64_tiny", 2, 64, 12, 13, 64, 3, 3, pad=1)
    x, w = syn.layer_inputs(lay, 101, exact_int=True)
    bias, res, alpha = _epi_inputs(lay, 9, True)
    ref = _oracle_layer(lay, x, w)
    got = _run(O, lay, x, w, plan, bias, None, "relu", alpha)
    assert np.array_equal(got, _round_like(oracle.epilogue(ref, bias.numpy(), None, "relu"), lay.dtype))
    got = _run(O, lay, x, w, plan, None, res, "none", alpha, in_place=True)      # y aliases residual
    assert np.array_equal(got, _round_like(oracle.epilogue(ref, None, res, "none"), lay.dtype))


def test_epilogue_errors(O):
    shp = O.conv_shape(1, 16, 8, 8, 16, 3, 3, 1)
    x = torch.zeros(1, 8, 8, 16, dtype=torch.bfloat16, device="cuda")
    wp = torch.zeros(9 * 16, 16, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(1, 8, 8, 16, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(O.OllieError) as e:
        O.conv2d_derived_ex(shp, O.BF16, x, wp, y, plan=O.PLAN_FUSED, epilogue=O.make_epilogue(act=2))
    assert e.value.status == O.E_INVALID
    with pytest.raises(O.OllieError) as e:
        O.conv2d_derived_ex(shp, O.BF16, x, wp, y, plan=O.PLAN_FUSED, epilogue=O.make_epilogue(act=7))
    assert e.value.status == O.E_INVALID
