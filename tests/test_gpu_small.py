"""GPU parity of OLLIE_PLAN_SMALL -- the fused derived program on CUDA cores for layers of at most
2^22 multiply-adds (include/ollie.h) -- against the fp64 oracle: the paper's motivating example
(BASELINE configs[0], TF32 storage), Conv2d / ConvTranspose2d with stride, dilation and padding,
bit-exact in integer mode and within the bars on random data, the NEXT-3 epilogue, AUTO choosing it
by measurement, and OLLIE_E_UNSUPPORTED above the size limit."""
import numpy as np
import pytest
import torch

import oracle
import ollie_synth as syn
from tests.test_gpu_parity import TOL, _max_rel, _oracle_layer, _round_like

pytestmark = pytest.mark.gpu

LAYERS = [
    syn.CONFIGS["motivating"][0],
    syn.Layer("s_c3", 2, 16, 9, 7, 12, 3, 3, pad=1),
    syn.Layer("s_s2d2", 1, 8, 11, 13, 4, 3, 3, pad=2, stride=2, dilation=2),
    syn.Layer("s_t4s2", 2, 16, 3, 4, 8, 4, 4, pad=1, stride=2, transposed=True),
    syn.Layer("s_t3s2op", 1, 8, 5, 3, 4, 3, 3, pad=1, stride=2, output_padding=1, transposed=True),
    syn.Layer("s_tf32", 1, 4, 6, 6, 5, 5, 5, pad=2, dtype="tf32"),
]


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("lay", LAYERS, ids=[l.name for l in LAYERS])
def test_small_plan_parity(O, lay, exact):
    from paper_2208_02025_b200 import DerivedConv
    x, w = syn.layer_inputs(lay, 950, exact_int=exact)
    conv = DerivedConv.from_layer(lay, plan=O.PLAN_SMALL, autotune=False).prepare(w.cuda())
    assert conv.resolved_plan() == "small"
    y = conv(x.cuda())
    torch.cuda.synchronize()
    ref = _oracle_layer(lay, x, w)
    got = y.double().cpu().numpy()
    if exact:
        assert np.array_equal(got, _round_like(ref, lay.dtype))
    else:
        assert _max_rel(got, ref) <= TOL[lay.dtype]


def test_small_plan_epilogue(O):
    from paper_2208_02025_b200 import DerivedConv
    lay = LAYERS[1]
    x, w = syn.layer_inputs(lay, 951, exact_int=True)
    bias = torch.arange(lay.f, dtype=torch.float32) - 5
    res = torch.ones(lay.n, lay.oh, lay.ow, lay.f, dtype=torch.bfloat16)
    conv = DerivedConv.from_layer(lay, plan=O.PLAN_SMALL, autotune=False).prepare(w.cuda())
    y = conv(x.cuda(), bias=bias.cuda(), residual=res.cuda(), act=O.ACT_RELU)
    torch.cuda.synchronize()
    ref = oracle.epilogue(oracle.conv2d(x, w, lay.pad, lay.stride, lay.dilation), bias.numpy(), res, "relu")
    assert np.array_equal(y.double().cpu().numpy(), _round_like(ref, "bf16"))


def test_small_plan_auto_measures_it(O):
    from paper_2208_02025_b200 import DerivedConv
    lay = LAYERS[0]
    x, w = syn.layer_inputs(lay, 952, exact_int=True)
    conv = DerivedConv.from_layer(lay).prepare(w.cuda())
    y = conv(x.cuda())
    y = conv(x.cuda())
    torch.cuda.synchronize()
    assert conv.resolved_plan() in ("small", "fused", "unfused", "rowstream", "gemm_red")
    assert np.array_equal(y.double().cpu().numpy(), _round_like(_oracle_layer(lay, x, w), lay.dtype))


def test_small_plan_size_limit(O):
    lay = syn.Layer("s_big", 1, 64, 56, 56, 64, 3, 3, pad=1)      # 115.6 M multiply-adds
    shp = O.conv_shape(lay.n, lay.c, lay.h, lay.w, lay.f, lay.r, lay.s, lay.pad)
    with pytest.raises(O.OllieError) as e:
        O.plan_describe(shp, O.BF16, O.PLAN_SMALL, False)
    assert e.value.status == O.E_UNSUPPORTED
