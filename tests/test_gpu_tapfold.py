"""GPU parity of the im2col ("tap folding") eOperator (ollie_tap_fold) -- bit-exact against
oracle.tap_fold (pure indexing) -- and of a few-channel first layer run as tap fold + 1x1 derived
conv through DerivedStack (integer mode bit-exact, random data within the bf16 bar)."""
import numpy as np
import pytest
import torch

import oracle
import ollie_synth as syn
from tests.test_gpu_parity import TOL, _max_rel, _oracle_layer, _round_like

pytestmark = pytest.mark.gpu

FOLD = [  # (n, h, w, c, r, s, pad, stride, dil, kp, dtype)
    (2, 9, 11, 1, 5, 5, 2, 1, 1, 32, "bf16"), (1, 7, 8, 3, 3, 3, 1, 2, 1, 32, "bf16"),
    (2, 6, 9, 2, 3, 3, 2, 1, 2, 24, "bf16"), (1, 5, 5, 1, 9, 9, 4, 1, 1, 88, "bf16"),
    (1, 6, 7, 1, 5, 5, 2, 1, 1, 28, "tf32"), (3, 4, 4, 3, 2, 2, 0, 1, 1, 16, "bf16"),
    # 16-byte staged rows (w * c a multiple of 8 bf16 / 4 fp32), halos wider than the pad, FSRCNN width
    (2, 5, 16, 1, 5, 5, 2, 1, 1, 32, "bf16"), (1, 6, 24, 2, 3, 3, 1, 2, 2, 24, "bf16"),
    (1, 3, 256, 1, 5, 5, 2, 1, 1, 32, "bf16"), (1, 4, 1, 1, 3, 3, 1, 1, 1, 16, "bf16"),
    (1, 5, 8, 4, 3, 3, 3, 1, 1, 40, "tf32"), (2, 7, 8, 1, 9, 9, 4, 2, 1, 88, "bf16"),
]


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


@pytest.mark.parametrize("n,h,w,c,r,s,pad,st,dil,kp,dtype", FOLD)
def test_tap_fold_bit_exact(O, n, h, w, c, r, s, pad, st, dil, kp, dtype):
    x = syn.uniform((n, h, w, c), 40 + h, dtype)
    shp = O.conv_shape(n, c, h, w, 1, r, s, pad, st, dil)
    oh, ow = O.output_hw(shp, False)
    out = torch.full((n, oh, ow, kp), float("nan"), dtype=syn.torch_dtype(dtype), device="cuda")
    O.tap_fold(shp, O.BF16 if dtype == "bf16" else O.TF32, x.cuda(), kp, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.double().cpu().numpy(), oracle.tap_fold(x, r, s, pad, st, dil, kp))


def test_tap_fold_errors(O):
    shp = O.conv_shape(1, 1, 8, 8, 1, 5, 5, 2)
    x = torch.zeros(1, 8, 8, 1, dtype=torch.bfloat16, device="cuda")
    out = torch.zeros(1, 8, 8, 32, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(O.OllieError) as e:
        O.tap_fold(shp, O.BF16, x, 24 - 1, out)           # kp < r*s*c
    assert e.value.status == O.E_INVALID
    with pytest.raises(O.OllieError) as e:
        O.tap_fold(shp, O.BF16, x, 28, out)               # 56-byte pixels: not a multiple of 16
    assert e.value.status == O.E_ALIGN


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("lay", [syn.Layer("fold_5x5_1to56", 2, 1, 33, 140, 56, 5, 5, pad=2),
                                 syn.Layer("fold_3x3s2_3to24", 2, 3, 17, 19, 24, 3, 3, pad=1, stride=2)],
                         ids=["fsrcnn_feat_like", "rgb_s2"])
def test_folded_first_layer(O, lay, exact):
    from paper_2208_02025_b200.stack import DerivedStack, foldable
    assert foldable(lay)
    st = DerivedStack([lay], False)
    assert st.layers[0].fold
    x, w = syn.layer_inputs(lay, 41, exact_int=exact)
    st.prepare([w.cuda()])
    y = st([x.cuda()])[0]
    y = st([x.cuda()])[0]                                  # the autotuned plan
    torch.cuda.synchronize()
    ref = _oracle_layer(lay, x, w)
    got = y.float().cpu().numpy()
    if exact:
        assert np.array_equal(got, _round_like(ref, "bf16"))
    else:
        assert _max_rel(got, ref) <= TOL["bf16"]
