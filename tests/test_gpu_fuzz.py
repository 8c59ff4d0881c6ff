"""Randomised parity sweep: seeded random Conv2d / ConvTranspose2d layers (channels multiple of 16
bytes, stride 1-3, dilation 1-3, pads, output_padding, bf16 and TF32) through every plan (AUTO with
autotuning, FUSED, UNFUSED, GEMM_RED) against the fp64 oracle, bit-exact in integer mode.  Plans a
shape does not support are skipped per case, never silently replaced."""
import numpy as np
import pytest
import torch

import oracle
import ollie_synth as syn
from tests.test_gpu_parity import _dev, _oracle_layer, _round_like

pytestmark = pytest.mark.gpu


def _random_layers(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        dtype = "tf32" if rng.random() < 0.25 else "bf16"
        q = 4 if dtype == "tf32" else 8
        transposed = rng.random() < 0.35
        n = int(rng.integers(1, 4))
        c = int(q * rng.integers(1, 9))
        f = int(rng.integers(1, 9) * (4 if rng.random() < 0.8 else 1))
        r = int(rng.choice([1, 2, 3, 4, 5]))
        s_ = int(rng.choice([1, 2, 3, 4, 5]))
        h, w = int(rng.integers(2, 20)), int(rng.integers(2, 24))
        if transposed:
            st = int(rng.integers(1, 3))
            dil = 1
            pad = int(rng.integers(0, min(r, s_)))
            op = int(rng.integers(0, st)) if st > 1 else 0
        else:
            st = int(rng.integers(1, 4))
            dil = int(rng.integers(1, 4))
            pad = int(rng.integers(0, dil * (min(r, s_) - 1) // 2 + 2))
            op = 0
        lay = syn.Layer(f"fz{len(out)}", n, c, h, w, f, r, s_, pad=pad, stride=st, dilation=dil, output_padding=op,
                        transposed=transposed, dtype=dtype)
        if lay.oh <= 0 or lay.ow <= 0:
            continue
        out.append(lay)
    return out


LAYERS = _random_layers(120, 20261017)


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


@pytest.mark.parametrize("lay", LAYERS, ids=[f"{l.name}-{'T' if l.transposed else 'C'}{l.r}x{l.s}s{l.stride}d{l.dilation}p{l.pad}-{l.dtype}"
                                            for l in LAYERS])
def test_fuzz_all_plans_integer_exact(O, lay):
    from paper_2208_02025_b200 import DerivedConv
    x, w = syn.layer_inputs(lay, 900, exact_int=True)
    ref = _round_like(_oracle_layer(lay, x, w), lay.dtype)
    ran = 0
    for plan in (O.PLAN_AUTO, O.PLAN_FUSED, O.PLAN_UNFUSED, O.PLAN_GEMM_RED, O.PLAN_SMALL):
        try:
            conv = DerivedConv.from_layer(lay, plan=plan).prepare(_dev(w))
            y = conv(_dev(x))
            torch.cuda.synchronize()
        except O.OllieError as e:
            assert e.status == O.E_UNSUPPORTED, f"plan {plan}: {e}"
            continue
        ran += 1
        got = y.float().cpu().numpy()
        assert np.array_equal(got, ref), f"plan {plan} ({conv.resolved_plan()}) differs"
    assert ran >= 1
