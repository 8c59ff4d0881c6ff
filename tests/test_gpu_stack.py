"""GPU: chained stacks through the C ABI (FSRCNN-like with channel-pad eOperators and
identity-eliminated 1x1 layers, DCGAN generator), checked layer by layer against the oracle on
the same (GPU-produced, already rounded) layer inputs, so rounding does not compound
(SURVEY 8(d) "Stacks (C4) are checked per layer")."""
from dataclasses import replace

import numpy as np
import pytest
import torch

import oracle
import ollie_synth as syn

pytestmark = pytest.mark.gpu


def _fsrcnn_small(n=2, hw=24):
    return [replace(l, n=n, h=hw, w=hw) for l in syn.CONFIGS["fsrcnn"]]


def _check_stack(layers, chained, exact):
    from paper_2208_02025_b200.stack import DerivedStack
    st = DerivedStack(layers, chained)
    xs, ws = [], []
    for i, l in enumerate(layers):
        x, w = syn.layer_inputs(l, 300 + i, exact_int=exact)
        xs.append(x)
        ws.append(w)
    st.prepare([w.cuda() for w in ws])
    outs = st(xs[0].cuda() if chained else [x.cuda() for x in xs])
    torch.cuda.synchronize()
    src = xs[0]
    for l, y, w in zip(layers, outs, ws):
        if l.transposed:
            ref = oracle.conv_transpose2d(src, w, l.pad, l.stride, l.dilation, l.output_padding)
        else:
            ref = oracle.conv2d(src, w, l.pad, l.stride, l.dilation)
        got = y.float().cpu().numpy()
        if exact:
            want = torch.from_numpy(ref).float().to(torch.bfloat16).float().numpy()
            assert np.array_equal(got, want), l.name
        else:
            err = np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-30)
            assert err <= 1e-2, (l.name, err)
        src = y.cpu()          # next layer's input is exactly what the GPU produced


def test_fsrcnn_stack_random():
    _check_stack(_fsrcnn_small(), True, exact=False)


def test_fsrcnn_stack_integer_exact():
    # integer mode through a deep stack overflows bf16's exact range, so use a 2-layer prefix
    # (pad eOp + fused 5x5 + identity-eliminated 1x1) and the deconv alone
    layers = _fsrcnn_small(1, 16)
    _check_stack(layers[:2], True, exact=True)
    _check_stack([layers[-1]], True, exact=True)


def test_dcgan_stack_random():
    layers = [replace(l, n=2) for l in syn.CONFIGS["dcgan"]]
    _check_stack(layers, True, exact=False)


def test_launch_counts():
    from paper_2208_02025_b200.stack import DerivedStack
    st = DerivedStack(_fsrcnn_small(1, 16), True)
    # f=12 layers write zero-padded 16-channel outputs instead of a separate pad launch; the c=1
    # network input is tap-folded (im2col eOperator) for its 5x5 layer, nothing else is padded
    assert sum(1 for sl in st.layers if sl.pad_eop is not None) == 0
    assert [sl.fold for sl in st.layers] == [True] + [False] * (len(st.layers) - 1)
    assert DerivedStack(_fsrcnn_small(1, 16), True, fold_taps=False).layers[0].pad_eop is not None
    assert st.launches() >= len(st.layers)
