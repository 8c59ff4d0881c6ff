"""Pins for oracle.epilogue (NEXT-3, reading Q19) -- closed forms, special cases that
reduce to textbook / library activations, and algebraic identities."""
import numpy as np
import pytest
import torch

import oracle


def _ones_conv(c=1, h=4, w=4):
    x = np.ones((1, h, w, c))
    wt = np.ones((1, c, 3, 3))
    return oracle.conv2d(x, wt, pad=1)


def test_bias_relu_on_allones_worked_example():
    # all-ones 4x4, 3x3, pad 1: corners 4, edges 6, interior 9.  Bias -6 then ReLU:
    # corners max(-2,0)=0, edges 0, interior 3 -- a value table a dropped bias or ReLU breaks.
    y = _ones_conv()
    out = oracle.epilogue(y, bias=np.array([-6.0]), act="relu")[0, :, :, 0]
    want = np.array([[0, 0, 0, 0], [0, 3, 3, 0], [0, 3, 3, 0], [0, 0, 0, 0]], dtype=np.float64)
    assert np.array_equal(out, want)


def test_prelu_on_allones_worked_example():
    y = _ones_conv()
    out = oracle.epilogue(y, bias=np.array([-6.0]), act="prelu", alpha=np.array([0.5]))[0, :, :, 0]
    want = np.array([[-1, 0, 0, -1], [0, 3, 3, 0], [0, 3, 3, 0], [-1, 0, 0, -1]], dtype=np.float64)
    assert np.array_equal(out, want)


def test_residual_cancels_exactly():
    rng = np.random.default_rng(0)
    y = rng.standard_normal((2, 3, 5, 7))
    assert np.array_equal(oracle.epilogue(y, residual=-y), np.zeros_like(y))


def test_prelu_special_cases_reduce_to_relu_and_identity():
    rng = np.random.default_rng(1)
    y = rng.standard_normal((2, 4, 4, 6))
    assert np.array_equal(oracle.epilogue(y, act="prelu", alpha=np.zeros(6)), oracle.epilogue(y, act="relu"))
    assert np.array_equal(oracle.epilogue(y, act="prelu", alpha=np.ones(6)), y)


def test_relu_identity_and_library():
    rng = np.random.default_rng(2)
    y = rng.standard_normal((1, 5, 5, 8))
    b = rng.standard_normal(8)
    r = rng.standard_normal(y.shape)
    got = oracle.epilogue(y, bias=b, residual=r, act="relu")
    v = y + b + r
    assert np.allclose(got, (v + np.abs(v)) / 2, rtol=0, atol=1e-15)
    assert np.array_equal(got, torch.relu(torch.from_numpy(v)).numpy())


def test_prelu_matches_torch_per_channel():
    rng = np.random.default_rng(3)
    y = rng.standard_normal((2, 3, 4, 5))
    a = rng.uniform(0, 0.5, 5)
    got = oracle.epilogue(y, act="prelu", alpha=a)
    # torch's PReLU is channel-first: move f to dim 1
    want = torch.nn.functional.prelu(torch.from_numpy(y).permute(0, 3, 1, 2), torch.from_numpy(a))
    assert np.array_equal(got, want.permute(0, 2, 3, 1).numpy())


def test_bias_broadcasts_over_channels_not_pixels():
    y = np.zeros((1, 2, 3, 4))
    out = oracle.epilogue(y, bias=np.arange(4.0))
    assert np.array_equal(out[0, 1, 2], np.arange(4.0))


def test_unknown_activation_rejected():
    with pytest.raises(ValueError):
        oracle.epilogue(np.zeros((1, 1, 1, 1)), act="gelu")
