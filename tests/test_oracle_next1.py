"""Pins for NEXT-1 (dilated -> dense derivation): the oracle's derivation equals the
direct dilated convolution (definition O1) exactly in integer mode; the product's layout eOperator
specs, run through the oracle's eOp interpreter (SPEC semantics), equal numpy strided slicing and
round-trip to the identity."""
import numpy as np
import pytest

import oracle
from paper_2208_02025_b200 import eops


def _ints(shape, seed):
    return np.random.default_rng(seed).integers(-4, 5, shape).astype(np.float64)


@pytest.mark.parametrize("n,h,w,c,f,d,r", [(1, 8, 8, 3, 2, 2, 3), (2, 7, 9, 2, 3, 2, 3), (1, 10, 11, 2, 2, 3, 3),
                                           (1, 9, 6, 1, 1, 2, 5)])
def test_derivation_equals_dilated_conv(n, h, w, c, f, d, r):
    x, wt = _ints((n, h, w, c), 1), _ints((f, c, r, r), 2)
    pad = d * (r - 1) // 2
    assert np.array_equal(oracle.conv2d_dilated_as_dense(x, wt, pad, d), oracle.conv2d(x, wt, pad=pad, dilation=d))


def test_derivation_rejects_pad_not_multiple_of_dilation():
    with pytest.raises(ValueError):
        oracle.conv2d_dilated_as_dense(np.zeros((1, 4, 4, 1)), np.zeros((1, 1, 3, 3)), 1, 2)


@pytest.mark.parametrize("n,h,w,c,d", [(2, 6, 4, 3, 2), (1, 7, 5, 2, 2), (2, 9, 9, 1, 3)])
def test_space_to_batch_spec_is_strided_slicing(n, h, w, c, d):
    x = _ints((n, h, w, c), 3)
    got = oracle.eop_eval(eops.space_to_batch(n, h, w, c, d), [x])
    hs, ws = -(-h // d), -(-w // d)
    got = got.reshape(d * d * n, hs, ws, c)
    for a in range(d):
        for b in range(d):
            want = np.zeros((n, hs, ws, c))
            sl = x[:, a::d, b::d, :]
            want[:, :sl.shape[1], :sl.shape[2], :] = sl
            assert np.array_equal(got[(a * d + b) * n:(a * d + b + 1) * n], want)


@pytest.mark.parametrize("n,h,w,c,d", [(2, 6, 4, 3, 2), (1, 7, 5, 2, 2), (2, 9, 9, 1, 3)])
def test_space_batch_round_trip_is_identity(n, h, w, c, d):
    x = _ints((n, h, w, c), 4)
    hs, ws = -(-h // d), -(-w // d)
    xs = oracle.eop_eval(eops.space_to_batch(n, h, w, c, d), [x]).reshape(d * d * n, hs, ws, c)
    back = oracle.eop_eval(eops.batch_to_space(n, hs, ws, c, d, h, w), [xs]).reshape(n, h, w, c)
    assert np.array_equal(back, x)
