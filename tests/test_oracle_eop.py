"""Pins for the literal eOperator interpreter (oracle/eop_oracle.py), CPU only.

 - DLT transpose == numpy transpose (library routine),
 - layout-A on NHWC is detected as the identity and a transpose is not,
 - DLT round trip Phi^-1 o Phi == identity, evaluated as a fused pair,
 - OffsetAdd / selective-add written as eOperators == the C oracle's a3 / a4 (which are
   pinned independently by the derivation identity in test_oracle_conv.py),
 - a fused pair == sequential evaluation, inline == memoised,
 - reads outside the pad band raise OutOfBoundsRead, empty ranges are invalid.
"""
import numpy as np
import pytest

import oracle
from oracle.eop_oracle import InvalidExpression, OutOfBoundsRead
from tests import eop_cases as ec


def _rand(shape, seed):
    return np.random.default_rng(seed).integers(-4, 5, size=shape).astype(np.float64)


def test_transpose_matches_numpy():
    x = _rand((2, 3, 4, 5), 0)
    out = oracle.eop_eval(ec.transpose_nchw_to_nhwc(2, 3, 4, 5), [x])
    assert np.array_equal(out, x.transpose(0, 2, 3, 1))


def test_identity_detection():
    assert oracle.eop_is_identity(ec.layout_a(3, 4, 5))
    assert not oracle.eop_is_identity(ec.transpose_nchw_to_nhwc(2, 3, 4, 5))
    assert oracle.eop_is_identity(ec.transpose_nchw_to_nhwc(1, 1, 4, 5))   # degenerate c = 1
    assert not oracle.eop_is_identity(ec.channel_pad(1, 2, 2, 3, 4))
    x = _rand((3, 4, 5), 1)
    assert np.array_equal(oracle.eop_eval(ec.layout_a(3, 4, 5), [x]), x.reshape(12, 5))


def test_dlt_round_trip_as_fused_pair():
    n, c, h, w = 2, 3, 4, 5
    fwd = ec.transpose_nchw_to_nhwc(n, c, h, w)["scopes"][0]          # inner: NCHW -> NHWC
    inv = {"trav": [[0, n], [0, c], [0, h], [0, w]], "sum": [],     # outer: NHWC -> NCHW
           "access": [{"tensor": -1, "index": [ec.idx(ec.I(0)), ec.idx(ec.I(2)), ec.idx(ec.I(3)),
                                               ec.idx(ec.I(1))]}],
           "body": [["acc", 0]]}
    expr = {"inputs": [{"shape": [n, c, h, w]}], "scopes": [inv, fwd]}
    x = _rand((n, c, h, w), 2)
    assert np.array_equal(oracle.eop_eval(expr, [x]), x)
    assert np.array_equal(oracle.eop_eval(expr, [x], memoize=True), x)


@pytest.mark.parametrize("n,h,w,f,r,s,pad,st,dil", [(2, 4, 5, 2, 3, 3, 1, 1, 1), (1, 6, 5, 3, 3, 3, 2, 1, 2),
                                                    (1, 7, 6, 2, 3, 3, 1, 2, 1), (1, 5, 5, 1, 5, 5, 2, 1, 1),
                                                    (2, 3, 4, 3, 1, 1, 0, 1, 1)])
def test_offset_add_eop_matches_c_oracle(n, h, w, f, r, s, pad, st, dil):
    T = _rand((n * h * w, r * s * f), 3 + h)
    want = oracle.offset_add(T, n, h, w, f, r, s, pad, st, dil)
    spec = ec.offset_add(n, h, w, f, r, s, pad, st, dil)
    assert oracle.eop_bounds_ok(spec)
    got = oracle.eop_eval(spec, [T.reshape(n, h, w, r * s * f)])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,h,w,f,r,s,pad,st,op", [(2, 2, 3, 2, 4, 4, 1, 2, 0), (1, 3, 3, 1, 9, 9, 4, 2, 1),
                                                   (1, 3, 2, 2, 3, 3, 1, 2, 1), (1, 2, 2, 1, 3, 3, 0, 3, 0),
                                                   (1, 3, 3, 2, 3, 3, 1, 1, 0)])
def test_selective_add_eop_matches_c_oracle(n, h, w, f, r, s, pad, st, op):
    T = _rand((n * h * w, r * s * f), 4 + h)
    want = oracle.selective_add(T, n, h, w, f, r, s, pad, st, 1, op)
    spec = ec.selective_add(n, h, w, f, r, s, pad, st, op)
    assert oracle.eop_bounds_ok(spec)
    got = oracle.eop_eval(spec, [T.reshape(n, h, w, r, s, f)])
    assert np.array_equal(got, want)


def test_fused_pair_equals_sequential():
    n, h, w, f, r, s, pad, extra = 1, 4, 5, 2, 3, 3, 1, 3
    nt = r * s * f
    T = _rand((n, h, w, nt), 5)
    spec = ec.fused_pad_then_offset_add(n, h, w, f, r, s, pad, extra)
    inline = oracle.eop_eval(spec, [T])
    memo = oracle.eop_eval(spec, [T], memoize=True)
    # sequential: evaluate the inner scope alone, then the outer OffsetAdd on its output
    inner_only = {"inputs": spec["inputs"], "scopes": [dict(spec["scopes"][1])]}
    inner_only["scopes"][0].pop("pad")
    mid = oracle.eop_eval(inner_only, [T])
    assert np.array_equal(mid[..., nt:], np.zeros((n, h, w, extra)))
    seq = oracle.offset_add(mid[..., :nt].reshape(-1, nt), n, h, w, f, r, s, pad)
    assert np.array_equal(inline, seq)
    assert np.array_equal(memo, seq)


def test_affine_mix_body_ops():
    n, c, h, w = 2, 3, 2, 4
    a, b = _rand((n, c, h, w), 6), _rand((h, w), 7)
    got = oracle.eop_eval(ec.affine_mix(n, c, h, w), [a, b])
    # f sits inside the summation: the max term is added once per k
    want = ((2 * a - b[None, None]) * 0.5 + np.maximum(b, 0)[None, None]).sum(axis=1)
    assert np.array_equal(got, want)


def test_out_of_bounds_read_rejected():
    spec = ec.offset_add(1, 4, 4, 1, 3, 3, 1)
    spec["inputs"][0]["pad"] = [[0, 0], [0, 0], [0, 0], [0, 0]]   # drop the pad band
    assert not oracle.eop_bounds_ok(spec)
    with pytest.raises(OutOfBoundsRead):
        oracle.eop_eval(spec, [np.zeros((1, 4, 4, 9))])


def test_empty_range_rejected():
    spec = ec.layout_a(2, 2, 2)
    spec["scopes"][0]["trav"][1] = [3, 3]
    with pytest.raises(InvalidExpression):
        oracle.eop_eval(spec, [np.zeros((2, 2, 2))])
