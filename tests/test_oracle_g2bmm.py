"""Pins for the G2BMM oracle (NEXT-4; iterator table, LongFormer P:1605; reading R4):
pure-Python brute force on tiny inputs, closed forms, the W = 0 special case (row-wise dot
products), the band symmetry of G2BMM(A, A), and the paper's dilated -> non-dilated derivation
(residue split) equal to the direct definition exactly in integer mode."""
import numpy as np
import pytest

import oracle


def _ints(shape, seed):
    return np.random.default_rng(seed).integers(-4, 5, shape).astype(np.float64)


def _brute(a, b, W, d):
    nb, L, K = a.shape
    out = np.zeros((nb, L, 2 * W + 1))
    for bb in range(nb):
        for m in range(L):
            for w in range(2 * W + 1):
                j = m + d * (w - W)
                if 0 <= j < L:
                    out[bb, m, w] = sum(a[bb, m, k] * b[bb, j, k] for k in range(K))
    return out


@pytest.mark.parametrize("nb,L,K,W,d", [(1, 7, 3, 2, 1), (2, 9, 4, 1, 3), (1, 12, 2, 3, 2), (1, 5, 1, 4, 1)])
def test_g2bmm_brute_force(nb, L, K, W, d):
    a, b = _ints((nb, L, K), 1), _ints((nb, L, K), 2)
    assert np.array_equal(oracle.g2bmm(a, b, W, d), _brute(a, b, W, d))


def test_g2bmm_allones_closed_form():
    # A = B = 1: out[m, w] = K if 0 <= m + d(w - W) < L else 0
    L, K, W, d = 20, 5, 3, 2
    out = oracle.g2bmm(np.ones((1, L, K)), np.ones((1, L, K)), W, d)[0]
    m, w = np.meshgrid(np.arange(L), np.arange(2 * W + 1), indexing="ij")
    j = m + d * (w - W)
    assert np.array_equal(out, np.where((j >= 0) & (j < L), float(K), 0.0))


def test_g2bmm_w0_is_rowwise_dot():
    a, b = _ints((2, 11, 6), 3), _ints((2, 11, 6), 4)
    assert np.array_equal(oracle.g2bmm(a, b, 0, 3)[..., 0], np.einsum("blk,blk->bl", a, b))


def test_g2bmm_band_symmetry():
    # G2BMM(A, A): out[m, w] = out[m + d(w - W), 2W - w] wherever the partner row exists
    a = _ints((1, 30, 4), 5)
    W, d = 3, 2
    out = oracle.g2bmm(a, a, W, d)[0]
    for m in range(30):
        for w in range(2 * W + 1):
            j = m + d * (w - W)
            if 0 <= j < 30:
                assert out[m, w] == out[j, 2 * W - w]


@pytest.mark.parametrize("L,W,d", [(40, 3, 4), (37, 5, 3), (16, 2, 2), (9, 4, 5)])
def test_residue_split_derivation_equals_definition(L, W, d):
    a, b = _ints((2, L, 8), 6), _ints((2, L, 8), 7)
    assert np.array_equal(oracle.g2bmm_residue_split(a, b, W, d), oracle.g2bmm(a, b, W, d))
