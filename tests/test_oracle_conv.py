"""Pins for the fp64 conv / convT / GEMM / OffsetAdd / selective-add oracle (CPU only).

Each pin comes from outside the oracle (SURVEY 8(c) "What pins each part"):
 - the S:502 worked example (tests/golden/allones_conv3x3_4x4.txt),
 - brute force by a second, textbook formulation (explicit im2col + matmul),
 - torch CPU fp64 F.conv2d / F.conv_transpose2d (independent library, test-only),
 - closed forms (all-ones input), 1x1 conv == matmul (BASELINE north_star),
 - adjointness <conv(x;W), y> == <x, convT(y;W)>,
 - ConvT == conv over the zero-inserted input with a flipped, transposed kernel,
 - the derivation identity conv == OffsetAdd(Matmul(A', DLT(K))), exact
   in integer mode, and the row-wrap sentinel of reading Q5,
 - the ConvT tap table (tests/golden/convt_tap_table_4x4_s2_p1.txt).
"""
import itertools
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as Fnn

import oracle
import ollie_synth as syn

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([int(v) for v in line.split()])
    return np.array(rows)


def _ints(shape, seed):
    return syn.integers(shape, seed, "tf32").double().numpy()


def _torch_conv(x, w, pad, st, dil):
    xt = torch.from_numpy(x).permute(0, 3, 1, 2)
    y = Fnn.conv2d(xt, torch.from_numpy(w), stride=st, padding=pad, dilation=dil)
    return y.permute(0, 2, 3, 1).numpy()


def _torch_convt(x, w, pad, st, dil, op):
    xt = torch.from_numpy(x).permute(0, 3, 1, 2)
    y = Fnn.conv_transpose2d(xt, torch.from_numpy(w), stride=st, padding=pad, dilation=dil,
                             output_padding=op)
    return y.permute(0, 2, 3, 1).numpy()


def _im2col_conv(x, w, pad, st, dil):
    """Textbook im2col: zero-pad, take every (dilated) window with numpy's
    sliding_window_view, flatten (i, j, c) and multiply by the flattened kernel."""
    n, h, wd, c = x.shape
    f, _, r, s = w.shape
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    win = np.lib.stride_tricks.sliding_window_view(xp, (dil * (r - 1) + 1, dil * (s - 1) + 1), axis=(1, 2))
    win = win[:, ::st, ::st, :, ::dil, ::dil]            # n, OH, OW, c, r, s
    cols = win.reshape(win.shape[0], win.shape[1], win.shape[2], -1)   # (c, r, s) flattened
    kmat = w.reshape(f, -1)                               # (c, r, s) flattened, same order
    return cols @ kmat.T


def test_worked_example_all_ones_s502():
    want = _golden("allones_conv3x3_4x4.txt")
    y = oracle.conv2d(np.ones((1, 4, 4, 1)), np.ones((1, 1, 3, 3)), pad=1)
    assert np.array_equal(y[0, :, :, 0], want)
    y2 = oracle.conv2d_derived(np.ones((1, 4, 4, 1)), np.ones((1, 1, 3, 3)), pad=1)
    assert np.array_equal(y2[0, :, :, 0], want)


GRID = [  # (h, w, c, f, r, s, pad, stride, dil)
    (5, 6, 3, 2, 3, 3, 1, 1, 1), (6, 5, 2, 3, 3, 3, 0, 1, 1), (7, 7, 2, 2, 3, 3, 1, 2, 1),
    (8, 6, 3, 2, 3, 3, 2, 1, 2), (6, 7, 1, 4, 5, 5, 2, 1, 1), (7, 8, 2, 2, 1, 1, 0, 1, 1),
    (9, 9, 2, 3, 4, 4, 1, 2, 1), (8, 8, 2, 2, 3, 2, 1, 3, 2), (4, 4, 3, 3, 2, 3, 0, 1, 1),
    (10, 9, 2, 2, 9, 9, 4, 2, 1), (3, 3, 2, 2, 3, 3, 1, 1, 2),
]


@pytest.mark.parametrize("h,w,c,f,r,s,pad,st,dil", GRID)
def test_conv_bruteforce_im2col_and_library(h, w, c, f, r, s, pad, st, dil):
    x = _ints((2, h, w, c), 11 + h)
    wt = _ints((f, c, r, s), 12 + w)
    y = oracle.conv2d(x, wt, pad, st, dil)
    assert np.array_equal(y, _im2col_conv(x, wt, pad, st, dil))
    assert np.array_equal(y, _torch_conv(x, wt, pad, st, dil))
    # random (non-integer) values against the library within fp64 rounding
    xr = np.random.default_rng(h).standard_normal((2, h, w, c))
    wr = np.random.default_rng(w).standard_normal((f, c, r, s))
    np.testing.assert_allclose(oracle.conv2d(xr, wr, pad, st, dil), _torch_conv(xr, wr, pad, st, dil),
                               rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("h,w,c,f,r,s,pad,st,dil", GRID)
def test_derivation_identity_conv_exact(h, w, c, f, r, s, pad, st, dil):
    """O1 == a3 o O3: the direct conv equals OffsetAdd of the merged GEMM."""
    x = _ints((2, h, w, c), 21 + h)
    wt = _ints((f, c, r, s), 22 + w)
    assert np.array_equal(oracle.conv2d(x, wt, pad, st, dil), oracle.conv2d_derived(x, wt, pad, st, dil))


GRID_T = [  # (h, w, c, f, r, s, pad, stride, dil, opad)
    (2, 2, 3, 2, 4, 4, 1, 2, 1, 0), (3, 4, 2, 3, 4, 4, 1, 2, 1, 0), (4, 3, 2, 2, 3, 3, 1, 1, 1, 0),
    (3, 3, 2, 2, 3, 3, 0, 2, 2, 1), (5, 4, 1, 2, 9, 9, 4, 2, 1, 1), (3, 3, 2, 2, 2, 3, 0, 3, 1, 2),
    (4, 4, 3, 1, 5, 5, 2, 1, 1, 0),
]


@pytest.mark.parametrize("h,w,c,f,r,s,pad,st,dil,op", GRID_T)
def test_convt_library_and_derivation_identity(h, w, c, f, r, s, pad, st, dil, op):
    x = _ints((2, h, w, c), 31 + h)
    wt = _ints((c, f, r, s), 32 + w)
    y = oracle.conv_transpose2d(x, wt, pad, st, dil, op)
    assert np.array_equal(y, _torch_convt(x, wt, pad, st, dil, op))
    assert np.array_equal(y, oracle.conv_transpose2d_derived(x, wt, pad, st, dil, op))


@pytest.mark.parametrize("h,w,c,f,r,s,pad,st,dil,op", GRID_T)
def test_convt_equals_conv_on_zero_inserted_input(h, w, c, f, r, s, pad, st, dil, op):
    """Textbook: ConvT = stride-1 conv over the zero-inserted input, padded by
    dil*(k-1)-pad (plus output_padding at the far end), with the kernel flipped and
    its in/out channels swapped."""
    x = _ints((1, h, w, c), 41 + h)
    wt = _ints((c, f, r, s), 42 + w)
    hz, wz = (h - 1) * st + 1, (w - 1) * st + 1
    xz = np.zeros((1, hz, wz, c))
    xz[:, ::st, ::st, :] = x
    ph, pw = dil * (r - 1) - pad, dil * (s - 1) - pad
    if ph < 0 or pw < 0:
        pytest.skip("negative equivalent padding")
    xz = np.pad(xz, ((0, 0), (ph, ph + op), (pw, pw + op), (0, 0)))
    wflip = np.ascontiguousarray(wt[:, :, ::-1, ::-1].transpose(1, 0, 2, 3))
    want = oracle.conv2d(xz, wflip, 0, 1, dil)
    assert np.array_equal(oracle.conv_transpose2d(x, wt, pad, st, dil, op), want)


@pytest.mark.parametrize("h,w,c,f,r,s,pad,st,dil", GRID)
def test_adjointness(h, w, c, f, r, s, pad, st, dil):
    """<conv(x;W), y> == <x, convT(y;W)>, output_padding chosen so shapes match."""
    x = _ints((1, h, w, c), 51 + h)
    wt = _ints((f, c, r, s), 52 + w)
    y0 = oracle.conv2d(x, wt, pad, st, dil)
    oh = y0.shape[1]
    ow = y0.shape[2]
    oph = h - ((oh - 1) * st - 2 * pad + dil * (r - 1) + 1)
    opw = w - ((ow - 1) * st - 2 * pad + dil * (s - 1) + 1)
    if oph != opw or not (0 <= oph < max(st, dil)):
        pytest.skip("output_padding not representable")
    yv = _ints(y0.shape, 53 + h)
    xt = oracle.conv_transpose2d(yv, wt, pad, st, dil, oph)   # wt is [f,c,r,s] = convT [in=f, out=c]
    assert xt.shape == x.shape
    assert float(np.sum(y0 * yv)) == float(np.sum(x * xt))


@pytest.mark.parametrize("pad,st,dil,r,s", [(1, 1, 1, 3, 3), (0, 1, 1, 3, 3), (2, 2, 1, 5, 5),
                                            (2, 1, 2, 3, 3), (0, 2, 1, 4, 4), (4, 2, 1, 9, 9)])
def test_closed_form_all_ones(pad, st, dil, r, s):
    """X == 1, W == 1: Y = C * (number of window positions that land in the image),
    counted here by summing a zero-padded indicator over numpy windows."""
    h, w, c, f = 9, 8, 3, 2
    y = oracle.conv2d(np.ones((1, h, w, c)), np.ones((f, c, r, s)), pad, st, dil)
    ind = np.pad(np.ones((h, w)), pad)
    win = np.lib.stride_tricks.sliding_window_view(ind, (dil * (r - 1) + 1, dil * (s - 1) + 1))
    cnt = win[::st, ::st, ::dil, ::dil].sum(axis=(2, 3))
    for k in range(f):
        assert np.array_equal(y[0, :, :, k], c * cnt)


def test_1x1_conv_is_matmul():
    x = np.random.default_rng(0).standard_normal((2, 5, 7, 6))
    w = np.random.default_rng(1).standard_normal((4, 6, 1, 1))
    y = oracle.conv2d(x, w)
    np.testing.assert_allclose(y, x @ w[:, :, 0, 0].T, rtol=1e-13, atol=1e-13)
    # and OffsetAdd is the identity map for r = s = 1, p = 0 (SURVEY 8(d) note)
    T = oracle.merged_gemm(x, oracle.weight_dlt_conv2d(w))
    assert np.array_equal(oracle.offset_add(T, 2, 5, 7, 4, 1, 1).reshape(-1, 4), T)


def test_gemm_against_numpy():
    a = np.random.default_rng(2).standard_normal((37, 19))
    b = np.random.default_rng(3).standard_normal((23, 19))
    np.testing.assert_allclose(oracle.gemm_nt(a, b), a @ b.T, rtol=1e-13, atol=1e-13)


def test_weight_dlt_is_eq_layout_k():
    """Eq. layout-K realised with numpy reshapes: K[r,s,f,c] = W[f,c,r,s],
    K' = K flattened over (r, s, f) -> [(r*S+s)*F+f, c]; and it is a bijection."""
    f, c, r, s = 3, 5, 2, 4
    w = np.arange(f * c * r * s, dtype=np.float64).reshape(f, c, r, s)
    K = w.transpose(2, 3, 0, 1)
    assert np.array_equal(oracle.weight_dlt_conv2d(w), K.reshape(r * s * f, c))
    assert sorted(oracle.weight_dlt_conv2d(w).ravel()) == sorted(w.ravel())
    wt = np.arange(c * f * r * s, dtype=np.float64).reshape(c, f, r, s)
    assert np.array_equal(oracle.weight_dlt_convt(wt), wt.transpose(2, 3, 1, 0).reshape(r * s * f, c))


@pytest.mark.parametrize("where", ["row_end", "image_end"])
def test_row_wrap_sentinel_q5(where):
    """Reading Q5: bounds are per spatial dimension.  X one-hot at (0, W-1) [or
    (H-1, W-1)] of image 0, W == 1, 3x3 pad 1: only outputs whose 3x3 window covers
    that pixel are non-zero (= C); a flattened-m bound check would also light
    (1, 0) [or image 1's (0, 0)]."""
    n, h, w, c = 2, 4, 5, 3
    x = np.zeros((n, h, w, c))
    ph = 0 if where == "row_end" else h - 1
    x[0, ph, w - 1, :] = 1.0
    wt = np.ones((1, c, 3, 3))
    for y in (oracle.conv2d(x, wt, 1), oracle.conv2d_derived(x, wt, 1)):
        nz = {tuple(v) for v in np.argwhere(y[..., 0] != 0)}
        want = {(0, a, b) for a in range(h) for b in range(w) if abs(a - ph) <= 1 and abs(b - (w - 1)) <= 1}
        assert nz == want
        assert all(y[k][..., 0] == c for k in want)


def test_convt_tap_table_golden():
    """Probe the selective addition with one-hot T entries and compare the
    (output-row parity, kernel row, input-row offset) triples with the golden table."""
    table = {tuple(r) for r in _golden("convt_tap_table_4x4_s2_p1.txt")}
    n, h, w, f, r, s = 1, 4, 4, 1, 4, 4
    found = set()
    for ih, i in itertools.product(range(h), range(r)):
        T = np.zeros((n * h * w, r * s * f))
        T[ih * w + 1, (i * s + 1) * f] = 1.0          # input column 1, kernel column 1
        y = oracle.selective_add(T, n, h, w, f, r, s, pad=1, stride=2)
        for oh, ow in np.argwhere(y[0, :, :, 0] != 0):
            q, par = divmod(int(oh), 2)
            found.add((par, i, ih - q))
    assert found == table
    # every interior output sums exactly 2x2 = 4 of the 16 taps
    y1 = oracle.selective_add(np.ones((n * h * w, r * s * f)), n, h, w, f, r, s, pad=1, stride=2)
    assert np.all(y1[0, 1:-1, 1:-1, 0] == 4)


def test_offset_add_counts_in_bounds_taps():
    n, h, w, f, r, s = 2, 5, 6, 2, 3, 3
    y = oracle.offset_add(np.ones((n * h * w, r * s * f)), n, h, w, f, r, s, pad=1)
    ones = oracle.conv2d(np.ones((n, h, w, 1)), np.ones((1, 1, r, s)), pad=1)
    assert np.array_equal(y, np.repeat(ones, f, axis=3))


def test_configured_layers_sampled_small():
    """The configured shapes (ollie_synth) at reduced batch: derived == direct, integer mode."""
    for name in ("motivating", "infogan"):
        for li, layer in enumerate(syn.CONFIGS[name]):
            lay = layer.with_batch(1)
            x, w = syn.layer_inputs(lay, syn.config_seed(name, li), exact_int=True)
            if lay.transposed:
                a = oracle.conv_transpose2d(x, w, lay.pad, lay.stride, lay.dilation, lay.output_padding)
                b = oracle.conv_transpose2d_derived(x, w, lay.pad, lay.stride, lay.dilation, lay.output_padding)
            else:
                a = oracle.conv2d(x, w, lay.pad, lay.stride, lay.dilation)
                b = oracle.conv2d_derived(x, w, lay.pad, lay.stride, lay.dilation)
            assert a.shape == (1, lay.oh, lay.ow, lay.f)
            assert np.array_equal(a, b)


# ----------------------------------------------------------------------------- im2col ("tap folding") eOperator
FOLD = [  # (h, w, c, f, r, s, pad, stride, dil, kp)
    (6, 7, 1, 4, 5, 5, 2, 1, 1, 32), (5, 6, 3, 2, 3, 3, 1, 1, 1, 32), (7, 7, 2, 2, 3, 3, 1, 2, 1, 24),
    (8, 6, 1, 3, 3, 3, 2, 1, 2, 16), (9, 9, 1, 2, 9, 9, 4, 1, 1, 88),
]


@pytest.mark.parametrize("h,w,c,f,r,s,pad,st,dil,kp", FOLD)
def test_tap_fold_derivation_exact(h, w, c, f, r, s, pad, st, dil, kp):
    """conv(X, W) == tap_fold(X) . weight_fold(W)^T exactly in integer mode (the im2col derivation),
    tap_fold's columns are the textbook sliding windows in (i, j, c) order, and the padding columns
    k >= r*s*c are zero."""
    x = _ints((2, h, w, c), 31 + h)
    wt = _ints((f, c, r, s), 32 + w)
    a = oracle.tap_fold(x, r, s, pad, st, dil, kp)
    wf = oracle.weight_fold(wt, kp)
    assert np.array_equal(a @ wf.T, oracle.conv2d(x, wt, pad, st, dil))
    assert not a[..., r * s * c:].any()
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    win = np.lib.stride_tricks.sliding_window_view(xp, (dil * (r - 1) + 1, dil * (s - 1) + 1), axis=(1, 2))
    win = win[:, ::st, ::st, :, ::dil, ::dil]                        # n, OH, OW, c, r, s
    cols = win.transpose(0, 1, 2, 4, 5, 3).reshape(win.shape[0], win.shape[1], win.shape[2], -1)   # (r, s, c)
    assert np.array_equal(a[..., :r * s * c], cols)


def test_tap_fold_one_hot_positions():
    """A single one at input pixel (2, 3): column (i, j) of output (oy, ox) is 1 exactly where
    oy - 2 + i = 2 and ox - 2 + j = 3 (5x5, pad 2, stride 1)."""
    x = np.zeros((1, 6, 7, 1))
    x[0, 2, 3, 0] = 1
    a = oracle.tap_fold(x, 5, 5, 2, 1, 1, 25)
    for oy in range(6):
        for ox in range(7):
            for i in range(5):
                for j in range(5):
                    want = 1.0 if (oy - 2 + i == 2 and ox - 2 + j == 3) else 0.0
                    assert a[0, oy, ox, i * 5 + j] == want
