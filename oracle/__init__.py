"""CPU oracle for the derived-convolution hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product package
``paper_2208_02025_b200`` never imports it and shares no code with it; the two
meet only in the seeded input generators of ``ollie_synth.py``.

Everything is fp64.  Conv / ConvT / GEMM / OffsetAdd / selective-add / weight DLT
are nested C loops in ``conv_oracle.c`` (built with gcc, OpenMP); the eOperator
interpreter is pure Python in ``eop_oracle.py`` (small cases only).

Pins (all in ``tests/test_oracle_*.py``, marked ``not gpu``): brute force by
explicit im2col, torch CPU fp64 ``F.conv2d`` / ``F.conv_transpose2d`` as an
independent library, the all-ones worked example, closed forms,
adjointness, the derivation identity, the row-wrap sentinel (Q5),
the ConvT tap table, identity / permutation / round-trip checks for eOps.
The im2col ("tap folding") eOperator and its weight side are pinned by the exact
derivation identity conv == fold(X) . fold(W)^T and by textbook sliding windows.
No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from .eop_oracle import eop_eval, eop_is_identity, eop_bounds_ok  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "conv_oracle.c")
_LIB_DIR = os.path.join(_HERE, "_build")
_LIB = os.path.join(_LIB_DIR, "liboracle.so")
_lock = threading.Lock()
_lib = None

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)


def build_oracle(force: bool = False) -> str:
    """Compile conv_oracle.c with gcc (-O2 -fopenmp).  Building the checker is not using it."""
    os.makedirs(_LIB_DIR, exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build_oracle())
            I = _i64
            lib.oracle_conv_out_size.restype = I
            lib.oracle_conv_out_size.argtypes = [I] * 5
            lib.oracle_convt_out_size.restype = I
            lib.oracle_convt_out_size.argtypes = [I] * 6
            lib.oracle_conv2d.argtypes = [I] * 10 + [_dp] * 3
            lib.oracle_convtranspose2d.argtypes = [I] * 11 + [_dp] * 3
            lib.oracle_gemm_nt.argtypes = [I] * 3 + [_dp] * 3
            lib.oracle_weight_dlt_conv2d.argtypes = [I] * 4 + [_dp] * 2
            lib.oracle_weight_dlt_convt.argtypes = [I] * 4 + [_dp] * 2
            lib.oracle_offset_add.argtypes = [I] * 9 + [_dp] * 2
            lib.oracle_g2bmm.argtypes = [I] * 5 + [_dp] * 3
            lib.oracle_selective_add.argtypes = [I] * 10 + [_dp] * 2
            lib.oracle_num_threads.restype = ctypes.c_int
            lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
            _lib = lib
    return _lib


def _f64(a) -> np.ndarray:
    """Upcast the (already rounded) generated values to contiguous fp64."""
    if hasattr(a, "detach"):  # torch tensor
        a = a.detach().to("cpu").double().numpy()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP thread count for later oracle calls (no effect on the arithmetic)."""
    _load().oracle_set_num_threads(int(n))


def conv_out_size(n, k, pad, stride, dil) -> int:
    return int(_load().oracle_conv_out_size(n, k, pad, stride, dil))


def convt_out_size(n, k, pad, stride, dil, opad=0) -> int:
    return int(_load().oracle_convt_out_size(n, k, pad, stride, dil, opad))


def conv2d(x_nhwc, w_fcrs, pad=0, stride=1, dilation=1) -> np.ndarray:
    """O1: direct Conv2d (cross-correlation, zero padding).  x [n,h,w,c], w [f,c,r,s] -> y [n,OH,OW,f]."""
    x = _f64(x_nhwc)
    w = _f64(w_fcrs)
    n, h, wd, c = x.shape
    f, c2, r, s = w.shape
    assert c == c2
    oh = conv_out_size(h, r, pad, stride, dilation)
    ow = conv_out_size(wd, s, pad, stride, dilation)
    y = np.zeros((n, oh, ow, f), np.float64)
    _load().oracle_conv2d(n, c, h, wd, f, r, s, pad, stride, dilation, _p(x), _p(w), _p(y))
    return y


def conv_transpose2d(x_nhwc, w_cfrs, pad=0, stride=1, dilation=1, output_padding=0) -> np.ndarray:
    """O2: ConvTranspose2d in scatter form.  x [n,h,w,c], w [c,f,r,s] -> y [n,OH,OW,f]."""
    x = _f64(x_nhwc)
    w = _f64(w_cfrs)
    n, h, wd, c = x.shape
    c2, f, r, s = w.shape
    assert c == c2
    oh = convt_out_size(h, r, pad, stride, dilation, output_padding)
    ow = convt_out_size(wd, s, pad, stride, dilation, output_padding)
    y = np.zeros((n, oh, ow, f), np.float64)
    _load().oracle_convtranspose2d(n, c, h, wd, f, r, s, pad, stride, dilation, output_padding,
                                   _p(x), _p(w), _p(y))
    return y


def gemm_nt(a_mk, b_nk) -> np.ndarray:
    """O5: C[m,n] = sum_k A[m,k] B[n,k]."""
    a = _f64(a_mk)
    b = _f64(b_nk)
    m, k = a.shape
    n, k2 = b.shape
    assert k == k2
    cm = np.zeros((m, n), np.float64)
    _load().oracle_gemm_nt(m, n, k, _p(a), _p(b), _p(cm))
    return cm


def weight_dlt_conv2d(w_fcrs) -> np.ndarray:
    """a0 for Conv2d: wp[(i*S+j)*F+f, c] = W[f,c,i,j]  (Eq. layout-K transposed)."""
    w = _f64(w_fcrs)
    f, c, r, s = w.shape
    wp = np.zeros((r * s * f, c), np.float64)
    _load().oracle_weight_dlt_conv2d(f, c, r, s, _p(w), _p(wp))
    return wp


def weight_dlt_convt(w_cfrs) -> np.ndarray:
    """a0 for ConvTranspose2d: wp[(i*S+j)*F+f, c] = W[c,f,i,j]."""
    w = _f64(w_cfrs)
    c, f, r, s = w.shape
    wp = np.zeros((r * s * f, c), np.float64)
    _load().oracle_weight_dlt_convt(c, f, r, s, _p(w), _p(wp))
    return wp


def merged_gemm(x_nhwc, wp) -> np.ndarray:
    """a1+a2: T[n*h*w, r*s*f] = A'[m, c] . K'[c, n]; A' = A is the identity on NHWC."""
    x = _f64(x_nhwc)
    n, h, w, c = x.shape
    return gemm_nt(x.reshape(n * h * w, c), wp)


def offset_add(T, n, h, w, f, r, s, pad=0, stride=1, dilation=1) -> np.ndarray:
    """a3: OffsetAdd eOperator (E7), per-dimension bounds on the 5-D view of T."""
    t = _f64(T)
    assert t.shape == (n * h * w, r * s * f), t.shape
    oh = conv_out_size(h, r, pad, stride, dilation)
    ow = conv_out_size(w, s, pad, stride, dilation)
    y = np.zeros((n, oh, ow, f), np.float64)
    _load().oracle_offset_add(n, h, w, f, r, s, pad, stride, dilation, _p(t), _p(y))
    return y


def selective_add(T, n, h, w, f, r, s, pad=0, stride=1, dilation=1, output_padding=0) -> np.ndarray:
    """a4: ConvTranspose selective addition over the Matmul outputs."""
    t = _f64(T)
    assert t.shape == (n * h * w, r * s * f), t.shape
    oh = convt_out_size(h, r, pad, stride, dilation, output_padding)
    ow = convt_out_size(w, s, pad, stride, dilation, output_padding)
    y = np.zeros((n, oh, ow, f), np.float64)
    _load().oracle_selective_add(n, h, w, f, r, s, pad, stride, dilation, output_padding,
                                 _p(t), _p(y))
    return y


def conv2d_derived(x_nhwc, w_fcrs, pad=0, stride=1, dilation=1) -> np.ndarray:
    """O3 for Conv2d: OffsetAdd(Matmul(A', DLT(K))) -- the paper's derived program, step by step."""
    x = _f64(x_nhwc)
    n, h, w, c = x.shape
    f, _, r, s = np.shape(w_fcrs)
    T = merged_gemm(x, weight_dlt_conv2d(w_fcrs))
    return offset_add(T, n, h, w, f, r, s, pad, stride, dilation)


def conv_transpose2d_derived(x_nhwc, w_cfrs, pad=0, stride=1, dilation=1, output_padding=0):
    """O3 for ConvTranspose2d: SelectiveAdd(Matmul(A', DLT(K))) on the unpadded input."""
    x = _f64(x_nhwc)
    n, h, w, c = x.shape
    _, f, r, s = np.shape(w_cfrs)
    T = merged_gemm(x, weight_dlt_convt(w_cfrs))
    return selective_add(T, n, h, w, f, r, s, pad, stride, dilation, output_padding)


# ----------------------------------------------------------------------------- NEXT-3 epilogue
def epilogue(y, bias=None, residual=None, act: str = "none", alpha=None) -> np.ndarray:
    """Element-wise operators following the convolution ("fused with following
    element-wise operators"; reading Q19), written out in fp64:
        v = y + bias[f] + residual;   relu: max(v, 0);   prelu: v if v > 0 else alpha[f] * v
    y / residual are NHWC [n, OH, OW, f]; bias / alpha are [f]."""
    v = _f64(y).copy()
    if bias is not None:
        v = v + _f64(bias)[None, None, None, :]
    if residual is not None:
        v = v + _f64(residual)
    if act == "relu":
        v = np.where(v > 0, v, 0.0)
    elif act == "prelu":
        v = np.where(v > 0, v, _f64(alpha)[None, None, None, :] * v)
    elif act != "none":
        raise ValueError(f"unknown activation {act!r}")
    return v


# ----------------------------------------------------------------------------- NEXT-1 derivation
def conv2d_dilated_as_dense(x_nhwc, w_fcrs, pad: int, dilation: int) -> np.ndarray:
    """The dilated -> non-dilated derivation ("transforms the dilated convolution into
    non-dilated convolution by expression derivation"), written out step by step: for pad = d*k,
    output rows d*u + a read input rows d*(u + i - k) + a only, so
        X_ab = X[:, a::d, b::d, :]                     (space-to-batch, residue class (a, b))
        Y[:, a::d, b::d, :] = conv2d(X_ab, W, pad=k)   (dense 3x3, same weights)
    Stride 1; pad must be a multiple of the dilation (reading R3)."""
    x = _f64(x_nhwc)
    d = int(dilation)
    if pad % d:
        raise ValueError("pad must be a multiple of the dilation")
    n, h, w, _ = x.shape
    f = np.asarray(w_fcrs).shape[0]
    oh = conv_out_size(h, np.asarray(w_fcrs).shape[2], pad, 1, d)
    ow = conv_out_size(w, np.asarray(w_fcrs).shape[3], pad, 1, d)
    y = np.zeros((n, oh, ow, f))
    for a in range(d):
        for b in range(d):
            xab = x[:, a::d, b::d, :]
            if xab.shape[1] == 0 or xab.shape[2] == 0:
                continue
            yab = conv2d(xab, w_fcrs, pad=pad // d)
            rows, cols = y[:, a::d, b::d, :].shape[1:3]
            y[:, a::d, b::d, :] = yab[:, :rows, :cols, :]
    return y


# ----------------------------------------------------------------------------- NEXT-4 G2BMM
def g2bmm(a_blk, b_blk, W: int, d: int) -> np.ndarray:
    """General-to-band matrix multiplication (P:1109-1118 iterator table; LongFormer),
    reading R4: out[b, m, w] = sum_k A[b, m, k] * B[b, m + d*(w - W), k] for w in [0, 2W],
    0 where the B row leaves [0, L).  fp64 C loops (conv_oracle.c)."""
    lib = _load()
    a, b = _f64(a_blk), _f64(b_blk)
    nb, L, K = a.shape
    out = np.zeros((nb, L, 2 * W + 1))
    lib.oracle_g2bmm(ctypes.c_int64(nb), ctypes.c_int64(L), ctypes.c_int64(K), ctypes.c_int64(W),
                     ctypes.c_int64(d), _p(a), _p(b), _p(out))
    return out


def g2bmm_residue_split(a_blk, b_blk, W: int, d: int) -> np.ndarray:
    """The paper's dilated -> non-dilated derivation of G2BMM, step by step: rows of
    residue r (m = d*u + r) only meet B rows of the same residue, m + d*(w - W) = d*(u + w - W) + r,
    so out[:, r::d] = G2BMM_{d=1}(A[:, r::d], B[:, r::d]) -- a non-dilated band product per class."""
    a, b = _f64(a_blk), _f64(b_blk)
    nb, L, _ = a.shape
    out = np.zeros((nb, L, 2 * W + 1))
    for r in range(d):
        if r < L:
            out[:, r::d] = g2bmm(a[:, r::d], b[:, r::d], W, 1)
    return out


# ----------------------------------------------------------------------------- im2col ("tap folding") eOperator
def tap_fold(x_nhwc, r: int, s: int, pad: int = 0, stride: int = 1, dilation: int = 1, kp: int | None = None) -> np.ndarray:
    """The im2col layout eOperator of a Conv2d -- variable substitution of the conv expression
    (E1) that moves the taps into the reduction index so operator matching
    sees a plain Matmul with k = (i, j, c):
        A'[b, oy, ox, (i*S + j)*C + c] = X[b, oy*st - p + i*d, ox*st - p + j*d, c]
    zero outside the image and for k >= r*s*C up to the padded width kp.  Written out
    per (i, j) tap by strided slicing of the zero-padded input."""
    x = _f64(x_nhwc)
    n, h, w, c = x.shape
    oh = conv_out_size(h, r, pad, stride, dilation)
    ow = conv_out_size(w, s, pad, stride, dilation)
    kp = r * s * c if kp is None else int(kp)
    if kp < r * s * c:
        raise ValueError("kp must cover r*s*c")
    xp = np.zeros((n, h + 2 * pad, w + 2 * pad, c))
    xp[:, pad:pad + h, pad:pad + w, :] = x
    out = np.zeros((n, oh, ow, kp))
    for i in range(r):
        for j in range(s):
            k0 = (i * s + j) * c
            y0, x0 = i * dilation, j * dilation
            out[:, :, :, k0:k0 + c] = xp[:, y0:y0 + stride * (oh - 1) + 1:stride, x0:x0 + stride * (ow - 1) + 1:stride, :]
    return out


def weight_fold(w_fcrs, kp: int | None = None) -> np.ndarray:
    """The weight side of the im2col derivation: W''[f, (i*S + j)*C + c] = W[f, c, i, j], zero for
    k >= r*s*C (the 1x1 conv / Matmul weight that pairs with tap_fold)."""
    w = _f64(w_fcrs)
    f, c, r, s = w.shape
    kp = r * s * c if kp is None else int(kp)
    out = np.zeros((f, kp))
    out[:, :r * s * c] = w.transpose(0, 2, 3, 1).reshape(f, r * s * c)
    return out
