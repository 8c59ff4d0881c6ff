"""Thin ctypes binding of libollie (include/ollie.h) -- argument marshalling only.

Every function here has the name of the C entry point without the ``ollie_`` prefix,
takes torch CUDA tensors (or raw device pointers) and the current torch stream, and
raises :class:`OllieError` on a non-OK status.  No step of the hot path runs in
Python: if ``libollie.so`` is missing or fails to load, importing this module raises
(there is no CPU fallback).  PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_char_p, c_float, c_int, c_int32, c_int64, c_size_t, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libollie.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libollie.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

# ----------------------------------------------------------------------------- ABI types
OK, E_INVALID, E_UNSUPPORTED, E_WORKSPACE, E_OOB, E_ALIGN, E_CUDA = 0, -1, -2, -3, -4, -5, -6
BF16, TF32, FP32 = 0, 1, 2
PLAN_AUTO, PLAN_FUSED, PLAN_UNFUSED, PLAN_GEMM_RED, PLAN_ROWSTREAM = 0, 1, 2, 3, 4
PLAN_ROWSTREAM_YSUM, PLAN_ROWSTREAM_DIRECT = 5, 6
PLAN_SMALL = 7                      # the fused program on CUDA cores, layers of <= 2^22 multiply-adds
ATOM_ITER, ATOM_FLOORDIV, ATOM_MOD = 0, 1, 2
OP_PUSH_ACCESS, OP_PUSH_CONST, OP_ADD, OP_MUL, OP_SUB, OP_NEG, OP_MAX, OP_MIN = range(8)
MAX_DIMS, MAX_TERMS, MAX_ACCESS, MAX_INSTR, MAX_INPUTS = 8, 8, 8, 32, 8
ACT_NONE, ACT_RELU, ACT_PRELU = 0, 1, 2
G2BMM_DERIVED, G2BMM_DIRECT = 0, 1


class ConvShape(Structure):
    _fields_ = [("n", c_int64), ("c", c_int64), ("h", c_int64), ("w", c_int64),
                ("f", c_int64), ("r", c_int64), ("s", c_int64),
                ("pad", c_int32), ("stride", c_int32), ("dilation", c_int32), ("output_padding", c_int32)]


class Term(Structure):
    _fields_ = [("iter", c_int32), ("kind", c_int32), ("div", c_int64), ("coef", c_int64)]


class Index(Structure):
    _fields_ = [("nterms", c_int32), ("term", Term * MAX_TERMS), ("c0", c_int64)]


class Access(Structure):
    _fields_ = [("tensor", c_int32), ("ndim", c_int32), ("idx", Index * MAX_DIMS)]


class Tensor(Structure):
    _fields_ = [("ndim", c_int32), ("shape", c_int64 * MAX_DIMS), ("pad_lo", c_int64 * MAX_DIMS),
                ("pad_hi", c_int64 * MAX_DIMS), ("dtype", c_int)]


class Instr(Structure):
    _fields_ = [("op", c_int32), ("arg", c_int32), ("cval", c_float)]


class Scope(Structure):
    _fields_ = [("n_trav", c_int32), ("trav_lo", c_int64 * MAX_DIMS), ("trav_hi", c_int64 * MAX_DIMS),
                ("n_sum", c_int32), ("sum_lo", c_int64 * MAX_DIMS), ("sum_hi", c_int64 * MAX_DIMS),
                ("n_acc", c_int32), ("acc", Access * MAX_ACCESS),
                ("n_ins", c_int32), ("body", Instr * MAX_INSTR),
                ("pad_lo", c_int64 * MAX_DIMS), ("pad_hi", c_int64 * MAX_DIMS)]


class Eop(Structure):
    _fields_ = [("n_in", c_int32), ("in_", Tensor * MAX_INPUTS), ("out_dtype", c_int),
                ("n_scopes", c_int32), ("scope", Scope * 2)]


class Epilogue(Structure):
    _fields_ = [("bias", c_void_p), ("residual", c_void_p), ("act", c_int32), ("alpha", c_void_p)]


class EopInfo(Structure):
    _fields_ = [("is_identity", c_int32), ("pure_indexing", c_int32), ("out_elems", c_int64),
                ("bytes_in", c_int64), ("bytes_out", c_int64)]


_P = POINTER
_sig = {
    "ollie_abi_version": (c_int, []),
    "ollie_status_string": (c_char_p, [c_int]),
    "ollie_last_error": (c_char_p, []),
    "ollie_output_hw": (c_int, [_P(ConvShape), c_int, _P(c_int64), _P(c_int64)]),
    "ollie_prepared_weight_bytes": (c_size_t, [_P(ConvShape), c_int]),
    "ollie_prepare_weight_conv2d": (c_int, [_P(ConvShape), c_int, c_void_p, c_void_p, c_void_p]),
    "ollie_prepare_weight_convtranspose2d": (c_int, [_P(ConvShape), c_int, c_void_p, c_void_p, c_void_p]),
    "ollie_workspace_bytes": (c_size_t, [_P(ConvShape), c_int, c_int, c_int]),
    "ollie_conv2d_derived": (c_int, [_P(ConvShape), c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                     c_int, c_void_p]),
    "ollie_convtranspose2d_derived": (c_int, [_P(ConvShape), c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                              c_size_t, c_int, c_void_p]),
    "ollie_conv2d_derived_ex": (c_int, [_P(ConvShape), c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                        c_int, _P(Epilogue), c_void_p]),
    "ollie_convtranspose2d_derived_ex": (c_int, [_P(ConvShape), c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                                 c_size_t, c_int, _P(Epilogue), c_void_p]),
    "ollie_plan_describe": (c_int, [_P(ConvShape), c_int, c_int, c_int, c_char_p, c_size_t]),
    "ollie_autotune_derived": (c_int, [_P(ConvShape), c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_size_t, c_void_p, _P(c_float)]),
    "ollie_autotune_derived_cold": (c_int, [_P(ConvShape), c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_size_t, c_void_p, c_size_t, c_void_p, _P(c_float)]),
    "ollie_merged_gemm": (c_int, [c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_int64,
                                  c_void_p]),
    "ollie_offset_add": (c_int, [_P(ConvShape), c_int, c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "ollie_tap_fold": (c_int, [_P(ConvShape), c_int, c_void_p, c_int64, c_void_p, c_void_p]),
    "ollie_eop_analyze": (c_int, [_P(Eop), _P(EopInfo)]),
    "ollie_g2bmm": (c_int, [c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_int64,
                            c_int, c_void_p]),
    "ollie_eop_eval": (c_int, [_P(Eop), _P(c_void_p), c_void_p, c_void_p]),
}
for _name, (_res, _args) in _sig.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_sig)


class OllieError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        name = _lib.ollie_status_string(status).decode()
        detail = _lib.ollie_last_error().decode()
        super().__init__(f"{where}: {name}: {detail}")


def _check(st: int, where: str):
    if st != OK:
        raise OllieError(st, where)


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream=None) -> int:
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    import torch
    return torch.cuda.current_stream().cuda_stream


def abi_version() -> int:
    return _lib.ollie_abi_version()


def status_string(st: int) -> str:
    return _lib.ollie_status_string(st).decode()


def last_error() -> str:
    return _lib.ollie_last_error().decode()


def conv_shape(n, c, h, w, f, r, s, pad=0, stride=1, dilation=1, output_padding=0) -> ConvShape:
    return ConvShape(n, c, h, w, f, r, s, pad, stride, dilation, output_padding)


def shape_of_layer(layer) -> ConvShape:
    return conv_shape(layer.n, layer.c, layer.h, layer.w, layer.f, layer.r, layer.s, layer.pad, layer.stride,
                      layer.dilation, layer.output_padding)


def output_hw(shape: ConvShape, transposed: bool):
    oh, ow = c_int64(), c_int64()
    _check(_lib.ollie_output_hw(ctypes.byref(shape), int(transposed), ctypes.byref(oh), ctypes.byref(ow)),
           "ollie_output_hw")
    return oh.value, ow.value


def prepared_weight_bytes(shape: ConvShape, dtype: int) -> int:
    return _lib.ollie_prepared_weight_bytes(ctypes.byref(shape), dtype)


def prepare_weight_conv2d(shape: ConvShape, dtype: int, w, w_prep, stream=None):
    _check(_lib.ollie_prepare_weight_conv2d(ctypes.byref(shape), dtype, _ptr(w), _ptr(w_prep), _stream(stream)),
           "ollie_prepare_weight_conv2d")


def prepare_weight_convtranspose2d(shape: ConvShape, dtype: int, w, w_prep, stream=None):
    _check(_lib.ollie_prepare_weight_convtranspose2d(ctypes.byref(shape), dtype, _ptr(w), _ptr(w_prep),
                                                     _stream(stream)), "ollie_prepare_weight_convtranspose2d")


def workspace_bytes(shape: ConvShape, dtype: int, plan: int = PLAN_AUTO, transposed: bool = False) -> int:
    return _lib.ollie_workspace_bytes(ctypes.byref(shape), dtype, plan, int(transposed))


def conv2d_derived(shape: ConvShape, dtype: int, x, w_prep, y, ws=None, ws_bytes: int = 0,
                   plan: int = PLAN_AUTO, stream=None):
    _check(_lib.ollie_conv2d_derived(ctypes.byref(shape), dtype, _ptr(x), _ptr(w_prep), _ptr(y), _ptr(ws),
                                     ws_bytes, plan, _stream(stream)), "ollie_conv2d_derived")


def convtranspose2d_derived(shape: ConvShape, dtype: int, x, w_prep, y, ws=None, ws_bytes: int = 0,
                            plan: int = PLAN_AUTO, stream=None):
    _check(_lib.ollie_convtranspose2d_derived(ctypes.byref(shape), dtype, _ptr(x), _ptr(w_prep), _ptr(y),
                                              _ptr(ws), ws_bytes, plan, _stream(stream)),
           "ollie_convtranspose2d_derived")


def make_epilogue(bias=None, residual=None, act: int = ACT_NONE, alpha=None) -> Epilogue:
    """NEXT-3 epilogue descriptor: Y = act(acc + bias[f] + residual); tensors must outlive the call."""
    return Epilogue(_ptr(bias), _ptr(residual), int(act), _ptr(alpha))


def conv2d_derived_ex(shape: ConvShape, dtype: int, x, w_prep, y, ws=None, ws_bytes: int = 0,
                      plan: int = PLAN_AUTO, epilogue: Epilogue | None = None, stream=None):
    _check(_lib.ollie_conv2d_derived_ex(ctypes.byref(shape), dtype, _ptr(x), _ptr(w_prep), _ptr(y), _ptr(ws),
                                        ws_bytes, plan, ctypes.byref(epilogue) if epilogue is not None else None,
                                        _stream(stream)), "ollie_conv2d_derived_ex")


def convtranspose2d_derived_ex(shape: ConvShape, dtype: int, x, w_prep, y, ws=None, ws_bytes: int = 0,
                               plan: int = PLAN_AUTO, epilogue: Epilogue | None = None, stream=None):
    _check(_lib.ollie_convtranspose2d_derived_ex(ctypes.byref(shape), dtype, _ptr(x), _ptr(w_prep), _ptr(y),
                                                 _ptr(ws), ws_bytes, plan,
                                                 ctypes.byref(epilogue) if epilogue is not None else None,
                                                 _stream(stream)), "ollie_convtranspose2d_derived_ex")


def plan_describe(shape: ConvShape, dtype: int, plan: int = PLAN_AUTO, transposed: bool = False) -> str:
    buf = ctypes.create_string_buffer(512)
    _check(_lib.ollie_plan_describe(ctypes.byref(shape), dtype, plan, int(transposed), buf, 512), "ollie_plan_describe")
    return buf.value.decode()


def autotune_derived(shape: ConvShape, dtype: int, transposed: bool, x, w_prep, y, ws=None, ws_bytes: int = 0,
                     stream=None) -> float:
    """Time the candidate plans on the device; OLLIE_PLAN_AUTO uses the winner from then on."""
    best = c_float(0.0)
    _check(_lib.ollie_autotune_derived(ctypes.byref(shape), dtype, int(transposed), _ptr(x), _ptr(w_prep), _ptr(y),
                                       _ptr(ws), ws_bytes, _stream(stream), ctypes.byref(best)),
           "ollie_autotune_derived")
    return best.value


def autotune_derived_cold(shape: ConvShape, dtype: int, transposed: bool, x, w_prep, y, flush, ws=None,
                          ws_bytes: int = 0, stream=None) -> float:
    """Same, every candidate timed from an evicted L2 (`flush`: a device buffer >= 2x the L2 size)."""
    best = c_float(0.0)
    _check(_lib.ollie_autotune_derived_cold(ctypes.byref(shape), dtype, int(transposed), _ptr(x), _ptr(w_prep),
                                            _ptr(y), _ptr(ws), ws_bytes, _ptr(flush), flush.numel() * flush.element_size(),
                                            _stream(stream), ctypes.byref(best)),
           "ollie_autotune_derived_cold")
    return best.value


def merged_gemm(M: int, N: int, K: int, dtype: int, A, B, T, ldT: int, stream=None):
    _check(_lib.ollie_merged_gemm(M, N, K, dtype, _ptr(A), _ptr(B), _ptr(T), ldT, _stream(stream)),
           "ollie_merged_gemm")


def offset_add(shape: ConvShape, transposed: bool, T, ldT: int, y_dtype: int, y, stream=None):
    _check(_lib.ollie_offset_add(ctypes.byref(shape), int(transposed), _ptr(T), ldT, y_dtype, _ptr(y),
                                 _stream(stream)), "ollie_offset_add")


def tap_fold(shape: ConvShape, dtype: int, x, kp: int, out, stream=None):
    """im2col ("tap folding") eOperator: out[b, oy, ox, (i*s + j)*c + ch] = x[b, oy*st-p+i*d, ox*st-p+j*d, ch]."""
    _check(_lib.ollie_tap_fold(ctypes.byref(shape), dtype, _ptr(x), kp, _ptr(out), _stream(stream)), "ollie_tap_fold")


# ----------------------------------------------------------------------------- eOperators
_KIND = {"id": ATOM_ITER, "div": ATOM_FLOORDIV, "mod": ATOM_MOD}
_OPS = {"acc": OP_PUSH_ACCESS, "const": OP_PUSH_CONST, "add": OP_ADD, "mul": OP_MUL, "sub": OP_SUB,
        "neg": OP_NEG, "max": OP_MAX, "min": OP_MIN}


def _fill_scope(dst: Scope, sc: dict):
    trav, sums = sc["trav"], sc.get("sum", [])
    dst.n_trav = len(trav)
    for d, (lo, hi) in enumerate(trav):
        dst.trav_lo[d], dst.trav_hi[d] = lo, hi
    dst.n_sum = len(sums)
    for d, (lo, hi) in enumerate(sums):
        dst.sum_lo[d], dst.sum_hi[d] = lo, hi
    dst.n_acc = len(sc["access"])
    for a, acc in enumerate(sc["access"]):
        dst.acc[a].tensor = acc["tensor"]
        dst.acc[a].ndim = len(acc["index"])
        for d, ix in enumerate(acc["index"]):
            dst.acc[a].idx[d].nterms = len(ix["terms"])
            dst.acc[a].idx[d].c0 = ix.get("const", 0)
            for t, (coef, it, kind, div) in enumerate(ix["terms"]):
                dst.acc[a].idx[d].term[t] = Term(it, _KIND[kind], div, coef)
    dst.n_ins = len(sc["body"])
    for p, ins in enumerate(sc["body"]):
        op = _OPS[ins[0]]
        arg = ins[1] if op == OP_PUSH_ACCESS else 0
        cval = float(ins[1]) if op == OP_PUSH_CONST else 0.0
        dst.body[p] = Instr(op, arg, cval)
    for d, (lo, hi) in enumerate(sc.get("pad", []) or []):
        dst.pad_lo[d], dst.pad_hi[d] = lo, hi


def make_eop(spec: dict, in_dtypes=None, out_dtype: int = FP32) -> Eop:
    """Translate the plain-data eOperator spec into the C struct."""
    e = Eop()
    ins = spec["inputs"]
    if len(ins) > MAX_INPUTS or len(spec["scopes"]) > 2:
        raise ValueError("eOperator too large for the ABI")
    e.n_in = len(ins)
    for k, t in enumerate(ins):
        e.in_[k].ndim = len(t["shape"])
        for d, v in enumerate(t["shape"]):
            e.in_[k].shape[d] = v
        for d, (lo, hi) in enumerate(t.get("pad", []) or []):
            e.in_[k].pad_lo[d], e.in_[k].pad_hi[d] = lo, hi
        e.in_[k].dtype = (in_dtypes[k] if in_dtypes is not None else FP32)
    e.out_dtype = out_dtype
    e.n_scopes = len(spec["scopes"])
    for k, sc in enumerate(spec["scopes"]):
        _fill_scope(e.scope[k], sc)
    return e


def eop_analyze(eop: Eop) -> dict:
    info = EopInfo()
    _check(_lib.ollie_eop_analyze(ctypes.byref(eop), ctypes.byref(info)), "ollie_eop_analyze")
    return {"is_identity": bool(info.is_identity), "pure_indexing": bool(info.pure_indexing),
            "out_elems": info.out_elems, "bytes_in": info.bytes_in, "bytes_out": info.bytes_out}


def eop_eval(eop: Eop, inputs, output, stream=None):
    arr = (c_void_p * max(1, len(inputs)))(*[_ptr(t) for t in inputs])
    _check(_lib.ollie_eop_eval(ctypes.byref(eop), arr, _ptr(output), _stream(stream)), "ollie_eop_eval")


def g2bmm(batch: int, L: int, K: int, W: int, d: int, dtype: int, A, B, out, ldo: int | None = None,
          form: int = G2BMM_DERIVED, stream=None):
    """NEXT-4 G2BMM: out[b, m, w] = sum_k A[b, m, k] B[b, m + d(w - W), k], w in [0, 2W] (include/ollie.h)."""
    _check(_lib.ollie_g2bmm(batch, L, K, W, d, dtype, _ptr(A), _ptr(B), _ptr(out),
                            2 * W + 1 if ldo is None else ldo, form, _stream(stream)), "ollie_g2bmm")
