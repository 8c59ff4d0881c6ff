"""NEXT-1: the dilated -> non-dilated derivation of CSRNet's dilated convolution (SURVEY
8(f) NEXT-1), run entirely in libollie kernels:

    Y = batch_to_space( dense_conv_{pad = p/d}( space_to_batch(X) ) )

For stride 1 and pad p = d*k, output row d*u + a of a dilation-d convolution reads input rows
d*(u + i - k) + a only, i.e. the residue class a of the input, densely (expression splitting by
residue).  space_to_batch / batch_to_space are layout DLT eOperators (eops.py; affine
when the image is a multiple of d, so they take the gather fast path) and the middle step is the
ordinary derived convolution on d*d*n images of (h/d) x (w/d) with the same weights.  The direct
form (the fused kernel with tap offsets scaled by d) is the comparison (C2).
"""
from __future__ import annotations

import torch

from . import eops
from . import ollie as _o
from .layers import DerivedConv

_TORCH = {"bf16": torch.bfloat16, "tf32": torch.float32}
_CODE = {"bf16": _o.BF16, "tf32": _o.FP32}   # eOperator storage codes


class DilatedAsDense:
    """Conv2d with dilation d > 1, stride 1, pad a multiple of d, as s2b -> dense conv -> b2s."""

    def __init__(self, n, c, h, w, f, r, s, pad, dilation, dtype="bf16", plan=_o.PLAN_AUTO, device="cuda"):
        d = int(dilation)
        if d < 2 or pad % d:
            raise ValueError("DilatedAsDense needs dilation >= 2 and pad a multiple of the dilation")
        self.n, self.c, self.h, self.w, self.f, self.d = n, c, h, w, f, d
        self.oh = h + 2 * pad - d * (r - 1)
        self.ow = w + 2 * pad - d * (s - 1)
        self.hs, self.ws = -(-h // d), -(-w // d)
        code = _CODE[dtype]
        self.s2b = _o.make_eop(eops.space_to_batch(n, h, w, c, d), [code], code)
        self.conv = DerivedConv(d * d * n, c, self.hs, self.ws, f, r, s, pad=pad // d, dtype=dtype, plan=plan,
                                device=device)
        # the dense conv's output may exceed oh x ow by < d rows / cols (cropped by b2s)
        self.b2s = _o.make_eop(eops.batch_to_space(n, self.conv.oh, self.conv.ow, f, d, self.oh, self.ow), [code], code)
        self.xs = torch.empty(d * d * n, self.hs, self.ws, c, dtype=_TORCH[dtype], device=device)
        self.ys = self.conv.new_output()

    @classmethod
    def from_layer(cls, layer, plan=_o.PLAN_AUTO, device="cuda"):
        assert layer.stride == 1 and not layer.transposed
        return cls(layer.n, layer.c, layer.h, layer.w, layer.f, layer.r, layer.s, layer.pad, layer.dilation,
                   layer.dtype, plan, device)

    def prepare(self, weight: torch.Tensor):
        self.conv.prepare(weight)
        return self

    def new_output(self):
        return torch.empty(self.n, self.oh, self.ow, self.f, dtype=self.xs.dtype, device=self.xs.device)

    def __call__(self, x: torch.Tensor, y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        if y is None:
            y = self.new_output()
        _o.eop_eval(self.s2b, [x], self.xs, stream)
        self.conv(self.xs, self.ys, stream)
        _o.eop_eval(self.b2s, [self.ys], y, stream)
        return y

    def launches(self) -> int:
        return 2 + (2 if self.conv.resolved_plan() == "unfused" else 1)
