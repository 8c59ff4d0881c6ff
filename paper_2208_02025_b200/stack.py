"""A sequence of derived layers run through the C ABI, with the layout eOperators the
path needs inserted automatically: when an activation row (c * sizeof(elem))
is not a multiple of 16 bytes, a channel-pad eOperator widens it and the layer's weight
is zero-padded along c at prepare time (a compile-time, weight-only expression,
P:1445-1447) -- both through libollie kernels.  Chained stacks (FSRCNN, DCGAN) feed each
output to the next layer; independent stacks (ResNet-18 stages) give every layer its
own input."""
from __future__ import annotations

from dataclasses import replace

import torch

from . import eops
from . import ollie as _o
from .layers import DerivedConv

_ES = {"bf16": 2, "tf32": 4}
_TORCH = {"bf16": torch.bfloat16, "tf32": torch.float32}
_CODE = {"bf16": _o.BF16, "tf32": _o.FP32}   # eOperator storage codes


def padded_channels(c: int, dtype: str) -> int:
    q = 16 // _ES[dtype]
    return -(-c // q) * q


class StackLayer:
    def __init__(self, layer, plan, device):
        self.layer = layer
        self.cp = padded_channels(layer.c, layer.dtype)
        self.padded = replace(layer, c=self.cp)
        self.conv = DerivedConv.from_layer(self.padded, plan=plan, device=device)
        self.pad_eop = None
        if self.cp != layer.c:
            self.pad_eop = _o.make_eop(eops.channel_pad(layer.n, layer.h, layer.w, layer.c, self.cp),
                                       [_CODE[layer.dtype]], _CODE[layer.dtype])
            self.x_pad = torch.empty(layer.n, layer.h, layer.w, self.cp, dtype=_TORCH[layer.dtype], device=device)
        self.y = self.conv.new_output()

    def prepare(self, w: torch.Tensor):
        """w in PyTorch layout ([f,c,r,s] conv, [c,f,r,s] convT), on the device."""
        lay = self.layer
        if self.cp != lay.c:
            code = _CODE[lay.dtype]
            if lay.transposed:     # [c, f, r, s] -> [cp, f, r, s]
                spec = {"inputs": [{"shape": [lay.c, lay.f * lay.r * lay.s], "pad": [[0, self.cp - lay.c], [0, 0]]}],
                        "scopes": [{"trav": [[0, self.cp], [0, lay.f * lay.r * lay.s]], "sum": [],
                                    "access": [{"tensor": 0, "index": [{"terms": [[1, 0, "id", 1]], "const": 0},
                                                                       {"terms": [[1, 1, "id", 1]], "const": 0}]}],
                                    "body": [["acc", 0]]}]}
                wp = torch.empty(self.cp, lay.f, lay.r, lay.s, dtype=w.dtype, device=w.device)
            else:                  # [f, c, r, s] -> [f, cp, r, s]
                spec = {"inputs": [{"shape": [lay.f, lay.c, lay.r * lay.s],
                                    "pad": [[0, 0], [0, self.cp - lay.c], [0, 0]]}],
                        "scopes": [{"trav": [[0, lay.f], [0, self.cp], [0, lay.r * lay.s]], "sum": [],
                                    "access": [{"tensor": 0, "index": [{"terms": [[1, 0, "id", 1]], "const": 0},
                                                                       {"terms": [[1, 1, "id", 1]], "const": 0},
                                                                       {"terms": [[1, 2, "id", 1]], "const": 0}]}],
                                    "body": [["acc", 0]]}]}
                wp = torch.empty(lay.f, self.cp, lay.r, lay.s, dtype=w.dtype, device=w.device)
            _o.eop_eval(_o.make_eop(spec, [code], code), [w.contiguous()], wp)
            w = wp
        self.conv.prepare(w)
        return self

    def __call__(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        if self.pad_eop is not None:
            _o.eop_eval(self.pad_eop, [x], self.x_pad, stream)
            x = self.x_pad
        return self.conv(x, self.y, stream)

    def launches(self) -> int:
        """Kernels one call launches (pad eOp + 1 fused / identity-eliminated, or 2 unfused)."""
        n = 1 if self.pad_eop is not None else 0
        return n + (1 if self.conv.ws_bytes == 0 else 2)


class DerivedStack:
    def __init__(self, layers, chained: bool, plan=_o.PLAN_AUTO, device="cuda"):
        self.layers = [StackLayer(l, plan, device) for l in layers]
        self.chained = chained
        if chained:
            for a, b in zip(layers, layers[1:]):
                assert (a.n, a.oh, a.ow, a.f) == (b.n, b.h, b.w, b.c), f"{a.name} -> {b.name} does not chain"

    def prepare(self, weights):
        for sl, w in zip(self.layers, weights):
            sl.prepare(w)
        return self

    def __call__(self, inputs, stream=None):
        """inputs: one tensor (chained) or one per layer (independent).  Returns outputs."""
        outs = []
        x = inputs if self.chained else None
        for k, sl in enumerate(self.layers):
            src = x if self.chained else inputs[k]
            y = sl(src, stream)
            outs.append(y)
            x = y
        return outs

    def launches(self) -> int:
        return sum(sl.launches() for sl in self.layers)
