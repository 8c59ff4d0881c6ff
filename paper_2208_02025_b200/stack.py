"""A sequence of derived layers run through the C ABI, with the layout eOperators the path needs
(TMA wants 16-byte activation rows).

 - The network input, if its rows are narrower than 16 bytes (FSRCNN's c=1), goes through the
   im2col ("tap folding") eOperator when its r*s*c taps fit a 64-wide Matmul K (the layer then
   runs as a 1x1 conv), else through a channel-pad layout eOperator (`eops.channel_pad`).
 - Inside a chained stack, a layer whose output rows would be misaligned for the next layer
   (FSRCNN's f=12) writes its output with zero-padded channels instead: its weight is padded
   with zero output channels at prepare time, so the "channel-pad o OffsetAdd" eOperator pair
   is evaluated inside the layer (fused pair) and no pad launch is needed.
 - Weight padding is a weight-only expression, evaluated once at prepare ("compile") time
    by the libollie eOperator kernel.
Chained stacks (FSRCNN, DCGAN) feed each output to the next layer; independent stacks
(ResNet-18 stages) give every layer its own input.
"""
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


def _pad_spec_3d(d0, d1, d2, p0, p1):
    """[d0, d1, d2] -> [d0 + p0, d1 + p1, d2], zero in the new rows (pad band on dims 0, 1)."""
    ix = lambda it: {"terms": [[1, it, "id", 1]], "const": 0}  # noqa: E731
    return {"inputs": [{"shape": [d0, d1, d2], "pad": [[0, p0], [0, p1], [0, 0]]}],
            "scopes": [{"trav": [[0, d0 + p0], [0, d1 + p1], [0, d2]], "sum": [],
                        "access": [{"tensor": 0, "index": [ix(0), ix(1), ix(2)]}],
                        "body": [["acc", 0]]}]}


def _transpose_spec_4d(d0, d1, d2, d3):
    """[d0, d1, d2, d3] -> [d0, d2, d3, d1] (W[f, c, i, j] -> W[f, i, j, c])."""
    ix = lambda it: {"terms": [[1, it, "id", 1]], "const": 0}  # noqa: E731
    return {"inputs": [{"shape": [d0, d1, d2, d3]}],
            "scopes": [{"trav": [[0, d0], [0, d2], [0, d3], [0, d1]], "sum": [],
                        "access": [{"tensor": 0, "index": [ix(0), ix(3), ix(1), ix(2)]}],
                        "body": [["acc", 0]]}]}


def fold_width(layer) -> int:
    """Padded Matmul K of a tap-folded layer: r*s*c rounded up to a multiple of 16."""
    return -(-(layer.r * layer.s * layer.c) // 16) * 16


def foldable(layer) -> bool:
    """Few-channel Conv2d (pixel rows narrower than 16 bytes, e.g. FSRCNN's c = 1 feature
    extraction) with a multi-tap kernel: run it as im2col ("tap folding") eOperator + 1x1 conv."""
    return (not layer.transposed and layer.r * layer.s > 1 and (layer.c * _ES[layer.dtype]) % 16 != 0
            and fold_width(layer) <= 64)


class StackLayer:
    """One derived layer computing `fout` output channels from `cin` input channels, where
    cin >= layer.c and fout >= layer.f carry zero padding.  fold=True: the layer's input is first
    folded by the im2col eOperator (ollie_tap_fold: the taps move into the Matmul's k, P:993 ->
    P:1342-1352) and the layer runs as a 1x1 conv over fold_width(layer)-wide pixels."""

    def __init__(self, layer, cin, fout, pad_input, plan, device, fold=False):
        self.layer = layer
        self.cin, self.fout = cin, fout
        self.fold = bool(fold)
        self.pad_eop = None
        if self.fold:
            self.kp = fold_width(layer)
            self.padded = replace(layer, c=self.kp, h=layer.oh, w=layer.ow, f=fout, r=1, s=1, pad=0, stride=1,
                                  dilation=1)
            self.fold_shape = _o.conv_shape(layer.n, layer.c, layer.h, layer.w, fout, layer.r, layer.s, layer.pad,
                                            layer.stride, layer.dilation)
            self.x_fold = torch.empty(layer.n, layer.oh, layer.ow, self.kp, dtype=_TORCH[layer.dtype], device=device)
        else:
            self.padded = replace(layer, c=cin, f=fout)
            if pad_input:
                self.pad_eop = _o.make_eop(eops.channel_pad(layer.n, layer.h, layer.w, layer.c, cin),
                                           [_CODE[layer.dtype]], _CODE[layer.dtype])
                self.x_pad = torch.empty(layer.n, layer.h, layer.w, cin, dtype=_TORCH[layer.dtype], device=device)
        self.conv = DerivedConv.from_layer(self.padded, plan=plan, device=device)
        self.y = self.conv.new_output()

    @property
    def y_logical(self):
        """The layer's output without the zero padding channels (a view)."""
        return self.y[..., : self.layer.f]

    def prepare(self, w: torch.Tensor):
        """w in PyTorch layout ([f,c,r,s] conv, [c,f,r,s] convT), on the device."""
        lay = self.layer
        if self.fold:
            # W''[f, (i*S + j)*C + c] = W[f, c, i, j], zero for k >= r*s*c and f >= F (weight-only
            # expressions, evaluated once by the eOperator kernel)
            code = _CODE[lay.dtype]
            rsc = lay.r * lay.s * lay.c
            wt = torch.empty(lay.f, lay.r, lay.s, lay.c, dtype=w.dtype, device=w.device)
            _o.eop_eval(_o.make_eop(_transpose_spec_4d(lay.f, lay.c, lay.r, lay.s), [code], code), [w.contiguous()], wt)
            wp = torch.empty(self.fout, self.kp, 1, dtype=w.dtype, device=w.device)
            _o.eop_eval(_o.make_eop(_pad_spec_3d(lay.f, rsc, 1, self.fout - lay.f, self.kp - rsc), [code], code),
                        [wt.view(lay.f, rsc, 1)], wp)
            self.conv.prepare(wp.view(self.fout, self.kp, 1, 1))
            return self
        if self.cin != lay.c or self.fout != lay.f:
            code = _CODE[lay.dtype]
            rs = lay.r * lay.s
            if lay.transposed:     # [c, f, r, s] -> [cin, fout, r, s]
                spec = _pad_spec_3d(lay.c, lay.f, rs, self.cin - lay.c, self.fout - lay.f)
                wp = torch.empty(self.cin, self.fout, lay.r, lay.s, dtype=w.dtype, device=w.device)
            else:                  # [f, c, r, s] -> [fout, cin, r, s]
                spec = _pad_spec_3d(lay.f, lay.c, rs, self.fout - lay.f, self.cin - lay.c)
                wp = torch.empty(self.fout, self.cin, lay.r, lay.s, dtype=w.dtype, device=w.device)
            _o.eop_eval(_o.make_eop(spec, [code], code), [w.contiguous()], wp)
            w = wp
        self.conv.prepare(w)
        return self

    def __call__(self, x: torch.Tensor, stream=None, y: torch.Tensor | None = None) -> torch.Tensor:
        """y: optional caller-owned output (same shape as self.y) instead of the layer's own buffer."""
        if self.fold:
            _o.tap_fold(self.fold_shape, self.conv.code, x, self.kp, self.x_fold, stream)
            x = self.x_fold
        elif self.pad_eop is not None:
            _o.eop_eval(self.pad_eop, [x], self.x_pad, stream)
            x = self.x_pad
        return self.conv(x, self.y if y is None else y, stream)

    def launches(self) -> int:
        """Kernels one call launches (pad eOp + 1 fused / identity-eliminated, 2 unfused, or 3 for
        GEMM_RED: memset node, GEMM with reductions, finish)."""
        n = 1 if (self.pad_eop is not None or self.fold) else 0
        return n + {"unfused": 2, "gemm_red": 3}.get(self.conv.resolved_plan(), 1)


class DerivedStack:
    def __init__(self, layers, chained: bool, plan=_o.PLAN_AUTO, device="cuda", fold_taps=True):
        self.chained = chained
        self.layers = []
        if chained:
            for a, b in zip(layers, layers[1:]):
                assert (a.n, a.oh, a.ow, a.f) == (b.n, b.h, b.w, b.c), f"{a.name} -> {b.name} does not chain"
        prev_fout = None
        for k, l in enumerate(layers):
            fold = False
            if chained and k > 0:
                cin, pad_in = prev_fout, False
            else:
                cin = padded_channels(l.c, l.dtype)
                pad_in = cin != l.c
                fold = fold_taps and foldable(l)
            last = (not chained) or k == len(layers) - 1
            fout = l.f if last else padded_channels(l.f, l.dtype)
            self.layers.append(StackLayer(l, cin, fout, pad_in, plan, device, fold=fold))
            prev_fout = fout

    def prepare(self, weights):
        for sl, w in zip(self.layers, weights):
            sl.prepare(w)
        return self

    def __call__(self, inputs, stream=None, out=None):
        """inputs: one tensor (chained) or one per layer (independent).  Returns the layers'
        logical outputs (views without padding channels).  out (optional): caller-owned output of
        the last layer (chained) or one per layer (independent), written instead of the layers'
        own buffers -- e.g. a micro-batch's slice of a rank's output shard (parallel.BlockCyclic)."""
        outs = []
        x = inputs if self.chained else None
        last = len(self.layers) - 1
        for k, sl in enumerate(self.layers):
            src = x if self.chained else inputs[k]
            dst = None
            if out is not None and (not self.chained or k == last):
                dst = out if self.chained else out[k]
            y = sl(src, stream, dst)
            outs.append(y[..., : sl.layer.f] if dst is None else y)
            x = y
        return outs

    def launches(self) -> int:
        return sum(sl.launches() for sl in self.layers)
