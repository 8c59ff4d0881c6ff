"""Layer objects over the C ABI: own the prepared weight (compile-time DLT)
and the unfused-plan workspace; calling one runs the derived program on the GPU.
Device memory comes from torch; every computation is a libollie kernel."""
from __future__ import annotations

import os

import torch

from . import ollie as _o

_DT = {"bf16": _o.BF16, "tf32": _o.TF32}

# Plans are tuned with back-to-back bursts (warm L2, the PDL overlap of a chain of layers included);
# OLLIE_TUNE_COLD=1 times every candidate from an evicted L2 instead (ollie_autotune_derived_cold).
# Measured on the bench's flushed steps (r02): cold tuning changed a few small-layer plans and made
# the ResNet-18 / DCGAN steps 2-4% slower, so warm stays the default.
_TUNE_COLD = os.environ.get("OLLIE_TUNE_COLD", "0") == "1"
_FLUSH = {}


def _flush_buffer(device):
    """A device buffer of 2x the L2 size, allocated once per device (autotune's L2 eviction)."""
    key = torch.device(device).index or 0
    if key not in _FLUSH:
        l2 = torch.cuda.get_device_properties(key).L2_cache_size
        _FLUSH[key] = torch.empty(max(2 * l2, 64 << 20), dtype=torch.uint8, device=device)
    return _FLUSH[key]
_TORCH = {"bf16": torch.bfloat16, "tf32": torch.float32}


class DerivedConv:
    """Conv2d (transposed=False) or ConvTranspose2d (transposed=True) as the derived
    program merged-GEMM + OffsetAdd / selective addition."""

    def __init__(self, n, c, h, w, f, r, s, pad=0, stride=1, dilation=1, output_padding=0,
                 transposed=False, dtype="bf16", plan=_o.PLAN_AUTO, device="cuda", autotune=True):
        self.shape = _o.conv_shape(n, c, h, w, f, r, s, pad, stride, dilation, output_padding)
        self.transposed = bool(transposed)
        self.dtype = dtype
        self.code = _DT[dtype]
        self.plan = plan
        self.device = torch.device(device)
        self.oh, self.ow = _o.output_hw(self.shape, self.transposed)
        self.w_prep = torch.empty(r * s * f, c, dtype=_TORCH[dtype], device=self.device)
        nbytes = _o.workspace_bytes(self.shape, self.code, plan, self.transposed)
        self.autotune = autotune and plan == _o.PLAN_AUTO
        if self.autotune:
            # the unfused and GEMM_RED plans are autotune candidates when their workspaces fit a few
            # GB (B200: 180 GB HBM; FSRCNN's 9x9 ConvT needs a 1.4 GB T)
            unf = _o.workspace_bytes(self.shape, self.code, _o.PLAN_UNFUSED, self.transposed)
            if unf <= (4 << 30):
                nbytes = max(nbytes, unf)
            red = _o.workspace_bytes(self.shape, self.code, _o.PLAN_GEMM_RED, self.transposed)
            if red <= (4 << 30):
                nbytes = max(nbytes, red)
        self.ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=self.device) if nbytes else None
        self.ws_bytes = nbytes
        self._tuned = False

    @classmethod
    def from_layer(cls, layer, plan=_o.PLAN_AUTO, device="cuda", autotune=True):
        return cls(layer.n, layer.c, layer.h, layer.w, layer.f, layer.r, layer.s, layer.pad, layer.stride,
                   layer.dilation, layer.output_padding, layer.transposed, layer.dtype, plan, device, autotune)

    def prepare(self, weight: torch.Tensor, stream=None):
        """a0: weight DLT, once ("compile time").  weight is PyTorch-layout, on the device."""
        weight = weight.contiguous()
        if self.transposed:
            _o.prepare_weight_convtranspose2d(self.shape, self.code, weight, self.w_prep, stream)
        else:
            _o.prepare_weight_conv2d(self.shape, self.code, weight, self.w_prep, stream)
        return self

    def resolved_plan(self) -> str:
        """'fused', 'unfused', 'gemm_red' or 'identity' (unfused GEMM writing Y; OffsetAdd eliminated)."""
        d = _o.plan_describe(self.shape, self.code, self.plan, self.transposed)
        return "identity" if d.startswith("unfused-identity") else d.split()[0]

    def out_shape(self):
        return (self.shape.n, self.oh, self.ow, self.shape.f)

    def new_output(self):
        return torch.empty(self.out_shape(), dtype=_TORCH[self.dtype], device=self.device)

    def __call__(self, x: torch.Tensor, y: torch.Tensor | None = None, stream=None, *, bias=None, residual=None,
                 act: int = _o.ACT_NONE, alpha=None) -> torch.Tensor:
        """Y = act(conv(x) + bias[f] + residual) -- the element-wise epilogue (NEXT-3) runs
        inside whichever kernel writes Y; bias / alpha are fp32 [f], residual is NHWC like Y."""
        if y is None:
            y = self.new_output()
        epi = None
        if bias is not None or residual is not None or act != _o.ACT_NONE:
            epi = _o.make_epilogue(bias, residual, act, alpha)
        if self.autotune and not self._tuned:
            # first call: pick the plan by measurement; not during graph capture
            if not torch.cuda.is_current_stream_capturing():
                # candidates write a scratch output: y may alias the residual (in-place epilogue)
                scratch = self.new_output()
                if _TUNE_COLD:
                    _o.autotune_derived_cold(self.shape, self.code, self.transposed, x, self.w_prep, scratch,
                                             _flush_buffer(self.device), self.ws, self.ws_bytes, stream)
                else:
                    _o.autotune_derived(self.shape, self.code, self.transposed, x, self.w_prep, scratch,
                                        self.ws, self.ws_bytes, stream)
                # the last candidate launch still writes `scratch` on `stream`: finish it before the
                # caching allocator may hand the block to other work (one-time cost per layer)
                torch.cuda.synchronize(self.device)
                del scratch
                self._tuned = True
        if epi is None:
            fn = _o.convtranspose2d_derived if self.transposed else _o.conv2d_derived
            fn(self.shape, self.code, x, self.w_prep, y, self.ws, self.ws_bytes, self.plan, stream)
        else:
            fn = _o.convtranspose2d_derived_ex if self.transposed else _o.conv2d_derived_ex
            fn(self.shape, self.code, x, self.w_prep, y, self.ws, self.ws_bytes, self.plan, epi, stream)
        return y
