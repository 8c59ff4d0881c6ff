"""Seeded synthetic inputs and the configured layer shapes.

This module is the ONLY code shared by the oracle side (tests, bench cpu_baseline)
and the product side (bench, smoke).  It holds no arithmetic of the method: just
the layer table (BASELINE.json configs, restated in SURVEY.md 8(d)) and seeded
random tensors drawn in fp32 on the CPU and rounded once to the storage dtype
(SURVEY 8(d) "Value distributions"):

    X ~ U(-1, 1)                (zero mean, reading Q12)
    W ~ N(0, 1 / (c*r*s))
    integer mode: X, W uniform over the integers [-4, 4]

Both sides consume the identical rounded host tensors; the oracle upcasts to fp64.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import torch


@dataclass(frozen=True)
class Layer:
    """One Conv2d / ConvTranspose2d layer (P:806-807 caption; SPEC OpNode attrs S:134)."""
    name: str
    n: int
    c: int
    h: int
    w: int
    f: int
    r: int
    s: int
    pad: int = 0
    stride: int = 1
    dilation: int = 1
    output_padding: int = 0
    transposed: bool = False
    dtype: str = "bf16"          # "bf16" | "tf32" (fp32 storage, TF32 MMA)

    @property
    def oh(self) -> int:
        if self.transposed:
            return (self.h - 1) * self.stride - 2 * self.pad + self.dilation * (self.r - 1) + self.output_padding + 1
        return (self.h + 2 * self.pad - self.dilation * (self.r - 1) - 1) // self.stride + 1

    @property
    def ow(self) -> int:
        if self.transposed:
            return (self.w - 1) * self.stride - 2 * self.pad + self.dilation * (self.s - 1) + self.output_padding + 1
        return (self.w + 2 * self.pad - self.dilation * (self.s - 1) - 1) // self.stride + 1

    @property
    def useful_flops(self) -> int:
        """conv 2*n*OH*OW*f*c*r*s (minus nothing for padding: the
        conventional count); convT 2*n*h*w*c*f*r*s."""
        if self.transposed:
            return 2 * self.n * self.h * self.w * self.c * self.f * self.r * self.s
        return 2 * self.n * self.oh * self.ow * self.f * self.c * self.r * self.s

    @property
    def gemm_mnk(self):
        return (self.n * self.h * self.w, self.r * self.s * self.f, self.c)

    def with_batch(self, n: int) -> "Layer":
        return replace(self, n=n)


def _r18(n):
    return [Layer(f"r18_{c}x{hw}_b{n}", n, c, hw, hw, c, 3, 3, pad=1)
            for c, hw in ((64, 56), (128, 28), (256, 14), (512, 7))]


def _r18s2(n):
    return [Layer(f"r18s2_{c}to{2 * c}_b{n}", n, c, hw, hw, 2 * c, 3, 3, pad=1, stride=2)
            for c, hw in ((64, 56), (128, 28), (256, 14))]


# BASELINE.json "configs" restated as concrete layers (seeds 1000+row).
CONFIGS = {
    # configs[0]: motivating example, fp32 storage -> TF32 path
    "motivating": [Layer("motivating_c4_8x8", 1, 4, 8, 8, 4, 3, 3, pad=1, dtype="tf32")],
    # configs[1]: ResNet-18 3x3 layers, batch 16 and batch 1, bf16
    "resnet18": _r18(16) + _r18(1),
    "resnet18_b16": _r18(16),
    "resnet18_b1": _r18(1),
    "resnet18_s2": _r18s2(16),
    # configs[2]: CSRNet back-end dilated 3x3
    "csrnet": [Layer("csrnet_d2_512x64_b16", 16, 512, 64, 64, 512, 3, 3, pad=2, dilation=2)],
    # configs[3]: InfoGAN ConvT (paper Table shape; f=448 reading Q18) and DCGAN generator
    "infogan": [Layer("infogan_t256to448_b16", 16, 256, 2, 2, 448, 4, 4, pad=1, stride=2, transposed=True)],
    # the same layer with fp32 storage / TF32 MMA: the paper's Table row is fp32 (reading Q1)
    "infogan_tf32": [Layer("infogan_t256to448_b16_tf32", 16, 256, 2, 2, 448, 4, 4, pad=1, stride=2,
                           transposed=True, dtype="tf32")],
    "dcgan": [Layer(f"dcgan_t{c}to{f}_b16", 16, c, hw, hw, f, 4, 4, pad=1, stride=2, transposed=True)
              for c, f, hw in ((512, 256, 4), (256, 128, 8), (128, 64, 16), (64, 3, 32))],
    # configs[4]: FSRCNN(56,12,4) x2, batch 64, LR 256x256 (reading Q17).  c=1 and c=12
    # inputs are channel-padded to 8 / 16 by a layout eOperator (TMA 16-B rule, H3).
    "fsrcnn": [
        Layer("fsrcnn_feat_5x5_1to56", 64, 1, 256, 256, 56, 5, 5, pad=2),
        Layer("fsrcnn_shrink_1x1_56to12", 64, 56, 256, 256, 12, 1, 1, pad=0),
        *[Layer(f"fsrcnn_map{k}_3x3_12to12", 64, 12, 256, 256, 12, 3, 3, pad=1) for k in range(4)],
        Layer("fsrcnn_expand_1x1_12to56", 64, 12, 256, 256, 56, 1, 1, pad=0),
        Layer("fsrcnn_deconv_9x9s2_56to1", 64, 56, 256, 256, 1, 9, 9, pad=4, stride=2,
              output_padding=1, transposed=True),
    ],
    # paper Table conv-perf-detail Conv3x3 row, fp32 storage -> TF32
    "paper_conv3x3": [Layer("paper_conv3x3_512x7_b1", 1, 512, 7, 7, 512, 3, 3, pad=1, dtype="tf32")],
}


def torch_dtype(dtype: str) -> torch.dtype:
    return {"bf16": torch.bfloat16, "tf32": torch.float32, "fp32": torch.float32}[dtype]


def _gen(seed: int) -> torch.Generator:
    return torch.Generator().manual_seed(int(seed))


def uniform(shape, seed: int, dtype: str = "bf16", lo: float = -1.0, hi: float = 1.0) -> torch.Tensor:
    g = _gen(seed)
    t = torch.rand(tuple(shape), generator=g, dtype=torch.float32) * (hi - lo) + lo
    return t.to(torch_dtype(dtype))


def normal(shape, seed: int, std: float, dtype: str = "bf16") -> torch.Tensor:
    g = _gen(seed)
    t = torch.randn(tuple(shape), generator=g, dtype=torch.float32) * std
    return t.to(torch_dtype(dtype))


def integers(shape, seed: int, dtype: str = "bf16", lo: int = -4, hi: int = 4) -> torch.Tensor:
    """Integer mode: exact in bf16 / TF32, so fp32 accumulation is exact."""
    g = _gen(seed)
    t = torch.randint(lo, hi + 1, tuple(shape), generator=g, dtype=torch.int64).to(torch.float32)
    return t.to(torch_dtype(dtype))


def layer_inputs(layer: Layer, seed: int, exact_int: bool = False):
    """(x_nhwc, w) on the CPU, already rounded to the layer's storage dtype.
    w is [f,c,r,s] for Conv2d and [c,f,r,s] for ConvTranspose2d (PyTorch layouts)."""
    xs = (layer.n, layer.h, layer.w, layer.c)
    ws = (layer.c, layer.f, layer.r, layer.s) if layer.transposed else (layer.f, layer.c, layer.r, layer.s)
    if exact_int:
        return integers(xs, seed, layer.dtype), integers(ws, seed + 1, layer.dtype)
    std = (1.0 / (layer.c * layer.r * layer.s)) ** 0.5
    return uniform(xs, seed, layer.dtype), normal(ws, seed + 1, std, layer.dtype)


def config_seed(config_name: str, layer_index: int) -> int:
    """seed = 1000 + row index (stable per config / layer)."""
    base = sorted(CONFIGS).index(config_name) * 100
    return 1000 + base + layer_index


# --------------------------------------------------------------------------- NEXT-4 G2BMM workload
@dataclass(frozen=True)
class G2:
    """LongFormer dilated sliding-window attention scores as G2BMM:
    A = queries, B = keys, [batch, L, K]; band half-width W and dilation d (reading R4)."""
    name: str
    batch: int
    L: int
    K: int
    W: int
    d: int
    dtype: str = "bf16"

    @property
    def flops(self) -> float:        # multiply-adds inside the sequence count, x2
        n = 0
        for w in range(2 * self.W + 1):
            off = self.d * (w - self.W)
            n += max(0, self.L - abs(off))
        return 2.0 * self.batch * self.K * n

    @property
    def bytes(self) -> float:        # |A| + |B| + |out|
        es = 2 if self.dtype == "bf16" else 4
        return es * (2 * self.batch * self.L * self.K + self.batch * self.L * (2 * self.W + 1))


G2_CONFIGS = {
    "longformer": [G2("longformer_8x10000x64_w256_d4", 8, 10000, 64, 256, 4)],
}


def g2bmm_inputs(g: G2, seed: int, exact_int: bool = False):
    """A, B ~ U(-1, 1) rounded to the storage dtype (or integers in [-4, 4]), [batch, L, K]."""
    gen = torch.Generator().manual_seed(seed)
    shp = (g.batch, g.L, g.K)
    if exact_int:
        a = torch.randint(-4, 5, shp, generator=gen).float()
        b = torch.randint(-4, 5, shp, generator=gen).float()
    else:
        a = torch.rand(shp, generator=gen) * 2 - 1
        b = torch.rand(shp, generator=gen) * 2 - 1
    dt = torch_dtype(g.dtype)
    return a.to(dt), b.to(dt)
