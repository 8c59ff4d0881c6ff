#!/usr/bin/env python
"""Benchmark of the derived-convolution hot path (Ollie, arXiv 2208.02025) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config csrnet] [--impl ours|reference]

A "step" is one pass of the whole hot path over one batch of the configured workload: every
layer of the config runs as its derived program (merged tcgen05 GEMM + OffsetAdd / selective
add, fused or unfused, plus the layout eOperators it needs) through the C ABI.

Headline workload: the largest single-GPU configuration of
BASELINE.json, configs[2] = CSRNet's dilated 3x3 conv (c = f = 512, 64x64, dilation 2) at
batch 16, bf16 -- 309 useful GFLOP per step.  Metric: useful TFLOP/s of the step (higher is
better), with us per layer against same-box cuDNN.  Every other BASELINE config (motivating
example, ResNet-18 b16/b1 and stride-2 stages, InfoGAN in bf16 and TF32, DCGAN, FSRCNN b64,
the paper's Conv3x3 [1,512,7,7] in TF32), the eOperator configs E-b..E-f (OffsetAdd GB/s) and
the G2BMM workload are reported as sub-records of the same JSON line ("suite"): per layer, ours
and cuDNN timed by the SAME method (each layer captured alone in a CUDA graph; "flushed" = L2
flushed before every replay; "warm" = 10 back-to-back calls in one graph), TFLOP/s, GB/s,
fraction of the attainable roofline and the speedup over cuDNN.

Timing: W untimed warm-up steps; then exactly K steps, each preceded by an L2
flush (a 2x L2-size write, then a read of it that retires the dirty lines; both outside the
per-step events), each one CUDA graph replay bracketed by CUDA events on the launching
stream; a barrier + synchronize on both sides of the K steps; max over ranks.

N > 1 (torchrun, NCCL): strong scaling -- the configured batch is sharded block-cyclically
over the ranks (parallel.BlockCyclic; every rank draws the full batch from the same seed as
the 1-GPU run and keeps its images), each rank runs its shard, `value` = the whole batch's
useful flops / the max-over-ranks step time with outputs left sharded; the
a9 all-gather of Y is timed as well, serial and chunk-overlapped on a side stream (8(e) (ii)),
in the "allgather" sub-record.  Layers whose batch does not split run replicated.

`--impl reference` times the fp64 CPU oracle on a bounded sample of the same workload (the
reference arm for this tier); it is the only other place besides tests/ and
__graft_entry__.smoke() that executes oracle/ code, together with the cpu_baseline leg.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import replace

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import ollie_synth as syn  # noqa: E402

HEADLINE = "csrnet"
CHAINED = {"fsrcnn", "dcgan"}
CONFIG_TEXT = {
    "resnet18": "ResNet-18 3x3 conv layers (c=f=64..512, 56x56..7x7) batch 1 and 16, bf16",
    "csrnet": "CSRNet dilated 3x3 conv (dilation=2, c=f=512, 64x64) batch 16",
    "infogan": "InfoGAN ConvTranspose2d 4x4 stride 2 (256->448, 2x2) batch 16, bf16",
    "infogan_tf32": "InfoGAN ConvTranspose2d 4x4 stride 2 (256->448, 2x2) batch 16, TF32 (paper Table row)",
    "dcgan": "DCGAN ConvTranspose2d 4x4 stride 2 generator stack batch 16",
    "fsrcnn": "FSRCNN full conv+convT stack batch 64",
    "motivating": "motivating example 3x3 Conv2d n=1 c=4 h=w=8 f=4 (TF32)",
    "paper_conv3x3": "paper Table Conv3x3 [1,512,7,7] (TF32)",
    "resnet18_s2": "ResNet-18 stride-2 3x3 layers batch 16 (strided extension)",
    "resnet18_b16": "ResNet-18 3x3 conv layers batch 16",
    "resnet18_b1": "ResNet-18 3x3 conv layers batch 1",
}
SUITE = ["motivating", "resnet18", "resnet18_s2", "infogan", "infogan_tf32", "dcgan", "fsrcnn", "paper_conv3x3"]


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            mp = json.load(fh)
        return {"hbm_gbs": mp["hbm_gbs"], "bf16_tflops": mp["bf16_tflops"],
                "bf16_tflops_sustained": mp.get("bf16_tflops_sustained"), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def _es(dtype):
    return 2 if dtype == "bf16" else 4


def _cpu_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "omp_num_threads_env": os.environ.get("OMP_NUM_THREADS")}


# ------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [v.strip() for v in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------- oracle arm
def _oracle_sample(layers, max_flop):
    """Bounded sample of the workload for the CPU oracle: the first images of each layer (a
    conv's images are independent), sized to ~max_flop useful flops (at least one image)."""
    per_layer = max_flop / max(1, len(layers))
    plan = []
    for li, lay in enumerate(layers):
        per_img = lay.useful_flops / lay.n
        k = int(max(1, min(lay.n, per_layer // per_img)))
        plan.append((li, lay, k))
    return plan


def run_oracle_sample(cfg, plan, crop_rows=None):
    """Oracle on the sampled images (crop_rows: only the first rows of each image -- the
    single-thread figure of a large layer); returns (useful flops computed, seconds)."""
    import oracle
    flops = 0
    t0 = time.perf_counter()
    for li, lay, k in plan:
        x, w = syn.layer_inputs(lay.with_batch(k), syn.config_seed(cfg, li))
        if crop_rows is not None and not lay.transposed and crop_rows < lay.h:
            x = x[:, :crop_rows]
            lay = replace(lay, h=crop_rows)
        if lay.transposed:
            oracle.conv_transpose2d(x, w, lay.pad, lay.stride, lay.dilation, lay.output_padding)
        else:
            oracle.conv2d(x, w, lay.pad, lay.stride, lay.dilation)
        flops += lay.useful_flops / lay.n * k
    return flops, time.perf_counter() - t0


def cpu_baseline(cfg, layers, seconds=10.0, max_flop=4e11):
    """The oracle as it stands, on the host cores, on a bounded sample (~`seconds` of work);
    plus a single-thread figure on a smaller sample (SURVEY 8(d) "CPU oracle")."""
    import oracle
    splan = _oracle_sample(layers, max_flop)
    f, t, passes = 0.0, 0.0, 0
    while passes == 0 or (t < seconds and passes < 50):
        f1, t1 = run_oracle_sample(cfg, splan)
        f, t, passes = f + f1, t + t1, passes + 1
    cores = oracle.num_threads()
    out = {"value": f / t / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
           "sample": f"{passes} pass(es) of: " + "; ".join(f"{lay.name}: {k}/{lay.n} images" for _, lay, k in splan),
           "seconds": t, **_cpu_info()}
    # single thread: one image of each layer, large images cropped to their first rows
    one = [(li, lay, 1) for li, lay, _ in splan]
    crop = None
    if sum(l.useful_flops / l.n for _, l, _ in one) > 3e9:
        crop = 8
    oracle.set_num_threads(1)
    try:
        f1, t1 = run_oracle_sample(cfg, one, crop_rows=crop)
    finally:
        oracle.set_num_threads(cores)
    out["single_thread"] = {"value": f1 / t1 / 1e12, "unit": "TFLOP/s", "seconds": t1,
                            "sample": "1 image per layer" + (f", first {crop} input rows" if crop else "")}
    return out


def reference_main(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    cfg = args.config
    layers = syn.CONFIGS[cfg]
    plan = _oracle_sample(layers, args.ref_flop)
    for _ in range(args.warmup):
        run_oracle_sample(cfg, plan)
    times, flops = [], 0
    for _ in range(args.steps):
        f, t = run_oracle_sample(cfg, plan)
        times.append(t)
        flops = f
    ms = 1e3 * statistics.mean(times)
    val = flops / (ms * 1e-3) / 1e12
    sample = "; ".join(f"{lay.name}: {k}/{lay.n} images" for _, lay, k in plan)
    line = {"metric": "derived conv useful TFLOP/s (whole step)", "value": val, "unit": "TFLOP/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, ollie_synth)",
            "config": {"workload": CONFIG_TEXT.get(cfg, cfg), "name": cfg, "sample": sample},
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": sample, **_cpu_info()},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------- GPU helpers
class Flusher:
    """Evicts L2: writes a buffer of 2x the L2 size, then reads it back so the dirty lines are
    retired here (outside the timed events) and not inside the next kernel."""

    def __init__(self, torch, dev):
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
        self.buf = torch.empty(max(2 * l2, 64 << 20), dtype=torch.uint8, device=dev)
        self.sink = torch.empty((), dtype=torch.int64, device=dev)
        self.torch = torch

    def __call__(self, k=0):
        self.buf.fill_(k & 0xFF)
        self.torch.sum(self.buf.view(self.torch.int64), dim=0, out=self.sink)


def _graph(torch, fn, stream, reps=1):
    """CUDA graph of `reps` calls of fn(stream) (after 2 eager warm-up calls)."""
    with torch.cuda.stream(stream):
        for _ in range(2):
            fn(stream)
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps):
            fn(stream)
    torch.cuda.synchronize()
    return g


def time_graph_flushed(torch, fn, stream, flusher, reps=20):
    """Device time (us) of one call of fn(stream) from an evicted L2, measured differentially: a CUDA
    graph of `reps` x (flush + fn) and a graph of `reps` x flush are each timed as one event pair,
    and the difference is divided by reps -- single short replays cannot be timed directly here
    (CUDA event timestamps on this box are quantised to ~2 us).  Median of 3 such measurements."""
    def cap(with_fn):
        gg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gg, stream=stream):
            for k in range(reps):
                flusher(k)
                if with_fn:
                    fn(stream)
        torch.cuda.synchronize()
        return gg
    with torch.cuda.stream(stream):
        fn(stream)                                   # (autotune / cuDNN algorithm choice outside capture)
    torch.cuda.synchronize()
    gf, gfl = cap(False), cap(True)
    out = []
    for _ in range(3):
        ts = []
        for gg in (gf, gfl):
            with torch.cuda.stream(stream):
                gg.replay()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                gg.replay()
                e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        out.append((ts[1] - ts[0]) / reps)
    return sorted(out)[1]


def time_graph(torch, g, stream, flush, reps=21, per=1):
    """Device time (us) of one replay of g: L2 flushed before each replay when `flush` is given
    (cold), else replays back to back after one warm replay; divided by `per`.  CUDA event
    timestamps on this box are quantised to ~2 us, so a single short replay is timed `reps` times
    and the mean of the middle 60% is reported (the start phase against the timer tick is random,
    so the mean resolves below the tick; a median would return a multiple of it)."""
    ts = []
    with torch.cuda.stream(stream):
        if flush is None:
            g.replay()
        for k in range(reps):
            if flush is not None:
                flush(k)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            ts.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 / per for a, b in ts)
    cut = len(v) // 5
    mid = v[cut:len(v) - cut] or v
    return sum(mid) / len(mid)


def layer_bytes(lay):
    """Fused minimum bytes |X| + |W'| + |Y| (SURVEY 8(d) "Algorithmic work per unit")."""
    es = _es(lay.dtype)
    return (lay.n * lay.h * lay.w * lay.c + lay.r * lay.s * lay.f * lay.c + lay.n * lay.oh * lay.ow * lay.f) * es


def roofline_entry(lay, us, peaks, tc_peak):
    """Useful TFLOP/s, algorithmic GB/s, the bound (arithmetic intensity vs the ridge) and the
    fraction of the attainable roofline = max(flops / TC peak, bytes / HBM peak) / time."""
    fl, by = lay.useful_flops, layer_bytes(lay)
    pk = tc_peak if lay.dtype == "bf16" else tc_peak / 2       # TF32: nominal 1.1 / 2.25 PF ratio
    t_tc, t_hbm = fl / (pk * 1e12), by / (peaks["hbm_gbs"] * 1e9)
    att = max(t_tc, t_hbm)
    return {"tflops": fl / (us * 1e-6) / 1e12, "gbs": by / (us * 1e-6) / 1e9,
            "bound": "tensor" if t_tc >= t_hbm else "hbm", "attainable_us": att * 1e6,
            "frac": att / (us * 1e-6), "tc_peak_tflops": pk}


class Workload:
    """The derived layers of one config on this rank: inputs (seeded, full batch, sharded when
    `shard` is given), prepared weights, the stack, its outputs."""

    def __init__(self, torch, cfg, dev, plan, shard=None, batch_override=None):
        from paper_2208_02025_b200.stack import DerivedStack
        self.cfg = cfg
        self.layers_full = syn.CONFIGS[cfg]
        self.chained = cfg in CHAINED
        self.shard = shard
        lays = self.layers_full
        if shard is not None:
            lays = [l.with_batch(shard.n_local) for l in lays]
        if batch_override is not None:
            lays = [l.with_batch(batch_override) for l in lays]
        self.layers = lays
        self.stack = DerivedStack(lays, self.chained, plan=plan, device=dev)
        self.x_host, w_dev = [], []
        for li, lay in enumerate(self.layers_full):
            x, w = syn.layer_inputs(lay, syn.config_seed(cfg, li))       # same data on every rank
            if shard is not None:
                x = shard.local(x)
            self.x_host.append(x)
            w_dev.append(w.to(dev))
        self.w_dev = w_dev
        self.stack.prepare(w_dev)
        if self.chained:
            self.x_dev = [self.x_host[0].to(dev)]
        else:
            self.x_dev = [x.to(dev) for x in self.x_host]
        self.outs = [sl.y for sl in self.stack.layers]

    @property
    def inputs(self):
        return self.x_dev[0] if self.chained else self.x_dev

    def step(self, stream):
        self.stack(self.inputs, stream=stream.cuda_stream)

    @property
    def flops(self):
        return sum(l.useful_flops for l in self.layers)

    def final_outputs(self):
        return [self.outs[-1]] if self.chained else self.outs


def _cudnn_fns(torch, layers, chained, x_host, w_dev, dev):
    """cuDNN through torch (channels_last, cudnn.benchmark) on the same inputs: one callable per
    layer (reading the previous layer's output in chained stacks) and the whole step."""
    import torch.nn.functional as F
    torch.backends.cudnn.benchmark = True
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    xs = [x.to(dev).permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last) for x in x_host]
    ws = [w.contiguous(memory_format=torch.channels_last) for w in w_dev]
    bufs = [None] * len(layers)

    def run_layer(li, src):
        lay = layers[li]
        if lay.transposed:
            return F.conv_transpose2d(src, ws[li], stride=lay.stride, padding=lay.pad,
                                      output_padding=lay.output_padding, dilation=lay.dilation)
        return F.conv2d(src, ws[li], stride=lay.stride, padding=lay.pad, dilation=lay.dilation)

    def src_of(li):
        if not chained:
            return xs[li]
        return xs[0] if li == 0 else bufs[li - 1]

    def step(_s=None):
        for li in range(len(layers)):
            bufs[li] = run_layer(li, src_of(li))

    step()                                  # cudnn.benchmark picks algorithms; fills bufs
    torch.cuda.synchronize()
    layer_fns = [(lambda li: (lambda _s=None: run_layer(li, src_of(li))))(li) for li in range(len(layers))]
    return step, layer_fns


def per_layer_records(torch, wl, stream, flush, peaks, tc_peak, with_cudnn=True):
    """Per layer: ours and cuDNN by the same method -- flushed (L2 evicted before each call,
    time_graph_flushed's differential graph timing) and warm (10 calls back to back in one graph)
    device times; the step likewise.  Every measurement of ours is taken before cuDNN runs at all
    (after cuDNN's graphs existed, one CSRNet step measurement came out ~40% slower than the same
    measurement in isolation)."""
    from paper_2208_02025_b200 import ollie as O
    recs = []
    srcs = []
    x = wl.inputs if wl.chained else None
    for li, sl in enumerate(wl.stack.layers):
        srcs.append(x if wl.chained else wl.inputs[li])
        x = sl.y
    step = {}
    step["ours_us"] = time_graph_flushed(torch, lambda s: wl.step(s), stream, flush)
    step["ours_tflops"] = wl.flops / (step["ours_us"] * 1e-6) / 1e12
    for li, (sl, lay) in enumerate(zip(wl.stack.layers, wl.layers)):
        fn = (lambda sl, src: (lambda s: sl(src, s.cuda_stream)))(sl, srcs[li])
        g10 = _graph(torch, fn, stream, reps=10)
        ours_f = time_graph_flushed(torch, fn, stream, flush)
        ours_w = time_graph(torch, g10, stream, None, per=10)
        del g10
        recs.append({"layer": lay.name, "plan": O.plan_describe(sl.conv.shape, sl.conv.code, sl.conv.plan, sl.conv.transposed),
                     "launches": sl.launches(), "useful_gflop": lay.useful_flops / 1e9, "alg_mb": layer_bytes(lay) / 1e6,
                     "ours_us": ours_f, "ours_warm_us": ours_w, **roofline_entry(lay, ours_f, peaks, tc_peak)})
    if not with_cudnn:
        return recs, step
    try:
        cud_step, cud_layers = _cudnn_fns(torch, wl.layers, wl.chained, wl.x_host, wl.w_dev, stream.device)
    except Exception as e:                                  # noqa: BLE001
        step["cudnn_error"] = f"cuDNN failed: {e!r}"[:200]
        return recs, step
    # cuDNN's step first, like ours (step, then layers): measured last, after the per-layer graphs, a
    # one-layer CSRNet cuDNN step once read 193 us against 167 us for the same call per layer
    step["cudnn_us"] = time_graph_flushed(torch, cud_step, stream, flush)
    for li, (rec, lay) in enumerate(zip(recs, wl.layers)):
        c10 = _graph(torch, cud_layers[li], stream, reps=10)
        cf = time_graph_flushed(torch, cud_layers[li], stream, flush)
        cw = time_graph(torch, c10, stream, None, per=10)
        del c10
        rec.update({"cudnn_us": cf, "cudnn_warm_us": cw, "cudnn_tflops": lay.useful_flops / (cf * 1e-6) / 1e12,
                    "speedup_vs_cudnn": cf / rec["ours_us"], "speedup_vs_cudnn_warm": cw / rec["ours_warm_us"]})
    step["cudnn_tflops"] = wl.flops / (step["cudnn_us"] * 1e-6) / 1e12
    step["speedup_vs_cudnn"] = step["cudnn_us"] / step["ours_us"]
    # the same comparison from the per-layer flushed times (sum over layers, both sides alike)
    step["speedup_vs_cudnn_layer_sum"] = sum(r["cudnn_us"] for r in recs) / sum(r["ours_us"] for r in recs)
    return recs, step


def eop_records(torch, dev, stream, flush, peaks):
    """SURVEY 8(d) eOperator configs E-b..E-f: GB/s = algorithmic (|in| + |out|) / device time,
    L2 flushed before each launch (median of 7)."""
    from paper_2208_02025_b200 import eops, ollie as O

    def timed(fn):
        ts = []
        with torch.cuda.stream(stream):
            fn()
            for k in range(7):
                flush(k)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                ts.append((e0, e1))
        torch.cuda.synchronize()
        v = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
        return v[len(v) // 2]

    s = stream.cuda_stream
    out = {}

    # same-method ceilings on this box: a 134 MB torch copy (read + write) and fill (write only) --
    # a channel pad writes 16x what it reads, so its bound is the write rate, not the copy rate
    cb = torch.empty(134217728, dtype=torch.uint8, device=dev)
    cd = torch.empty_like(cb)
    with torch.cuda.stream(stream):
        copy_gbs = 2 * cb.numel() / (timed(lambda: cd.copy_(cb)) * 1e-6) / 1e9
        fill_gbs = cb.numel() / (timed(lambda: cb.fill_(1)) * 1e-6) / 1e9
    del cb, cd
    out["ceilings (torch, same method, 134 MB)"] = {"copy_gbs": copy_gbs, "write_only_gbs": fill_gbs}

    def rec(name, nbytes, us, ok=True, write_bytes=None):
        out[name] = {"us": us, "gbs": nbytes / (us * 1e-6) / 1e9, "alg_mb": nbytes / 1e6,
                     "frac_of_hbm": nbytes / (us * 1e-6) / 1e9 / peaks["hbm_gbs"],
                     "frac_of_copy_ceiling": nbytes / (us * 1e-6) / 1e9 / copy_gbs, "bit_exact_vs_torch": ok}
        if write_bytes is not None:
            out[name]["frac_of_write_ceiling"] = write_bytes / (us * 1e-6) / 1e9 / fill_gbs

    g = torch.Generator(device="cpu").manual_seed(5)
    n, c, h, w = 16, 512, 64, 64                              # E-b: CSRNet input NCHW -> NHWC
    x = torch.randn(n, c, h, w, generator=g).to(torch.bfloat16).to(dev)
    y = torch.empty(n, h, w, c, device=dev, dtype=torch.bfloat16)
    e = O.make_eop(eops.nchw_to_nhwc(n, c, h, w), [O.BF16], O.BF16)
    us = timed(lambda: O.eop_eval(e, [x], y, s))
    rec("E-b nchw_to_nhwc [16,512,64,64] bf16", 2 * x.numel() * 2, us, bool(torch.equal(y, x.permute(0, 2, 3, 1))))
    for cc in (1, 12):                                        # E-c: FSRCNN channel pad
        x = torch.randn(64, 256, 256, cc, generator=g).to(torch.bfloat16).to(dev)
        y = torch.empty(64, 256, 256, 16, device=dev, dtype=torch.bfloat16)
        e = O.make_eop(eops.channel_pad(64, 256, 256, cc, 16), [O.BF16], O.BF16)
        us = timed(lambda: O.eop_eval(e, [x], y, s))
        ok = bool(torch.equal(y[..., :cc], x)) and not bool(y[..., cc:].any())
        rec(f"E-c channel_pad {cc}->16 [64,256,256] bf16", x.numel() * 2 + y.numel() * 2, us, ok, write_bytes=y.numel() * 2)
    shp = O.conv_shape(1, 512, 7, 7, 512, 3, 3, 1)           # E-d: weight DLT
    wt = torch.randn(512, 512, 3, 3, generator=g).to(torch.bfloat16).to(dev)
    wp = torch.empty(9 * 512, 512, device=dev, dtype=torch.bfloat16)
    us = timed(lambda: O.prepare_weight_conv2d(shp, O.BF16, wt, wp, s))
    rec("E-d weight DLT [512,512,3,3] bf16", 2 * wt.numel() * 2, us,
        bool(torch.equal(wp, wt.permute(2, 3, 0, 1).reshape(9 * 512, 512))))
    shp = O.conv_shape(16, 64, 56, 56, 64, 3, 3, 1)          # E-e: OffsetAdd (B-K2) R18 64x56 b16
    T = torch.randn(16 * 56 * 56, 576, generator=g).to(dev)
    Y = torch.empty(16, 56, 56, 64, device=dev, dtype=torch.bfloat16)
    us = timed(lambda: O.offset_add(shp, False, T, 576, O.BF16, Y, s))
    inb = 16 * (56 * 3 - 2) * (56 * 3 - 2) * 64 * 4          # in-bounds (pixel, tap) T reads
    rec("E-e OffsetAdd standalone R18 64x56^2 b16 (T fp32 -> Y bf16)", inb + Y.numel() * 2, us)
    shp = O.conv_shape(16, 128, 16, 16, 64, 4, 4, 1, 2)      # E-f: selective add DCGAN 128->64 b16
    T = torch.randn(16 * 16 * 16, 1024, generator=g).to(dev)
    Y = torch.empty(16, 32, 32, 64, device=dev, dtype=torch.bfloat16)
    us = timed(lambda: O.offset_add(shp, True, T, 1024, O.BF16, Y, s))
    rec("E-f selective add (residue classes, interleaved) DCGAN 128->64 16->32 b16",
        16 * 16 * 16 * 1024 * 4 * (15 * 15) / (16 * 16) + Y.numel() * 2, us)
    return out


def g2bmm_records(torch, dev, stream, flush, peaks):
    """NEXT-4 LongFormer G2BMM [8,10000,64], W=256, d=4 (reading R4), natural output pitch 2W+1."""
    from paper_2208_02025_b200 import ollie as O
    gcfg = syn.G2_CONFIGS["longformer"][0]
    a, b = syn.g2bmm_inputs(gcfg, 77)
    a, b = a.to(dev), b.to(dev)
    nw = 2 * gcfg.W + 1
    out = torch.empty(gcfg.batch, gcfg.L, nw, dtype=torch.bfloat16, device=dev)
    res = {}
    for form, name in ((O.G2BMM_DERIVED, "derived (dilated -> non-dilated)"), (O.G2BMM_DIRECT, "direct (dilated)")):
        fn = (lambda form: (lambda st: O.g2bmm(gcfg.batch, gcfg.L, gcfg.K, gcfg.W, gcfg.d, O.BF16, a, b, out, nw, form,
                                               st.cuda_stream)))(form)
        g = _graph(torch, fn, stream)
        us = time_graph(torch, g, stream, flush)
        res[name] = {"us": us, "gbs": gcfg.bytes / (us * 1e-6) / 1e9, "tflops": gcfg.flops / (us * 1e-6) / 1e12,
                     "frac_of_hbm": gcfg.bytes / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], "ldo": nw}
    return res


# ------------------------------------------------------------------------- GPU arm
def gpu_main(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # OLLIE_BENCH_BACKEND=gloo (ranks sharing the visible GPUs round-robin) exercises the N > 1 path
        # on a single-GPU box; the driver's multi-GPU runs use NCCL, one GPU per rank
        backend = os.environ.get("OLLIE_BENCH_BACKEND", "nccl")
        local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    from paper_2208_02025_b200 import ollie as O
    from paper_2208_02025_b200.parallel import BlockCyclic

    cfg = args.config
    layers_full = syn.CONFIGS[cfg]
    n_full = layers_full[0].n
    shardable = world > 1 and all(l.n == n_full for l in layers_full) and n_full % world == 0
    shard = BlockCyclic(n_full, world, rank, 1) if shardable else None
    plan = {"auto": O.PLAN_AUTO, "fused": O.PLAN_FUSED, "unfused": O.PLAN_UNFUSED}[args.plan]
    # pinned host memory for the e2e copies first, from early allocations (e2e)
    wl = Workload(torch, cfg, dev, plan, shard=shard)
    in_host = [x.pin_memory() for x in (wl.x_host[:1] if wl.chained else wl.x_host)]
    flush = Flusher(torch, dev)
    stream = torch.cuda.Stream(device=dev)
    peaks = _peaks()

    # warm-up (first call autotunes every layer's plan) + graph capture of one step
    with torch.cuda.stream(stream):
        for _ in range(max(1, args.warmup)):
            wl.step(stream)
    stream.synchronize()
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            wl.step(stream)
        torch.cuda.synchronize()

    def replay():
        if graph is not None:
            graph.replay()
        else:
            wl.step(stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            replay()
    torch.cuda.synchronize()

    # ---------------- timed region: K steps, L2 flushed before each, events per step
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        time.sleep(0.3)
        t_wall0 = time.perf_counter()
        # under `ncu --profile-from-start off` only the timed steps are captured
        torch.cuda.cudart().cudaProfilerStart()
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                flush(k)
                starts[k].record(stream)
                replay()
                ends[k].record(stream)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        if world > 1:
            dist.barrier()
        t_wall = time.perf_counter() - t_wall0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops_total = sum(l.useful_flops for l in layers_full)      # the whole batch, all ranks
    value = flops_total / (ms * 1e-3) / 1e12

    # ---------------- a9 all-gather (N > 1): serial and chunk-overlapped
    allgather = None
    if world > 1 and shardable and not args.no_allgather:
        allgather = allgather_records(torch, dist, wl, cfg, dev, plan, stream, flush, graph, args, world, rank)

    # ---------------- e2e: the same step through the public API with host buffers
    e2e = e2e_record(torch, dist, wl, in_host, stream, args, world, flops_total)

    # ---------------- per-layer in-graph records (ours vs cuDNN, same method) + roofline
    tc_peak = peaks["bf16_tflops"]
    recs, step_rec = per_layer_records(torch, wl, stream, flush, peaks, tc_peak, with_cudnn=not args.no_cudnn)
    # fractions against a tensor peak at least as high as any dense bf16 rate cuDNN reaches here
    seen = max([r.get("cudnn_tflops", 0.0) for r in recs if wl.layers[0].dtype == "bf16"] + [0.0])
    peak_src = f"MEASURED_PEAKS.json bf16_tflops ({peaks['source']})"
    if seen > tc_peak:
        tc_peak = seen
        peak_src = "max(MEASURED_PEAKS.json bf16_tflops, best cuDNN rate on this box in this run)"
        for r, lay in zip(recs, wl.layers):
            r.update(roofline_entry(lay, r["ours_us"], peaks, tc_peak))
    dom = max(range(len(recs)), key=lambda i: recs[i]["ours_us"])
    d, dl = recs[dom], wl.layers[dom]
    if d["bound"] == "tensor":
        pk = d["tc_peak_tflops"]
        nominal = 2250.0 if dl.dtype == "bf16" else 1125.0          # dense bf16 / TF32 per GPU (B200 spec)
        roof = {"kernel": d["layer"], "bound": "tensor", "achieved": d["tflops"], "peak": pk, "unit": "TFLOP/s",
                "frac": d["tflops"] / pk, "peak_source": peak_src,
                "frac_of_nominal": d["tflops"] / nominal, "nominal_peak": nominal}
    else:
        roof = {"kernel": d["layer"], "bound": "hbm", "achieved": d["gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": d["gbs"] / peaks["hbm_gbs"], "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peaks['source']})"}
    roof["traffic"] = _traffic_from_profiles(cfg, "fused_conv" if d["plan"].startswith("fused") else "merged_gemm")
    roof["alg_bytes_per_launch"] = layer_bytes(dl)
    roof["useful_flops_per_launch"] = dl.useful_flops
    roof["kernel_us"] = d["ours_us"]
    roof["share_of_step"] = d["ours_us"] / max(step_rec["ours_us"], 1e-9)
    roof["method"] = ("the dominant layer captured alone in a CUDA graph, L2 flushed before each replay, CUDA "
                      "events on its stream (the same conditions as a step: kernel_us <= ms_per_step)")

    suite = eops = g2 = None
    if rank == 0 and world == 1 and not args.no_suite:
        suite = {}
        for name in SUITE:
            if name == cfg:
                continue
            try:
                w2 = Workload(torch, name, dev, plan)
                with torch.cuda.stream(stream):
                    w2.step(stream)          # autotune
                    w2.step(stream)
                torch.cuda.synchronize()
                r2, s2 = per_layer_records(torch, w2, stream, flush, peaks, tc_peak, with_cudnn=not args.no_cudnn)
                suite[name] = {"workload": CONFIG_TEXT.get(name, name), "dtype": w2.layers[0].dtype,
                               "step": s2, "layers": r2}
                del w2
            except Exception as e:                              # noqa: BLE001
                suite[name] = {"error": repr(e)[:300]}
            torch.cuda.empty_cache()
        try:
            eops = eop_records(torch, dev, stream, flush, peaks)
        except Exception as e:                                  # noqa: BLE001
            eops = {"error": repr(e)[:300]}
        try:
            g2 = g2bmm_records(torch, dev, stream, flush, peaks)
        except Exception as e:                                  # noqa: BLE001
            g2 = {"error": repr(e)[:300]}

    result = None
    if rank == 0:
        clocks = clk.summary()
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg, layers_full, max_flop=args.cpu_flop)
        result = {
            "metric": "derived conv useful TFLOP/s (whole step)", "value": value, "unit": "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": layers_full[0].dtype, "data": "synthetic (seeded, ollie_synth; random-init weights)",
            "config": {"workload": CONFIG_TEXT.get(cfg, cfg), "name": cfg,
                       "layers": [l.name for l in layers_full], "plan": args.plan,
                       "global_batch": n_full,
                       "l2": "flushed before every step: 2x-L2 write, then read back (retires dirty lines), both outside the per-step events",
                       "timing": "CUDA graph replay per step, CUDA events on the launching stream, max over ranks",
                       "parallelism": (f"batch-sharded x{world} (block-cyclic), outputs left sharded; all-gather in 'allgather'"
                                       if shardable else (f"replicas x{world} (batch {n_full} does not split)" if world > 1 else "1 GPU"))},
            "us_per_layer": {r["layer"]: r["ours_us"] for r in recs},
            "cudnn_us_per_layer": {r["layer"]: r.get("cudnn_us") for r in recs},
            "vs_cudnn": step_rec.get("speedup_vs_cudnn"),
            "vs_cudnn_layer_sum": step_rec.get("speedup_vs_cudnn_layer_sum"),
            "e2e": e2e,
            "gpu_launches": wl.stack.launches() * args.steps,
            "roofline": roof,
            "layers": recs,
            "step": step_rec,
            "allgather": allgather,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "wall_s_timed_region": t_wall,
            "per_step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
            "suite": suite,
            "eops": eops,
            "g2bmm": g2,
        }
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def allgather_records(torch, dist, wl, cfg, dev, plan, stream, flush, graph, args, world, rank):
    """a9 end to end: the rank's shard computed, then every rank's Y all-gathered (NCCL) into
    preallocated full-batch buffers -- serial (one gather after the step) and overlapped (the
    shard in `chunks` micro-batches, chunk k's gather on a side stream under chunk k+1's compute;
    block-cyclic ownership makes each chunk's gather a contiguous slice of the full output)."""
    from paper_2208_02025_b200.parallel import BlockCyclic
    n = wl.layers_full[0].n
    y_loc = wl.final_outputs()
    y_full = [torch.empty((n,) + tuple(y.shape[1:]), dtype=y.dtype, device=dev) for y in y_loc]
    comm = torch.cuda.Stream(device=dev)
    res = {"chunks": 1}

    def timed(run, reps):
        ts = []
        for k in range(reps):
            flush(k)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                run()
                e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = torch.tensor([statistics.median(ts)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    shard1 = wl.shard

    def serial():
        graph.replay() if graph is not None else wl.step(stream)
        for yf, yl in zip(y_full, y_loc):
            shard1.gather_chunk(yf, yl, 0)

    ms_serial = timed(serial, max(3, min(args.steps, 10)))
    res["serial_ms"] = ms_serial
    chunks = BlockCyclic.max_chunks(n, world, args.chunks)
    if chunks > 1:
        sh = BlockCyclic(n, world, rank, chunks)
        wc = Workload(torch, cfg, dev, plan, shard=sh, batch_override=sh.cb)
        xl = [x.to(dev) for x in (wc.x_host[:1] if wc.chained else wc.x_host)]     # the rank's shard, chunk-major
        yl = [torch.empty((sh.n_local,) + tuple(y.shape[1:]), dtype=y.dtype, device=dev) for y in wc.final_outputs()]
        ylf = [torch.empty((n,) + tuple(y.shape[1:]), dtype=y.dtype, device=dev) for y in yl]

        def chunk_fn(k):
            def f(s):
                if wc.chained:
                    wc.stack(sh.chunk(xl[0], k), stream=s.cuda_stream, out=sh.chunk(yl[0], k))
                else:
                    wc.stack([sh.chunk(x, k) for x in xl], stream=s.cuda_stream, out=[sh.chunk(y, k) for y in yl])
            return f
        with torch.cuda.stream(stream):
            chunk_fn(0)(stream)                 # autotune at the chunk batch
        torch.cuda.synchronize()
        cgraphs = [_graph(torch, chunk_fn(k), stream) for k in range(chunks)]
        evs = [torch.cuda.Event() for _ in range(chunks)]

        def overlapped():
            comm.wait_stream(stream)
            for k in range(chunks):
                cgraphs[k].replay()
                evs[k].record(stream)
                comm.wait_event(evs[k])
                with torch.cuda.stream(comm):
                    for yf, y in zip(ylf, yl):
                        sh.gather_chunk(yf, y, k)
            stream.wait_stream(comm)

        res["chunks"] = chunks
        res["overlapped_ms"] = timed(overlapped, max(3, min(args.steps, 10)))
        # the overlapped (micro-batched) result against the serial one: the same images, but the chunk
        # batch may autotune to another tile plan (another fp32 summation order), so compare within the
        # bf16 bar rather than bit for bit (tests/test_gpu_multiproc.py checks bit equality in integer mode)
        diff = max(float((a.float() - b.float()).abs().max()) / max(float(b.float().abs().max()), 1e-30)
                   for a, b in zip(ylf, y_full))
        res["overlapped_vs_serial_max_rel"] = diff
        res["overlapped_matches_serial"] = diff <= 1e-2
    flops = sum(l.useful_flops for l in wl.layers_full)
    for k in ("serial_ms", "overlapped_ms"):
        if k in res:
            res[k.replace("_ms", "_tflops")] = flops / (res[k] * 1e-3) / 1e12
    res["gathered_bytes_per_rank"] = sum(y.numel() * y.element_size() for y in y_full) * (world - 1) // world
    return res


def e2e_record(torch, dist, wl, in_host, stream, args, world, flops_total):
    """The step through the public API with pinned host buffers: every step's H2D of the rank's
    inputs and D2H of its outputs inside the timed region, pipelined (two device buffer sets; H2D
    of step k+1 and D2H of step k on their own streams overlap step k's / k+1's layers)."""
    dev = stream.device
    outs_dev = wl.final_outputs()
    out_host = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in outs_dev]
    din = [[torch.empty_like(x, device=dev) for x in in_host] for _ in range(2)]
    dout = [[torch.empty_like(o) for o in outs_dev] for _ in range(2)]
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    h2d = sum(t.numel() * t.element_size() for t in in_host)
    d2h = sum(t.numel() * t.element_size() for t in out_host)

    def run_step(b):
        if wl.chained:
            wl.stack(din[b][0], stream=stream.cuda_stream, out=dout[b][0])
        else:
            wl.stack(din[b], stream=stream.cuda_stream, out=dout[b])

    def loop(nsteps):
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        h2d_s.wait_stream(stream)
        d2h_s.wait_stream(stream)
        for k in range(nsteps):
            b = k % 2
            if k >= 2:
                h2d_s.wait_event(ev_done[b])                 # step k-2's layers read this buffer
            with torch.cuda.stream(h2d_s):
                for dd, hh in zip(din[b], in_host):
                    dd.copy_(hh, non_blocking=True)
                ev_in[b].record(h2d_s)
            stream.wait_event(ev_in[b])
            if k >= 2:
                stream.wait_event(ev_out[b])                 # step k-2's D2H read this buffer
            run_step(b)
            ev_done[b].record(stream)
            d2h_s.wait_event(ev_done[b])
            with torch.cuda.stream(d2h_s):
                for hh, dd in zip(out_host, dout[b]):
                    hh.copy_(dd, non_blocking=True)
                ev_out[b].record(d2h_s)
        stream.wait_stream(h2d_s)
        stream.wait_stream(d2h_s)

    with torch.cuda.stream(stream):
        loop(2)
    torch.cuda.synchronize()
    runs = []
    for _ in range(3):
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            loop(args.steps)
            b.record(stream)
        torch.cuda.synchronize()
        runs.append(a.elapsed_time(b) / args.steps)
    e2e_ms = statistics.median(runs)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    return {"value": flops_total / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "ms_per_step_runs": runs,
            "mode": "eager API calls; H2D / layers / D2H pipelined on three streams, two device buffer sets"}


def _traffic_from_profiles(cfg, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(cfg, {}).get(kernel)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=HEADLINE, choices=sorted(syn.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--plan", default="auto", choices=["auto", "fused", "unfused"])
    ap.add_argument("--chunks", type=int, default=4, help="micro-batches per rank for the overlapped all-gather (N>1)")
    ap.add_argument("--no-allgather", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cudnn", action="store_true")
    ap.add_argument("--no-suite", action="store_true", help="skip the other BASELINE configs / eOps / G2BMM sub-records")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-flop", type=float, default=3e10, help="oracle sample per reference-arm step (flops)")
    ap.add_argument("--cpu-flop", type=float, default=2e11, help="oracle sample for cpu_baseline (flops)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_main(args)
    return gpu_main(args)


if __name__ == "__main__":
    sys.exit(main())
