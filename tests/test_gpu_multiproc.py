"""a9 / SURVEY 8(e) with the PRODUCT kernels under a process group: every rank runs the derived
stack (libollie) on its block-cyclic shard of the batch in micro-batches, each chunk's output is
all-gathered into its final slice of the full batch, and the result equals the 1-process run of
the same stack bit for bit (T5).  Integer-mode inputs: the per-rank batch differs from the
1-process batch, so autotuning may pick another plan (tile shape, split-K) whose fp32 summation
order differs; with exact integer sums every order gives the same bits.

  * NCCL over NVLink with world = min(8, visible GPUs), one GPU per rank (skipped below 2 GPUs);
  * two ranks sharing cuda:0 over gloo (its device collectives go through host staging in
    parallel._all_gather_into) -- the same code path on a single-GPU box.
"""
import os
import socket
from dataclasses import replace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ollie_synth as syn

pytestmark = pytest.mark.gpu

CFG = "csrnet"


def _layers(n):
    return [replace(l, n=n, h=24, w=24) for l in syn.CONFIGS[CFG]]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _single(n):
    from paper_2208_02025_b200.stack import DerivedStack
    lays = _layers(n)
    x, w = syn.layer_inputs(lays[0], 901, exact_int=True)
    st = DerivedStack(lays, False)
    st.prepare([w.cuda()])
    y = st([x.cuda()])[0]
    torch.cuda.synchronize()
    return y.cpu()


def _worker(rank, world, port, backend, n, chunks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    kw = {"device_id": torch.device("cuda", dev)} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        from paper_2208_02025_b200.parallel import BlockCyclic
        from paper_2208_02025_b200.stack import DerivedStack
        sh = BlockCyclic(n, world, rank, chunks)
        lays = _layers(n)
        x, w = syn.layer_inputs(lays[0], 901, exact_int=True)  # the full batch, same seed everywhere
        xl = sh.local(x).cuda()
        st = DerivedStack([l.with_batch(sh.cb) for l in lays], False)
        st.prepare([w.cuda()])
        yl = torch.empty((sh.n_local,) + tuple(st.layers[0].y.shape[1:]), dtype=torch.bfloat16, device="cuda")
        yf = torch.full((n,) + tuple(yl.shape[1:]), float("nan"), dtype=torch.bfloat16, device="cuda")
        comm = torch.cuda.Stream()
        for k in range(chunks):
            st([sh.chunk(xl, k)], out=[sh.chunk(yl, k)])
            ev = torch.cuda.Event()
            ev.record()
            comm.wait_event(ev)
            with torch.cuda.stream(comm):                     # chunk k's gather overlaps chunk k+1
                sh.gather_chunk(yf, yl, k)
        torch.cuda.current_stream().wait_stream(comm)
        torch.cuda.synchronize()
        q.put((rank, yf.float().cpu().numpy()))
    finally:
        dist.destroy_process_group()


def _run(world, backend, n, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, n, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = _single(n).float().numpy()
    for r in range(world):
        assert np.array_equal(res[r], want), f"rank {r}"


def test_two_ranks_one_gpu_gloo_product_kernels():
    _run(2, "gloo", 8, 2)


def test_nccl_all_gpus_product_kernels():
    world = min(8, torch.cuda.device_count())
    if world < 2:
        pytest.skip("needs >= 2 GPUs (gpurun boxes have one; covered by the gloo test above)")
    _run(world, "nccl", 2 * world, 2)
