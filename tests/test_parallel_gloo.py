"""a9 on CPU: world-size-2 gloo processes shard the batch, each computes its images (with the
fp64 oracle standing in for the per-rank kernels -- tests/test_gpu_multiproc.py runs the product
kernels), and the gathered output equals the
single-process result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ollie_synth as syn


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2208_02025_b200 import parallel as par
        lay = syn.Layer("t", n, 8, 6, 5, 4, 3, 3, pad=1)
        x, w = syn.layer_inputs(lay, 5, exact_int=True)
        xs = par.shard(x, rank, world)
        y = torch.from_numpy(oracle.conv2d(xs, w, 1)) if xs.shape[0] else torch.zeros(0, 6, 5, 4, dtype=torch.float64)
        full = par.gather_batch(y, n)
        q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [4, 5])
def test_batch_shard_allgather_matches_single_process(n):
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lay = syn.Layer("t", n, 8, 6, 5, 4, 3, 3, pad=1)
    x, w = syn.layer_inputs(lay, 5, exact_int=True)
    want = oracle.conv2d(x, w, 1)
    for r in range(world):
        assert np.array_equal(res[r], want)


def test_shard_range_partitions():
    from paper_2208_02025_b200 import parallel as par
    for n in (1, 7, 16, 64):
        for world in (1, 2, 3, 8):
            spans = [par.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - s for s, e in spans) - min(e - s for s, e in spans) <= 1


def _worker_cyclic(rank, world, port, n, chunks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2208_02025_b200 import parallel as par
        lay = syn.Layer("t", n, 8, 6, 5, 4, 3, 3, pad=1)
        x, w = syn.layer_inputs(lay, 6, exact_int=True)
        sh = par.BlockCyclic(n, world, rank, chunks)
        xl = sh.local(x)
        y_local = torch.empty(sh.n_local, 6, 5, 4, dtype=torch.float64)
        y_full = torch.full((n, 6, 5, 4), float("nan"), dtype=torch.float64)
        for k in range(chunks):                  # per chunk: compute, then gather its slice
            sh.chunk(y_local, k).copy_(torch.from_numpy(oracle.conv2d(sh.chunk(xl, k), w, 1)))
            sh.gather_chunk(y_full, y_local, k)
        y_cont = torch.empty(n, 6, 5, 4, dtype=torch.float64)   # contiguous shards, preallocated out
        xs = par.shard(x, rank, world)
        par.gather_batch(torch.from_numpy(oracle.conv2d(xs, w, 1)), n, out=y_cont)
        q.put((rank, y_full.numpy(), y_cont.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,chunks", [(8, 1), (8, 2), (12, 3)])
def test_block_cyclic_chunked_gather_matches_single_process(n, chunks):
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_cyclic, args=(r, world, port, n, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, a, b = q.get(timeout=120)
        res[r] = (a, b)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lay = syn.Layer("t", n, 8, 6, 5, 4, 3, 3, pad=1)
    x, w = syn.layer_inputs(lay, 6, exact_int=True)
    want = oracle.conv2d(x, w, 1)
    for r in range(world):
        assert np.array_equal(res[r][0], want)
        assert np.array_equal(res[r][1], want)


def test_block_cyclic_layout():
    from paper_2208_02025_b200 import parallel as par
    for n, world, chunks in ((16, 2, 4), (16, 8, 2), (64, 4, 4), (6, 3, 1)):
        owned = []
        for r in range(world):
            sh = par.BlockCyclic(n, world, r, chunks)
            assert len(sh.local_index) == sh.n_local == n // world
            owned += sh.local_index
            for k in range(chunks):        # chunk k of every rank tiles the slice [k*world*cb, (k+1)*world*cb)
                blk = sh.local_index[k * sh.cb:(k + 1) * sh.cb]
                assert blk == list(range((k * world + r) * sh.cb, (k * world + r + 1) * sh.cb))
        assert sorted(owned) == list(range(n))
    assert par.BlockCyclic.max_chunks(16, 8, 4) == 2
    assert par.BlockCyclic.max_chunks(64, 8, 4) == 4
    assert par.BlockCyclic.max_chunks(16, 3, 4) == 0
    with pytest.raises(ValueError):
        par.BlockCyclic(10, 4, 0, 1)
