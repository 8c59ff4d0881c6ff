"""a9 on CPU: world-size-2 gloo processes shard the batch, each computes its images (with the
fp64 oracle standing in for the per-rank kernels), and the gathered output equals the
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
