"""a9 -- batch sharding and the output all-gather (not in the paper,
which runs single-GPU inference).

Every image of a Conv2d / ConvTranspose2d is independent and the weights are replicated, so
rank k of g owns the contiguous images [start_k, stop_k) and runs exactly the 1-GPU kernels on
them; the only collective is an all-gather of the outputs (NCCL over NVLink on B200, gloo in
the CPU tests).  Because the per-image arithmetic is identical, the gathered tensor equals the
single-process result bit for bit.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """Balanced contiguous split of n images over `world` ranks (first n % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard(t: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    s, e = shard_range(t.shape[0], rank, world)
    return t[s:e]


def gather_batch(y_local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather batch shards (dim 0) into the full [n_total, ...] tensor on every rank."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    counts = [e - s for s, e in sizes]
    if len(set(counts)) == 1:
        out = torch.empty((n_total,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
        dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
        return out
    # uneven split: pad to the largest shard, gather, then trim
    m = max(counts)
    pad = torch.zeros((m,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    pad[: y_local.shape[0]] = y_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
