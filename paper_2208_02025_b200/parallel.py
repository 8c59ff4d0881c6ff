"""a9 -- batch sharding and the output all-gather (not in the paper,
which runs single-GPU inference).

Every image of a Conv2d / ConvTranspose2d is independent and the weights are replicated, so a
rank runs exactly the 1-GPU kernels on its images; the only collective is an all-gather of the
outputs (NCCL over NVLink on B200, gloo in the CPU tests).  Because the per-image arithmetic is
identical, the gathered tensor equals the single-process result bit for bit.

Two layouts of the shard:
  * contiguous (`shard_range` / `shard` / `gather_batch`): rank k owns images
    [start_k, stop_k) -- one all-gather of the whole shard after the compute;
  * block-cyclic (`BlockCyclic`): the batch is cut into `chunks * world` blocks of `cb` images
    and rank r owns blocks r, world + r, 2*world + r, ...  Its chunk k is then block k*world + r,
    so the all-gather of chunk k from every rank is the CONTIGUOUS slice
    [k*world*cb, (k+1)*world*cb) of the full output, in order: each chunk's gather writes its
    final place directly (no re-layout copy), and can run on a side stream while the rank
    computes chunk k+1 (SURVEY 8(e) "overlap").
Buffers are preallocated by the caller; nothing here allocates on the step path.
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


def _all_gather_into(out: torch.Tensor, inp: torch.Tensor, group=None, async_op=False):
    """all_gather_into_tensor; gloo with device tensors (the single-GPU multi-process test) goes
    through host staging, since gloo's collectives are host-side."""
    if inp.is_cuda and dist.get_backend(group) == "gloo":
        host_out = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(host_out, inp.cpu(), group=group)
        out.copy_(host_out)
        return None
    return dist.all_gather_into_tensor(out, inp, group=group, async_op=async_op)


def gather_batch(y_local: torch.Tensor, n_total: int, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather contiguous batch shards (dim 0) into the full [n_total, ...] tensor on every rank.
    `out` (preallocated, [n_total, ...]) is written in place when given."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    counts = [e - s for s, e in sizes]
    shape = (n_total,) + tuple(y_local.shape[1:])
    if out is None:
        out = torch.empty(shape, dtype=y_local.dtype, device=y_local.device)
    elif tuple(out.shape) != shape:
        raise ValueError(f"out has shape {tuple(out.shape)}, expected {shape}")
    if len(set(counts)) == 1:
        _all_gather_into(out, y_local.contiguous(), group)
        return out
    # uneven split: pad to the largest shard, gather, then trim
    m = max(counts)
    pad = torch.zeros((m,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    pad[: y_local.shape[0]] = y_local
    parts = torch.empty((world * m,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    _all_gather_into(parts, pad, group)
    for r, (s, e) in enumerate(sizes):
        out[s:e] = parts[r * m: r * m + (e - s)]
    return out


class BlockCyclic:
    """Block-cyclic batch shard of n images over `world` ranks in `chunks` micro-batches per rank.

    Rank r's chunk k holds images [(k*world + r)*cb, (k*world + r + 1)*cb), cb = n / (world*chunks);
    `local_index` lists the rank's images in its local order (chunk-major)."""

    def __init__(self, n: int, world: int, rank: int, chunks: int = 1):
        if world < 1 or not 0 <= rank < world or chunks < 1:
            raise ValueError("bad rank / world / chunks")
        if n % (world * chunks):
            raise ValueError(f"batch {n} does not split into {world} ranks x {chunks} chunks")
        self.n, self.world, self.rank, self.chunks = n, world, rank, chunks
        self.cb = n // (world * chunks)
        self.n_local = self.cb * chunks
        self.local_index = [(k * world + rank) * self.cb + i for k in range(chunks) for i in range(self.cb)]

    @staticmethod
    def max_chunks(n: int, world: int, limit: int) -> int:
        """Largest chunk count <= limit that divides the shard evenly."""
        if n % world:
            return 0
        per = n // world
        return max(c for c in range(1, max(1, min(limit, per)) + 1) if per % c == 0)

    def local(self, x_full: torch.Tensor) -> torch.Tensor:
        """The rank's images of a full-batch tensor, in local (chunk-major) order."""
        return x_full[self.local_index]

    def chunk(self, t_local: torch.Tensor, k: int) -> torch.Tensor:
        return t_local[k * self.cb:(k + 1) * self.cb]

    def full_slice(self, y_full: torch.Tensor, k: int) -> torch.Tensor:
        """Slice of the full output that chunk k's all-gather fills (every rank's chunk k, in order)."""
        return y_full[k * self.world * self.cb:(k + 1) * self.world * self.cb]

    def gather_chunk(self, y_full: torch.Tensor, y_local: torch.Tensor, k: int, group=None, async_op=False):
        return _all_gather_into(self.full_slice(y_full, k), self.chunk(y_local, k), group, async_op)
