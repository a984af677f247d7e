"""Batch sharding across GPUs.

Images are independent, so a batch of B images splits into contiguous per-rank slices; every rank
builds its own graph at its per-GPU batch, runs its own DP (schedules specialise by batch,
P:551-552) and executes its slice. There is no collective on the hot path: the only
communication is the barrier and the max-over-ranks timing reduction around the timed region,
and (off the clock) an optional gather of the outputs.
"""
from __future__ import annotations

from typing import List, Tuple


def shard_range(batch: int, world: int, rank: int) -> Tuple[int, int]:
    """[begin, end) of rank's images: contiguous slices, sizes differ by at most one."""
    if batch < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    base, extra = divmod(batch, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def shard_sizes(batch: int, world: int) -> List[int]:
    return [e - b for b, e in (shard_range(batch, world, r) for r in range(world))]


def gather_outputs(local, world: int, batch: int):
    """All-gather the per-rank output slices (torch tensors [b_r, ...]) into the full batch, off the
    timed region. Works with any torch.distributed backend (gloo on CPU, nccl on GPU)."""
    import torch
    import torch.distributed as dist
    sizes = shard_sizes(batch, world)
    tail = tuple(local.shape[1:])
    bufs = [torch.empty((s,) + tail, dtype=local.dtype, device=local.device) for s in sizes]
    if max(sizes) == min(sizes):
        dist.all_gather(bufs, local.contiguous())
    else:  # pad to equal sizes for all_gather, then trim
        m = max(sizes)
        pad = torch.zeros((m,) + tail, dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        tmp = [torch.empty_like(pad) for _ in sizes]
        dist.all_gather(tmp, pad)
        bufs = [t[:s] for t, s in zip(tmp, sizes)]
    return torch.cat(bufs, dim=0)


def max_over_ranks(value: float, device=None) -> float:
    """Device time is reported as the max over ranks (the slowest rank ends the step)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
