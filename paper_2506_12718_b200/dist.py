"""Multi-GPU plumbing for the batched hot path.

Signals are independent (convolution.cpp:45-52 touches one buffer per call)
and a Plan / PreparedFilter is immutable and shareable, so a
batch shards across ranks with no data-path collective.  The default is the
north star's partition: the config's FIXED global batch is
split into contiguous slices, batch / G per rank (strong scaling: config 4
is one volume per GPU at 8, config 5 512 per GPU).  `shard_weak` keeps a
fixed per-rank batch instead (opt-in weak scaling).  The only communication
is one broadcast of the prepared filter at setup (ncclBroadcast over NVLink
through torch.distributed's NCCL backend; gloo on CPU for the tests).
"""
from __future__ import annotations


def shard(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """(first signal index, count) of `rank`'s contiguous slice of a fixed
    global batch split over `world` ranks.  Counts differ by at most one
    (the first global_batch % world ranks take one more); every signal is
    owned by exactly one rank.  A rank may own zero signals when
    world > global_batch."""
    if global_batch < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad partition: global_batch={global_batch} world={world} rank={rank}")
    base, extra = divmod(global_batch, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def shard_weak(per_rank: int, rank: int) -> tuple[int, int]:
    """(first signal index, count) for a fixed per-rank batch (weak scaling,
    opt-in: every rank adds `per_rank` signals to the job)."""
    if per_rank < 0 or rank < 0:
        raise ValueError("per_rank and rank must be >= 0")
    return rank * per_rank, per_rank


def broadcast_filter_tensors(tensors, src: int = 0) -> None:
    """Broadcast the prepared filter's buffers (unscaled ghat and the kernel
    copy) from `src` to every rank, in place.  Works on any initialised
    torch.distributed backend (NCCL for device tensors, gloo for CPU ones)."""
    import torch.distributed as dist

    for t in tensors:
        dist.broadcast(t, src=src)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank timing across ranks (the bench's device-time rule)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
