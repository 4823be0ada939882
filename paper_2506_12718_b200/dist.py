"""Multi-GPU plumbing for the batched hot path.

Signals are independent, so a batch shards across ranks with no data-path
collective: rank r owns signals [r * per, (r + 1) * per) of the global batch
(a fixed per-GPU batch: weak scaling).  The only communication is one
broadcast of the prepared filter at setup (ncclBroadcast over NVLink through
torch.distributed's NCCL backend; gloo on CPU for the tests).
"""
from __future__ import annotations


def shard(per_rank: int, rank: int) -> tuple[int, int]:
    """(first signal index, count) owned by `rank` for a fixed per-rank batch."""
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
