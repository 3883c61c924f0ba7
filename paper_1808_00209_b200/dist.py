"""Data-parallel plumbing: contiguous batch shards, one process per GPU, and the one
exchange step of the path -- an all-gather of the int32 predictions over NCCL (NVLink / NVSwitch).

Images are independent, so no other collective exists on the data path.  The helpers are backend
agnostic so the same code is exercised with gloo on CPU (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(n_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: rank r owns images [r * n_per_rank, (r + 1) * n_per_rank) of the seeded stream."""
    return rank * n_per_rank, n_per_rank


def shard_total(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Strong scaling: contiguous near-equal shards of n_total images."""
    base, rem = divmod(n_total, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def gather_predictions(logits: torch.Tensor, cls: torch.Tensor, out_logits: torch.Tensor | None = None,
                       out_cls: torch.Tensor | None = None):
    """All-gather equal-size per-rank predictions into [world * n, ...] tensors (rank order)."""
    world = dist.get_world_size()
    n = logits.shape[0]
    if out_logits is None:
        out_logits = torch.empty((world * n,) + tuple(logits.shape[1:]), dtype=logits.dtype, device=logits.device)
    if out_cls is None:
        out_cls = torch.empty((world * n,), dtype=cls.dtype, device=cls.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out_logits, logits.contiguous())
        dist.all_gather_into_tensor(out_cls, cls.contiguous())
    else:
        dist.all_gather(list(out_logits.chunk(world)), logits.contiguous())
        dist.all_gather(list(out_cls.chunk(world)), cls.contiguous())
    return out_logits, out_cls


def max_over_ranks(value: float, device) -> float:
    """Timing rule: the job's time is the slowest rank's."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
