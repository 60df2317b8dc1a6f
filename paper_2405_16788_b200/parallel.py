"""Multi-GPU plumbing for the dipole engine.

Queries are independent given the tree, so the path shards with a REPLICATED
tree (every rank builds the same tree bit-for-bit from the same cloud) and
contiguous query shards. Forward needs no collective. The adjoint's only
exchange is the sum of the flushed per-point gradients (moments N x C,
normals N x 3, d_epsilon) across ranks — one NCCL all-reduce over NVLink
(torch.distributed, backend "nccl"; "gloo" in the CPU tests).
"""
from __future__ import annotations


def shard_range(total: int, rank: int, world: int):
    """Contiguous [lo, hi) slice of `total` items for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def allreduce_point_gradients(moments, normals, d_epsilon, group=None):
    """Sum flushed point gradients over ranks in place; returns the summed
    d_epsilon. `moments` / `normals` are torch tensors (CUDA for NCCL)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(d_epsilon)
    dist.all_reduce(moments, group=group)
    dist.all_reduce(normals, group=group)
    e = torch.tensor([float(d_epsilon)], dtype=torch.float64, device=moments.device)
    dist.all_reduce(e, group=group)
    return float(e.item())
