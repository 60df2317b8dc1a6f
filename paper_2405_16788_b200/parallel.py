"""Multi-GPU plumbing for the dipole engine.

Queries are independent given the tree, so the path shards with a REPLICATED
tree (every rank builds the same tree bit-for-bit from the same cloud) and
contiguous query shards. Forward needs no collective. The adjoint's only
exchange is the sum of the flushed per-point gradients (moments N x C,
normals N x 3, d_epsilon) across ranks — one NCCL all-reduce over NVLink
(torch.distributed, backend "nccl"; "gloo" in the CPU tests).

The config-5 training step shards the point update instead:
reduce-scatter of the gradients, Adam on each rank's 1/G of the points,
all-gather of the updated parameters, update_moments on every rank
(`sharded_point_update`).
"""
from __future__ import annotations

import contextlib


def _nullctx():
    return contextlib.nullcontext()


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


def flush_allreduce(tree, buffers, rows=None, chunks=8, group=None, out=None):
    """flush_gradients summed over ranks, overlapped chunk by chunk.

    Every rank holds the bit-identical tree, so gradient rows in TREE order line
    up across ranks: the push-down runs once (`flush_begin`), then for each of
    `chunks` contiguous sorted-point ranges the rows are computed on the tree's
    stream and handed to an asynchronous all-reduce — NCCL waits for that
    chunk only, so the sum of chunk k runs on the NCCL stream while chunk k+1
    is computed. The summed rows are scattered back to the original order
    (`flush_end`, which also zeroes the buffers). Returns
    (moments N x C, normals N x 3, d_epsilon summed over ranks).

    `rows`: optional preallocated N x (C + 3) fp32 CUDA tensor."""
    import torch
    import torch.distributed as dist

    n, C = tree.point_count(), tree.channels()
    if isinstance(buffers, (list, tuple)):
        b0 = buffers[0]
    else:
        b0, buffers = buffers, [buffers]
    if rows is None:
        rows = torch.empty((n, C + 3), dtype=torch.float32,
                           device=torch.device("cuda", torch.cuda.current_device()))
    dev = rows.device
    de = tree.flush_begin(buffers)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    works = []
    # torch's collectives order against torch's CURRENT stream: make it the
    # tree's stream (a library-owned stream is blocking, i.e. ordered with the
    # legacy default stream already)
    sp = getattr(tree, "stream_ptr", None)
    ctx = (torch.cuda.stream(torch.cuda.ExternalStream(sp)) if sp and dev.type == "cuda"
           else _nullctx())
    with ctx:
        e = torch.tensor([de], dtype=torch.float64, device=dev)
        for k in range(max(1, chunks)):
            lo, hi = shard_range(n, k, max(1, chunks))
            if hi <= lo:
                continue
            tree.flush_rows(b0, lo, hi, rows[lo:hi])
            if world > 1:
                works.append(dist.all_reduce(rows[lo:hi], group=group, async_op=True))
        if world > 1:
            works.append(dist.all_reduce(e, group=group, async_op=True))
        for w in works:
            w.wait()  # the tree's stream waits on the NCCL stream (no host sync)
    mom, nrm = tree.flush_end(buffers, rows, out=out)
    return mom, nrm, float(e.item()) if world > 1 else de


def point_chunk(n: int, rank: int, world: int):
    """Equal-size point slices [lo, hi) of ceil(n / world) (the last may be short):
    the layout reduce-scatter / all-gather need."""
    chunk = -(-n // world) if world > 0 else n
    lo = min(rank * chunk, n)
    return lo, min(lo + chunk, n), chunk


class TreeEngine:
    """The sharded update's device side on a DipoleTree + PointAdam."""

    def __init__(self, tree, opt):
        self.tree, self.opt = tree, opt

    def adam_range(self, g_mom, g_nrm, lo, hi):
        self.opt.step_range(g_mom, g_nrm, lo, hi)

    def get_range(self, lo, hi, nrm_out, mom_out):
        from .bhtree import get_points_range

        get_points_range(self.tree, lo, hi, nrm_out, mom_out)

    def set_all(self, nrm, mom):
        from .bhtree import set_points_range

        set_points_range(self.tree, 0, self.tree.point_count(), nrm, mom)

    def refresh(self):
        from .bhtree import refresh_moments

        refresh_moments(self.tree)


def sharded_point_update(engine, moments, normals, n, channels, group=None):
    """One sharded Trainer::step point update (optimizer.cpp:161-205 split over
    ranks): the flushed per-rank gradients `moments` (n x C) / `normals` (n x 3)
    (torch fp32, same device as the tree for NCCL) are summed and scattered so
    rank r gets the points of point_chunk(n, r, G); Adam runs on that slice
    only; the updated fp64 parameters are all-gathered and written back on
    every rank, then update_moments. Equal to the single-GPU PointAdam.step on
    the summed gradients. NCCL uses reduce_scatter_tensor / all_gather_into_tensor;
    other backends (gloo, CPU tests) all-reduce and all-gather lists."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi, chunk = point_chunk(n, rank, world)
    W = channels + 3
    dev = moments.device
    # gradients as one padded (G chunk) x (C + 3) block
    g = torch.zeros((world * chunk, W), dtype=torch.float32, device=dev)
    g[:n, :channels] = moments.reshape(n, channels)
    g[:n, channels:] = normals.reshape(n, 3)
    nccl = world > 1 and dist.get_backend(group) == "nccl"
    if world == 1:
        mine = g[:chunk]
    elif nccl:
        mine = torch.empty((chunk, W), dtype=torch.float32, device=dev)
        dist.reduce_scatter_tensor(mine, g, group=group)
    else:
        dist.all_reduce(g, group=group)
        mine = g[rank * chunk:(rank + 1) * chunk]
    k = hi - lo
    engine.adam_range(mine[:k, :channels].contiguous(), mine[:k, channels:].contiguous(), lo, hi)
    # updated parameters of the own slice, padded to the chunk
    part = torch.zeros((chunk, W), dtype=torch.float64, device=dev)
    p_mom = torch.empty((k, channels), dtype=torch.float64, device=dev)
    p_nrm = torch.empty((k, 3), dtype=torch.float64, device=dev)
    if k > 0:
        engine.get_range(lo, hi, p_nrm, p_mom)
        part[:k, :channels] = p_mom
        part[:k, channels:] = p_nrm
    if world == 1:
        full = part
    elif nccl:
        full = torch.empty((world * chunk, W), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(full, part, group=group)
    else:
        parts = [torch.empty_like(part) for _ in range(world)]
        dist.all_gather(parts, part, group=group)
        full = torch.cat(parts)
    engine.set_all(full[:n, channels:].contiguous(), full[:n, :channels].contiguous())
    engine.refresh()
