"""Multi-GPU host logic: view sharding (configs 3/4) and the gradient exchange (config 4).

One process per GPU (torch.distributed; NCCL on the B200 box, gloo in the CPU
tests).  Views are independent units of the forward pass:
primitives are replicated on every rank and each rank renders its own shard of
the views, so the forward has no data-path collective.  The training step has
one real exchange: the raw-parameter gradient buffer (n x scalar_count f32,
ABI layout) is summed across ranks and divided by the total number of views,
then every rank applies the same Adam update (replicas stay bit-identical
because NCCL's all-reduce returns the same sum on every rank).
"""
from __future__ import annotations

import numpy as np


def shard_views(n_views: int, world: int, rank: int, costs=None) -> list[int]:
    """Views rendered by `rank`.  With per-view cost estimates (e.g. tile-pair
    counts from a previous pass), greedy longest-processing-time assignment;
    otherwise contiguous equal blocks.  Every view is owned by exactly one rank."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    if costs is None:
        lo = n_views * rank // world
        hi = n_views * (rank + 1) // world
        return list(range(lo, hi))
    costs = np.asarray(costs, dtype=np.float64)
    if costs.shape != (n_views,):
        raise ValueError("one cost per view")
    load = np.zeros(world)
    owner = np.empty(n_views, dtype=np.int64)
    for v in np.argsort(-costs, kind="stable"):
        r = int(np.argmin(load))
        owner[v] = r
        load[r] += costs[v]
    return [int(v) for v in np.nonzero(owner == rank)[0]]


def allreduce_mean_(grad, total_views: int, group=None):
    """In-place sum of the per-rank accumulated gradients, divided by the
    total number of views (the multi-view gradient of SURVEY.md §8(d) is the
    mean over views of per-view backward_render)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    grad.mul_(1.0 / float(total_views))
    return grad


def params_checksum(params) -> float:
    """Order-independent fp64 checksum used to verify that replicas stay in sync."""
    import torch
    p = params.detach().to(torch.float64)
    return float((p * torch.arange(1, p.numel() + 1, dtype=torch.float64, device=p.device).reshape(p.shape)
                  .remainder(7.0).add(1.0)).sum())
