"""Seed-sharded data parallelism for the fused operator.

Every output row of the fused sample + mean depends only on (graph, features, seed node, the
seed's GLOBAL batch position, base seed) (kernels.py:155-198), so a global batch splits into
contiguous position ranges, one per rank, with no collective on the data path: rank g runs the
operator on positions [lo, hi) with ``root_offset = lo`` and its rows are bitwise identical to
the same rows of a single-device run.  Graph and features are replicated per GPU.

The only collective is the SAGE head's gradient all-reduce (train.py), one flattened buffer per
step, NCCL on GPUs (gloo in the CPU tests).
"""

from __future__ import annotations

from typing import Dict, Optional, Tuple

import torch

__all__ = ["shard_bounds", "shard_batch", "allreduce_grads", "dist_info"]


def dist_info(group=None) -> Tuple[int, int]:
    """(rank, world size) of the default (or given) process group; (0, 1) without one."""
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        return torch.distributed.get_rank(group), torch.distributed.get_world_size(group)
    return 0, 1


def shard_bounds(global_batch: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous global positions [lo, hi) of ``rank``; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    if global_batch < 0:
        raise ValueError("batch size must be >= 0")
    base, extra = divmod(global_batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_batch(seeds: torch.Tensor, rank: int, world: int) -> Tuple[torch.Tensor, int]:
    """This rank's slice of a global seed batch and its ``root_offset`` (= first position)."""
    lo, hi = shard_bounds(int(seeds.numel()), rank, world)
    return seeds[lo:hi], lo


def allreduce_grads(grads: Dict[str, torch.Tensor], group=None, average: bool = True,
                    flat: Optional[torch.Tensor] = None, weight: Optional[float] = None) -> Dict[str, torch.Tensor]:
    """All-reduce a dict of gradients in ONE collective on a flattened buffer (in place).

    ``weight`` (this rank's seeds / global seeds) scales each rank's batch means before the sum,
    giving the global-batch mean also when shard sizes differ by one (shard_bounds); without it
    ``average`` divides the sum by the world size (equal shards).  ``flat`` may supply a
    persistent buffer of the total size (no allocation, CUDA-graph friendly).  With an explicit
    ``weight`` the collective runs even in a world of one (a captured step keeps its shape)."""
    rank, world = dist_info(group)
    if world == 1 and weight is None:
        return grads
    names = list(grads)
    total = sum(grads[n].numel() for n in names)
    first = grads[names[0]]
    if flat is None:
        flat = torch.empty(total, dtype=first.dtype, device=first.device)
    off = 0
    for n in names:
        k = grads[n].numel()
        flat[off:off + k].copy_(grads[n].reshape(-1))
        off += k
    if weight is not None:
        flat.mul_(weight)
    if world > 1 or torch.distributed.is_initialized():
        torch.distributed.all_reduce(flat, op=torch.distributed.ReduceOp.SUM, group=group)
    if weight is None and average:
        flat.div_(world)
    off = 0
    for n in names:
        k = grads[n].numel()
        grads[n].copy_(flat[off:off + k].view_as(grads[n]))
        off += k
    return grads
