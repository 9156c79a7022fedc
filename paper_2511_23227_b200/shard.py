"""Multi-GPU plumbing for the batched config.

Whole point clouds of a batch are the unit of sharding: rank r of W owns the
contiguous scene range ``scene_range(n, r, W)``; neighbor build, forward and
input gradient never cross scenes (spatial.cpp:68-77), so no data-path
collective exists.  The one exchange is the weight gradient, a sum over
triplets (vvor.hpp:79-84): dW = sum over ranks, one all-reduce per layer
backward (NCCL over NVLink on the GPU box; gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def scene_range(n_scenes: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced (sizes differ by <= 1) scene range of `rank`."""
    base, extra = divmod(n_scenes, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def allreduce_weight_grad(grad_w: torch.Tensor, async_op: bool = False):
    """Sum the per-rank weight gradients in place (fp32 / fp64)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return None
    return dist.all_reduce(grad_w, op=dist.ReduceOp.SUM, async_op=async_op)
