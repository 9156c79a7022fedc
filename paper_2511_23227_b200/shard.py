"""Multi-GPU plumbing for the batched config.

Whole point clouds of a batch are the unit of sharding: rank r of W owns the
contiguous scene range ``scene_range(n, r, W)``; neighbor build, forward and
input gradient never cross scenes (spatial.cpp:68-77), so no data-path
collective exists.  The one exchange is the weight gradient, a sum over
triplets (vvor.hpp:79-84): dW = sum over ranks, one all-reduce per layer
backward (NCCL over NVLink on the GPU box; gloo in the CPU tests).

`DwComm` is the library's own all-reduce (npcg_allreduce_dw, NCCL on the
library's stream, include/npcg.h); torch.distributed only carries the NCCL
unique id from rank 0 to the others.  `allreduce_weight_grad` is the same
sum through torch.distributed (used for the gloo CPU tests).
"""
from __future__ import annotations

import ctypes as C

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


class DwComm:
    """NCCL communicator of the library (one per rank); `allreduce(dw)` sums a
    device weight gradient over ranks in place, stream-ordered on the
    library context's stream."""

    def __init__(self, rank: int, world: int, device=None):
        from . import _lib as L
        from . import npconv as npc
        self._L = L
        self.ctx = npc.context(device)
        idb = (C.c_uint8 * 128)()
        if rank == 0:
            self.ctx.check(L.lib().npcg_comm_unique_id(C.cast(idb, C.c_void_p)), "comm_unique_id")
        if world > 1:
            obj = [bytes(idb)]
            dist.broadcast_object_list(obj, src=0)
            C.memmove(idb, obj[0], 128)
        h = C.c_void_p()
        hc = self.ctx.bind()
        self.ctx.check(L.lib().npcg_comm_create(hc, world, rank, C.cast(idb, C.c_void_p),
                                                C.byref(h)), "comm_create")
        self.h = h
        self.world = world

    def allreduce(self, dw: torch.Tensor) -> torch.Tensor:
        from . import npconv as npc
        if not dw.is_contiguous():
            raise npc.ShapeError("allreduce: dW must be contiguous")
        code = {torch.float32: 0, torch.float64: 1}.get(dw.dtype)
        if code is None:
            raise npc.ShapeError("allreduce: dW must be float32 / float64")
        hc = self.ctx.bind()
        self.ctx.check(self._L.lib().npcg_allreduce_dw(hc, self.h, code, C.c_void_p(dw.data_ptr()),
                                                      dw.numel()), "allreduce_dw")
        return dw

    def close(self):
        if self.h:
            self._L.lib().npcg_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
