"""Layer stacks over one cached neighbor structure.

The reference composes layers by calling PointConvOp::forward layer after
layer (test_conv_op.cpp:291-309); each op keeps its own triplet cache keyed by
the cloud's identity (conv_op.hpp:106-127), so a stack of L layers on one
cloud builds L identical caches.  ConvStack keeps the operator semantics
(no bias, no activation, the saved forward inputs feed the backward) but
shares ONE device-resident neighbor handle across the layers of a geometry,
keeps every activation on the device, and can capture a whole
forward + backward step into a CUDA graph: after the first (plan-building)
step, a step is a fixed sequence of the library's kernel launches with no
host synchronisation, which a graph replays without per-launch CPU cost.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import npconv as npc


@dataclass
class StackGrads:
    grad_in: torch.Tensor          # w.r.t. the stack's input features
    grad_w: list[torch.Tensor]     # per layer, (K, G, C_out, C_in) (vvor.hpp:12-16)


class ConvStack:
    """Layers l = 0..L-1 with weights (K, G, C_l, C_{l+1}) sharing one geometry."""

    def __init__(self, weights: list[torch.Tensor], geometry: npc.ConvGeometry,
                 config: npc.ExecConfig = npc.ExecConfig(), comm=None):
        """comm: a shard.DwComm (data-parallel training over whole clouds,
        SURVEY.md §8e): each layer's weight gradient is summed over ranks on a
        side stream while the next (lower) layer's backward runs."""
        if not weights:
            raise npc.ShapeError("ConvStack: no layers")
        for a, b in zip(weights, weights[1:]):
            if a.shape[3] != b.shape[2] or a.shape[0] != b.shape[0] or a.shape[1] != b.shape[1]:
                raise npc.ShapeError("ConvStack: consecutive layer shapes do not chain")
        if geometry.mode != npc.ConvMode.native:
            # layer l >= 1 would see one row per site while the degraded forward
            # gathers fine rows through kept_index (conv_op.hpp:133-158)
            raise npc.ShapeError("ConvStack: degraded geometry is not chainable (native only)")
        self.ops = [npc.PointConvOp(w, geometry, config, copy_fin=False) for w in weights]
        self.geometry = geometry
        self.config = config
        self._nb: npc.Neighbors | None = None
        self._key = None
        self._acts: list[torch.Tensor] = []
        self._graph = None
        self.comm = comm
        self._comm_stream = None

    # -- shared cache (conv_op.hpp:106-127, one build for all layers) ----------
    def neighbors(self, cloud: npc.PointCloud) -> npc.Neighbors:
        key = (cloud.xyz.data_ptr(), cloud.n_points())
        if self._nb is None or key != self._key:
            self._nb = npc.build_neighbors(cloud, cloud, self.geometry)
            self._key = key
            self._graph = None
            for op in self.ops:  # every layer sees the same handle
                op._nb, op._key, op._sorted = self._nb, (key[0], key[0], key[1], key[1]), None
        return self._nb

    def forward(self, cloud: npc.PointCloud, fin: torch.Tensor) -> torch.Tensor:
        nb = self.neighbors(cloud)
        self._acts = [fin.contiguous()]
        h = self._acts[0]
        for op in self.ops:
            h = npc.conv_forward(nb, op.weights(), h, self.config)
            self._acts.append(h)
        return h

    def backward(self, gout: torch.Tensor) -> StackGrads:
        if len(self._acts) != len(self.ops) + 1:
            raise npc.StateError("ConvStack::backward: no cached forward inputs")
        g = gout.contiguous()
        gws = [None] * len(self.ops)
        main = torch.cuda.current_stream()
        if self.comm is not None and self._comm_stream is None:
            self._comm_stream = torch.cuda.Stream(device=main.device)
        for l in range(len(self.ops) - 1, -1, -1):
            # activations are the stack's own buffers, unmodified since the forward
            g, gws[l] = npc.conv_backward(self._nb, self.ops[l].weights(), self._acts[l], g,
                                          self.config, need_in=True, need_w=True,
                                          fin_unchanged=True)
            if self.comm is not None:
                # layer l's dW all-reduce overlaps layer l-1's backward (the one
                # exchange of data-parallel training)
                side = self._comm_stream
                side.wait_stream(main)
                gws[l].record_stream(side)
                with torch.cuda.stream(side):
                    self.comm.allreduce(gws[l])
        if self.comm is not None:
            main.wait_stream(self._comm_stream)
            npc.context(main.device).bind()  # the library context back on this stream
        return StackGrads(g, gws)

    # -- CUDA graph of one forward + backward step ------------------------------
    def capture(self, cloud: npc.PointCloud, fin: torch.Tensor, gout: torch.Tensor):
        """Warms the plans up eagerly, then records forward + backward into a
        CUDA graph over static input buffers (copy new inputs into
        `static_fin` / `static_gout`, call replay(), read `static_out` and
        `static_grads`).  Needs a plan without capacity spills (the spill
        path sizes its work on the host)."""
        self.forward(cloud, fin)
        self.backward(gout)
        torch.cuda.synchronize()
        self.static_fin = fin.clone()
        self.static_gout = gout.clone()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # one more eager step on the capture stream
            self.forward(cloud, self.static_fin)
            self.backward(self.static_gout)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.static_out = self.forward(cloud, self.static_fin)
            self.static_grads = self.backward(self.static_gout)
        self._graph = g
        return g

    def replay(self):
        if self._graph is None:
            raise npc.StateError("ConvStack::replay: no captured graph")
        self._graph.replay()
        return self.static_out, self.static_grads
