"""Attaching a PyTorch model to libgrass: layer-wise GRASS training with flat
per-block buffers.

GRASS samples whole decoder blocks.  The library's unit is one
flat, contiguous buffer per block (include/grass.h), so `GrassBlocks`
re-homes each block's parameters — and their gradients — into one flat buffer
per block, registers them with a `Grass` context (blocks first, then the
always-active groups such as embedding / head, DESIGN R19) and drives the
schedule:

    gb = GrassBlocks(model.blocks, always=[model.embed.parameters(), model.head.parameters()],
                     gamma=2, T_p=150, T_s=25, offload=True, residency=G.RESIDENCY_PERIOD)
    for step in range(n_steps):
        gb.begin_step(step)          # freezes the blocks not trained this step
        loss = model(batch).loss
        loss.backward()
        gb.end_step(step, lr)        # probing norms, or the fused norm + AdamW of the trainable set
        gb.zero_grad()

Or one call per step, `loss = gb.train_step(step, loss_fn, lr)`, where
loss_fn() runs the forward on the caller's (static) input tensors and returns
the scalar loss.  With step_graphs=True the WHOLE adaptive step — forward,
backward, the fused norm + AdamW of the trainable set and the gradient reset —
is one CUDA graph per sampling period: the period's first step runs eagerly
(and is the capture's warm-up), its second is captured and every later one is
a replay, with eta read from a device scalar (grass_set_lr_device).  Probing
steps and the period boundaries (commit / resample / prefetch, host work) stay
eager.  The caller refills its input tensors in place between steps.

This is plumbing (PyTorch owns the buffers and autograd); every step of the
hot path runs in libgrass.
"""
from __future__ import annotations

from typing import Iterable, Sequence

import torch

from .binding import DECIDE_PROBE, DTYPE_BF16, DTYPE_FP32, Grass
from .schedule import GrassSchedule


def flatten_params(params: Iterable[torch.nn.Parameter]):
    """Re-homes the parameters (and gradients) into two flat buffers of the
    parameters' dtype; the parameters become views.  Returns (flat, gflat)."""
    params = [p for p in params]
    if not params:
        raise ValueError("no parameters")
    dt, dev = params[0].dtype, params[0].device
    if any(p.dtype != dt or p.device != dev for p in params):
        raise ValueError("a flattened group needs one dtype and one device")
    n = sum(p.numel() for p in params)
    flat = torch.empty(n, dtype=dt, device=dev)
    gflat = torch.zeros(n, dtype=dt, device=dev)
    off = 0
    for p in params:
        k = p.numel()
        flat[off:off + k].copy_(p.data.reshape(-1))
        p.data = flat[off:off + k].view_as(p)
        p.grad = gflat[off:off + k].view_as(p)   # autograd accumulates into the flat buffer
        off += k
    return flat, gflat


class GrassBlocks:
    """A model's decoder blocks (sampled by GRASS) and optional always-active
    parameter groups, bound to one `Grass` context (keyword arguments are
    `Grass`'s, e.g. gamma, T_p, T_s, offload, residency, param_dtype)."""

    def __init__(self, blocks: Sequence[torch.nn.Module], always: Sequence[Iterable] = (), graphs: bool = False,
                 step_graphs: bool = False, **grass_kw):
        self.blocks = list(blocks)
        groups = [list(b.parameters()) for b in self.blocks] + [list(a) for a in always]
        self.flats = [flatten_params(g) for g in groups]
        dt = self.flats[0][0].dtype
        if dt not in (torch.float32, torch.bfloat16):
            raise ValueError("fp32 or bf16 parameters")
        grass_kw.setdefault("param_dtype", DTYPE_BF16 if dt == torch.bfloat16 else DTYPE_FP32)
        grass_kw.setdefault("device", self.flats[0][0].device.index or 0)
        self.grass = Grass([f.numel() for f, _ in self.flats], n_always=len(always), **grass_kw)
        if graphs and step_graphs:
            raise ValueError("graphs (update only) and step_graphs (whole step) are exclusive")
        self.schedule = GrassSchedule(self.grass, graphs=graphs)   # graphs: one captured update per period
        self.layers: list[int] = []
        self.step_graphs = step_graphs
        if step_graphs:
            cfg = self.grass.cfg
            if cfg.offload and cfg.residency != 1:
                raise ValueError("step_graphs: HBM-resident states or GRASS_RESIDENCY_PERIOD (cached layers)")
            dev = torch.device("cuda", self.flats[0][0].device.index or 0)
            self._lr = torch.zeros((), dtype=torch.float32, device=dev)
            self.grass.set_lr_device(self._lr)
            self._side = torch.cuda.Stream(device=dev)   # warm-up and capture stream
            self._warm_key = self._graph_key = None
            self._graph, self._graph_loss = None, None

    def begin_step(self, step: int) -> list[int]:
        """Sets requires_grad for this step (trainable blocks + always groups;
        every block while probing) and returns the layer ids of the step."""
        self.layers = self.schedule.begin_step(step)
        active = set(self.layers)
        for l, b in enumerate(self.blocks):
            for p in b.parameters():
                p.requires_grad_(l in active)
        return list(self.layers)

    def end_step(self, step: int, lr: float, stream=None):
        ids = self.layers
        self.schedule.end_step(step, [self.flats[l][0] for l in ids], [self.flats[l][1] for l in ids], lr,
                               stream=stream)

    def zero_grad(self):
        for _, g in self.flats:
            g.zero_()

    def train_step(self, step: int, loss_fn, lr: float) -> torch.Tensor:
        """One training step: begin_step, loss_fn() + backward, end_step,
        zero_grad.  Returns the (detached) loss; under step_graphs it is the
        graph's static loss tensor, valid until the next call."""
        ids = self.begin_step(step)
        if not self.step_graphs or self.schedule.decision(step) == DECIDE_PROBE:
            loss = loss_fn()
            loss.backward()
            self.end_step(step, lr)
            self.zero_grad()
            return loss.detach()
        self._lr.fill_(lr)
        key = (tuple(ids), self.schedule.period_index)
        cur = torch.cuda.current_stream()
        if key != self._warm_key:          # first step of the period: eager, on the capture stream
            self._warm_key = key
            self._side.wait_stream(cur)
            with torch.cuda.stream(self._side):
                loss = self._step_body(loss_fn)
            cur.wait_stream(self._side)
            loss.record_stream(cur)
            return loss
        if key != self._graph_key:         # second step: capture once (the graph is not run by capture)
            self._graph = self._graph_loss = None
            torch.cuda.synchronize()
            self.grass.sync()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=self._side):
                self._graph_loss = self._step_body(loss_fn)
            self._graph, self._graph_key = graph, key
        self._graph.replay()
        return self._graph_loss

    def _step_body(self, loss_fn) -> torch.Tensor:
        """forward, backward, the library update of the trainable set (eta from
        the device scalar) and the gradient reset, on the current stream."""
        loss = loss_fn()
        loss.backward()
        ids = self.layers
        self.grass.step_layers(ids, [self.flats[l][0] for l in ids], [self.flats[l][1] for l in ids], 0.0,
                               stream=torch.cuda.current_stream())
        self.zero_grad()
        return loss.detach()
