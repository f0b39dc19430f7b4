"""GrassSchedule — drives one Grass context through the paper's schedule
(SURVEY.md §1 layer L5):

  steps [0, T_p)        probing: every layer produces gradients, their norms
                        feed the MGN window (grass_mgn_accumulate), no update;
  step T_p, then every  commit the window (first commit / Eq. 4 EMA), Eq. 3
  T_u (multiple of T_s) probabilities (grass_update_probs);
  step T_p + k*T_s      resample the trainable set (grass_sample_layers) and,
                        with period residency, prefetch its optimizer states
                        (grass_prefetch_layers) so they move during fwd/bwd;
  other steps           keep the set; update it (grass_step_layers).

Always-active groups (Grass(n_always=k): embedding / head, DESIGN R19) are not
probed or sampled; they join every adaptive step's update.

graphs=True: the update of an adaptive step is a CUDA graph captured once
per trainable set (i.e. once per sampling period) and replayed on the other
steps of the period, with eta read from a device scalar (grass_set_lr_device)
— for HBM-resident states, the per-step offload pipeline and period
residency (the period's layers are prefetched, so they are cached).

trace_path: optional JSON-lines log of the sampling state (SPEC.md:313's
prob-trace): one record per commit {"step", "event": "commit", "m", "p"} and
per resample {"step", "event": "resample", "period", "sampled"}.

Host logic only: every step of the hot path runs in libgrass.so.

    sched = GrassSchedule(grass)
    for step in range(n_steps):
        layers = sched.begin_step(step)      # which layers need gradients
        ... forward / backward producing gradients of `layers` ...
        sched.end_step(step, params, grads, lr)
"""
from __future__ import annotations

import json
from typing import Sequence

from .binding import (DECIDE_COMMIT_RESAMPLE, DECIDE_PROBE, DECIDE_RESAMPLE, Grass,
                      schedule_decision)


class GrassSchedule:
    def __init__(self, grass: Grass, prefetch: bool | None = None, trace_path: str | None = None,
                 graphs: bool = False):
        self.g = grass
        self.trace_path = trace_path
        cfg = grass.cfg
        self.graphs = graphs
        self._graph, self._gkey, self._lr = None, None, None
        if graphs:
            if cfg.offload and cfg.residency == 2:
                raise ValueError("graphs: GRASS_RESIDENCY_STEP_PREFETCH fetches every step (not capturable)")
            import torch
            self._lr = torch.zeros((), dtype=torch.float32, device=torch.device("cuda", cfg.device))
            grass.set_lr_device(self._lr)
        self.T_p, self.T_s, self.T_u = cfg.T_p, cfg.T_s, cfg.T_u
        self.n_layers = grass.n_layers
        self.always = list(getattr(grass, "always_ids", []))
        self.n_sampled = self.n_layers - len(self.always)
        # prefetch needs whole-layer device slots: period residency prefetches at
        # each resample, the per-step round trip (STEP_PREFETCH) at every step
        slots = bool(cfg.offload) and cfg.residency in (1, 2)   # PERIOD, STEP_PREFETCH
        self.prefetch = slots if prefetch is None else (prefetch and slots)
        self.prefetch_every_step = bool(cfg.offload) and cfg.residency == 2
        self.trainable: list[int] = []
        self.probs: list[float] | None = None
        self.period_index = -1

    def decision(self, step: int) -> int:
        return schedule_decision(step, self.T_p, self.T_s, self.T_u)

    def begin_step(self, step: int, stream=None) -> list[int]:
        """Layers that must produce gradients this step (all of them while
        probing).  At period boundaries commits / resamples / prefetches."""
        d = self.decision(step)
        if d == DECIDE_PROBE:
            return list(range(self.n_sampled))
        if d == DECIDE_COMMIT_RESAMPLE:
            self.probs = self.g.update_probs()
            if self.trace_path:
                m = self.g.get_mgn()["m"] if hasattr(self.g, "get_mgn") else None
                self._log({"step": step, "event": "commit", "m": m, "p": self.probs})
        if d in (DECIDE_COMMIT_RESAMPLE, DECIDE_RESAMPLE) or not self.trainable:
            self.period_index = (step - self.T_p) // self.T_s
            self.trainable = self.g.sample_layers(self.period_index)
            if self.trace_path:
                self._log({"step": step, "event": "resample", "period": self.period_index,
                           "sampled": list(self.trainable)})
            if self.prefetch and not self.prefetch_every_step:
                self.g.prefetch_layers(self.trainable, stream=stream)
        if self.prefetch and self.prefetch_every_step:
            self.g.prefetch_layers(self.trainable, stream=stream)   # fetched during this step's forward
        return list(self.trainable) + self.always

    def end_step(self, step: int, params: Sequence, grads: Sequence, lr: float, stream=None):
        """params / grads: one entry per layer of begin_step(step), same order."""
        layers = (list(range(self.n_sampled)) if self.decision(step) == DECIDE_PROBE
                  else self.trainable + self.always)
        if len(grads) != len(layers):
            raise ValueError("one gradient per layer returned by begin_step")
        if self.decision(step) == DECIDE_PROBE:
            self.g.mgn_accumulate(layers, grads, stream=stream)   # no update
        else:
            if len(params) != len(layers):
                raise ValueError("one parameter buffer per trainable layer")
            if not self.graphs:
                self.g.step_layers(layers, params, grads, lr, stream=stream)
                return
            import torch
            key = (tuple(layers), tuple(p.data_ptr() for p in params), tuple(g.data_ptr() for g in grads))
            if key != self._gkey:                 # new trainable set (or buffers): capture once
                torch.cuda.synchronize()
                self.g.sync()                     # capture preconditions (copies / fills complete)
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    self.g.step_layers(layers, params, grads, 0.0, stream=torch.cuda.current_stream())
                self._graph, self._gkey = graph, key
            s = torch.cuda.current_stream() if stream is None else stream
            with torch.cuda.stream(s):
                self._lr.fill_(lr)
                self._graph.replay()

    def _log(self, rec: dict):
        with open(self.trace_path, "a") as f:
            f.write(json.dumps(rec) + "\n")
