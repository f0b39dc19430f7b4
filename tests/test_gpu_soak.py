"""Soak: the whole schedule (probe, commits, resamples, prefetch) for 300 steps
on three residency modes driven by GrassSchedule — resident, per-step offload
and period residency with prefetch — must stay bit-identical to each other
(parameters, m, v, t, MGN) and leak no host memory or device events per step.
"""
import os

import numpy as np
import pytest
import torch

import paper_2604_07808_b200 as G
from synth import grad_sigmas, layer_grad, layer_params

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _rss_mb():
    with open(f"/proc/{os.getpid()}/status") as f:
        for line in f:
            if line.startswith("VmRSS:"):
                return int(line.split()[1]) / 1024.0
    return 0.0


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def test_soak_300_steps_three_modes_bit_identical():
    nl = 12
    numel = [(1 << 18) + 4096 * (l % 5) + 4 * l for l in range(nl)]
    sig = grad_sigmas(nl, 5)
    common = dict(gamma=3, T_p=5, T_s=3, T_u=6, seed=77, weight_decay=0.01)
    modes = {"resident": {}, "offload": dict(offload=True, chunk_elems=1 << 16, ring_slots=2),
             "period": dict(offload=True, residency=G.RESIDENCY_PERIOD, cache_layers=4)}
    ctx = {k: G.Grass(numel, **common, **kw) for k, kw in modes.items()}
    sched = {k: G.GrassSchedule(g) for k, g in ctx.items()}
    base = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    P = {k: [b.clone() for b in base] for k in modes}
    rss = {}
    for step in range(300):
        layers = None
        for k in modes:
            ly = sched[k].begin_step(step)
            assert layers is None or ly == layers, (step, k)
            layers = ly
        grads = [layer_grad(numel[l], l, sig[l], step=step, device=DEV) for l in layers]
        for k in modes:
            sched[k].end_step(step, [P[k][l] for l in layers], grads, 1e-3)
        if step in (100, 299):
            torch.cuda.synchronize()
            rss[step] = _rss_mb()
    for g in ctx.values():
        g.sync()
    for k in ("offload", "period"):
        for l in range(nl):
            assert torch.equal(P["resident"][l], P[k][l]), (k, l)
            a, b = ctx["resident"].read_state(l), ctx[k].read_state(l)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2], (k, l)
        sa, sb = ctx["resident"].get_mgn(), ctx[k].get_mgn()
        assert sa["m"] == sb["m"] and sa["S"] == sb["S"] and sa["c"] == sb["c"]
    assert sum(ctx["resident"].read_state(l)[2] for l in range(nl)) == 3 * (300 - 5)
    assert rss[299] - rss[100] < 64, rss                 # no per-step host growth
