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


def test_soak_device_schedule_600_steps_equals_host_schedule():
    """600 device-resident steps (PDL launches, the fused commit in K3's last
    CTA, its done counter reused every step) on the paper's T_s = T_u = 3
    cadence with an always-active group, against the host-driven schedule:
    the same sampled ids at every period and, at the end, the same parameters,
    m, v, t, MGN and probabilities."""
    numel = [4096 * 3 + 8, 8192, 4096 * 5, 4096, 8192 + 4, 4096 * 2]     # last: always active
    nl, ns = len(numel), len(numel) - 1
    sig = grad_sigmas(nl, 4)
    mk = lambda: G.Grass(numel, gamma=2, T_p=1, T_s=3, T_u=3, seed=21, n_always=1, alpha=0.3, weight_decay=0.01)
    host, dev = mk(), mk()
    Ph = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    Pd = [p.clone() for p in Ph]
    Gr = [torch.zeros(n, device=DEV) for n in numel]
    fill = lambda step: [Gr[l].copy_(layer_grad(n, l, sig[l], step=step % 7, device=DEV)) for l, n in enumerate(numel)]
    fill(0)
    for c in (host, dev):
        c.mgn_accumulate(list(range(ns)), Gr[:ns])
        c.update_probs()
    dev.register_layers(Pd, Gr)
    dev.device_schedule_begin(0)
    ids, period = host.sample_layers(0), 0
    for step in range(1, 601):
        fill(step)
        layers = ids + [ns]
        host.step_layers(layers, [Ph[l] for l in layers], [Gr[l] for l in layers], 1e-3)
        boundary = step % 3 == 0
        dev.device_step(1e-3, commit=boundary, resample=boundary)
        if boundary:
            host.update_probs()
            period += 1
            ids = host.sample_layers(period)
        if step % 150 == 0:
            torch.cuda.synchronize()
    assert dev.device_schedule_end() == ids
    torch.cuda.synchronize()
    for l in range(nl):
        assert torch.equal(Ph[l], Pd[l]), l
        a, b = host.read_state(l), dev.read_state(l)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2], l
    sa, sb = host.get_mgn(), dev.get_mgn()
    assert sa["S"] == sb["S"] and sa["c"] == sb["c"]
    np.testing.assert_allclose(sb["m"], sa["m"], rtol=1e-15, atol=0)
    np.testing.assert_allclose(sb["probs"], sa["probs"], rtol=1e-14, atol=0)
