"""The DP tolerance of the parity tests (tests/dp_tolerance.py) pinned on CPU:
the fp32 rank-order evaluation of the DP mean (reading R20, what both GPU data
paths compute) stays within dp_sum_bound of the fp64 mean (O.dp_average) for
every world size, with cancelling ranks included, and the bound is not
vacuous (~1e-7 relative where the ranks do not cancel)."""
import numpy as np
import pytest
import torch

from dp_tolerance import adamw_allowance, dp_sum_bound
from oracle import grass_oracle as O


def rank_order_fp32(grads):
    """R20 written with torch fp32 tensor ops (not the kernel): sum in
    ascending rank order, then x fp32(1/W)."""
    acc = torch.from_numpy(np.asarray(grads[0], np.float32).copy())
    for g in grads[1:]:
        acc = acc + torch.from_numpy(np.asarray(g, np.float32))
    return (acc * torch.tensor(1.0 / len(grads), dtype=torch.float32)).numpy()


@pytest.mark.parametrize("W", [1, 2, 3, 4, 5, 8])
def test_rank_order_fp32_mean_within_bound(W):
    rng = np.random.default_rng(W)
    n = 200_000
    sig = 10.0 ** rng.uniform(-5, -3, size=W)
    grads = [(rng.standard_normal(n) * s).astype(np.float32) for s in sig]
    if W > 1:   # cancelling ranks on the first 1000 elements
        grads[-1][:1000] = -np.sum(np.stack([g[:1000] for g in grads[:-1]]), axis=0).astype(np.float32)
    mean, dg = O.dp_average(grads), dp_sum_bound(grads)
    err = np.abs(rank_order_fp32(grads).astype(np.float64) - mean)
    assert (err <= dg).all()
    ok = np.abs(mean) * W >= 0.5 * sum(np.abs(g.astype(np.float64)) for g in grads)
    assert np.median(dg[ok] / np.abs(mean[ok])) < 1e-6


def test_allowance_first_order_and_small():
    g = np.array([1e-3, -2e-4, 1e-9, 0.0])
    dg = np.array([1e-10, 1e-11, 1e-12, 0.0])
    m = 0.1 * g
    v = 0.001 * g * g
    th, dm, dv = adamw_allowance(m, v, g, dg, 1, 3e-5)
    assert np.allclose(dm, 2 * 0.1 * dg, rtol=1e-12, atol=0) and (dv >= 0).all() and np.isfinite(th).all()
    assert th[-1] == 0.0 and dm[-1] == 0.0
    assert th[0] < 1e-6 * 3e-5            # ~1e-7 of the step where g >> eps
