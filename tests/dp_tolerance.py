"""Tolerances of the data-parallel parity tests (test infrastructure, no
method arithmetic beyond error bounds).

The oracle defines the DP gradient as the fp64 mean over ranks (O.dp_average,
reading R9).  Both GPU data paths (P2P and NCCL) form it as reading R20 says:
an fp32 sum in ascending rank order, then x fp32(1/W).  The standard bound of
that evaluation — W - 1 fp32 additions, each rounding by at most 2^-24 of its
partial sum (|partial| <= sum_r |g_r|), then one more rounding for the scale
(exact for power-of-two W) — is

    |g_fp32 - g_mean| <= dg = ((W - 1) * sum_r |g_r| / W + 2 |g_mean|) * 2^-24

elementwise.  The parity bars of DESIGN §6 (norms 1e-6 relative; theta, m, v
1e-5 of the operands of their final rounding) are checked against the oracle
fed with the fp64 mean, with dg propagated through one AdamW step to first
order (times 2) added to the theta / m / v bars.  Where the ranks' gradients
cancel, an fp32 sum cannot be relatively accurate, so no fixed relative bar
alone could hold there; everywhere else the allowance is ~1e-7 relative.
"""
import math

import numpy as np

U = 2.0 ** -24


def dp_sum_bound(grads_per_rank):
    """dg above, fp64 elementwise."""
    g = [np.asarray(x, np.float64) for x in grads_per_rank]
    W = len(g)
    mean = sum(g) / W
    return ((W - 1) * sum(np.abs(x) for x in g) / W + 2.0 * np.abs(mean)) * U


def adamw_allowance(m_out, v_out, g_mean, dg, t, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """First-order effect of a gradient error dg on (theta', m', v') of one
    AdamW step, x 2: dm = (1-b1) dg; dv = (1-b2)(2|g| dg + dg^2); theta' =
    theta1 - s m'/D with D = sqrt(v')/sqrt(bc2) + eps, s = lr/bc1:
    |d theta'| <= s dm / D + s |m'| dD / D^2, dD = min(dv / (2 sqrt v'), sqrt dv) / sqrt(bc2)."""
    m_out, v_out = np.asarray(m_out, np.float64), np.asarray(v_out, np.float64)
    g, dg = np.abs(np.asarray(g_mean, np.float64)), np.asarray(dg, np.float64)
    s = lr / (1.0 - beta1 ** t)
    ibc2 = 1.0 / math.sqrt(1.0 - beta2 ** t)
    dm = (1.0 - beta1) * dg
    dv = (1.0 - beta2) * (2.0 * g * dg + dg * dg)
    sq = np.sqrt(v_out)
    with np.errstate(divide="ignore", invalid="ignore"):
        dD = ibc2 * np.minimum(np.where(sq > 0, dv / (2.0 * sq), np.inf), np.sqrt(dv))
    D = sq * ibc2 + eps
    dth = s * dm / D + s * np.abs(m_out) * dD / (D * D)
    return 2.0 * dth, 2.0 * dm, 2.0 * dv


def assert_dp_state_close(th, m, v, th_o, m_o, v_o, th_in, m_in, g_mean, dg, t, lr, rtol=1e-5, where=""):
    """theta / m / v of the GPU vs the oracle fed with the fp64 mean: the DESIGN
    §6 bars (operand scales) + the propagated DP-summation allowance."""
    th, m, v = (np.asarray(x, np.float64) for x in (th, m, v))
    th_o, m_o, v_o = (np.asarray(x, np.float64) for x in (th_o, m_o, v_o))
    th_in, m_in, g = (np.asarray(x, np.float64) for x in (th_in, m_in, g_mean))
    a_th, a_m, a_v = adamw_allowance(m_o, v_o, g, dg, t, lr)
    s_th = np.maximum(np.abs(th_o), np.abs(th_in))
    s_m = np.maximum.reduce([np.abs(m_o), np.abs(m_in), 0.1 * np.abs(g)])
    s_v = np.abs(v_o)
    for name, a, b, s, al in (("theta", th, th_o, s_th, a_th), ("m", m, m_o, s_m, a_m), ("v", v, v_o, s_v, a_v)):
        err = np.abs(a - b)
        bad = err > rtol * s + al + 1e-30
        assert not bad.any(), (where, name, int(bad.sum()), float((err / np.maximum(rtol * s + al, 1e-300)).max()))
