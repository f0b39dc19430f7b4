"""Pins the ORACLE to things other than itself (CPU only).

Each check is chosen so a plausible mistake in oracle/grass_oracle.py (a
dropped term, a wrong sign or index, a transposed operand, a wrong rounding
point) fails at least one of them: exact rational arithmetic, published test
vectors, closed forms, limits, invariants and library routines
(scipy/torch) — never a re-typed copy of the oracle's own formula.
"""
import math
import random
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import grass_oracle as O

pytestmark = pytest.mark.filterwarnings("ignore")


# ----------------------------------------------------------------- Eq. 2 norm
def test_norm_spec_examples(golden):
    for ex in golden("spec_examples.json")["norm"]:
        g = np.array(ex["g"], np.float32)
        assert O.rms_norm(O.sq_norm(g), g.size) == ex["rms"], ex["cite"]


@pytest.mark.parametrize("n", [1, 7, 1000, 40_000])
def test_sq_norm_equals_exact_rational_sum(n):
    rng = np.random.default_rng(n)
    g = (rng.standard_normal(n) * rng.uniform(1e-6, 10.0)).astype(np.float32)
    exact = sum(Fraction(float(x)) ** 2 for x in g)       # exact, no rounding at all
    assert O.sq_norm(g) == float(exact)                    # correctly rounded


def test_sq_norm_integer_grads_exact_chunked_path():
    # > _FSUM_LIMIT elements exercises the chunked path; integer squares sum exactly.
    rng = np.random.default_rng(3)
    g = rng.integers(-3, 4, size=(1 << 23) + 13).astype(np.float32)
    exact = int(np.sum(g.astype(np.int64) ** 2))
    assert O.sq_norm(g) == float(exact)


def test_rms_constant_grad_is_abs_value():
    for c in (0.5, -3.0, 2.0 ** -20):
        g = np.full(1 << 17, c, np.float32)
        assert O.rms_norm(O.sq_norm(g), g.size) == abs(c)


def test_rms_uses_true_numel_not_padding():
    g = np.array([3.0, 4.0, 0.0, 0.0], np.float32)   # padded by two zeros
    assert O.rms_norm(O.sq_norm(g), 2) == math.sqrt(12.5)
    assert O.rms_norm(O.sq_norm(g), 4) == math.sqrt(6.25)


def test_dp_average_is_mean_over_ranks():
    a = np.array([1.0, 2.0], np.float32)
    b = np.array([3.0, -2.0], np.float32)
    assert O.dp_average([a, b]).tolist() == [2.0, 0.0]
    assert O.dp_average([a]).tolist() == [1.0, 2.0]


# ------------------------------------------------------ Eq. 2 window + Eq. 4 EMA
def test_window_and_ema_spec_examples(golden):
    ex = golden("spec_examples.json")
    for w in ex["window"]:
        st = O.MgnState(1)
        for r in w["r"]:
            st.record(0, r)
        assert st.commit(0.5)[0] == pytest.approx(w["mgn"], rel=0, abs=1e-15), w["cite"]
    for e in ex["ema"]:
        st = O.MgnState(1)
        st.record(0, e["prev"]); st.commit(e["alpha"])           # first commit = window
        st.record(0, e["window"])
        assert st.commit(e["alpha"])[0] == e["out"], e["cite"]


def test_first_commit_has_no_ema():
    st = O.MgnState(2)
    st.record(0, 1.0); st.record(1, 5.0)
    assert st.commit(0.25) == [1.0, 5.0]


def test_streaming_commit_equals_bruteforce_recomputation():
    # retain every raw gradient, evaluate Eq. 2 + Eq. 4 directly
    # with exact rationals, compare with the streaming state machine.
    rng = np.random.default_rng(0)
    n_layers, numel, alpha = 4, 33, 0.5
    st = O.MgnState(n_layers)
    committed = [None] * n_layers
    for window in range(5):
        raw = {l: [] for l in range(n_layers)}
        for t in range(10):
            active = range(n_layers) if window == 0 else rng.choice(n_layers, 2, replace=False)
            for l in active:
                g = rng.standard_normal(numel).astype(np.float32) * (l + 1)
                raw[int(l)].append(g)
                st.record(int(l), O.rms_norm(O.sq_norm(g), numel))
        got = st.commit(alpha)
        for l in range(n_layers):
            if raw[l]:
                rs = [math.sqrt(float(sum(Fraction(float(x)) ** 2 for x in g)) / numel) for g in raw[l]]
                w = sum(rs) / len(rs)
                committed[l] = w if committed[l] is None else alpha * w + (1 - alpha) * committed[l]
            assert got[l] == pytest.approx(committed[l], rel=1e-12), (window, l)


def test_frozen_layers_retain_and_fixed_point():
    st = O.MgnState(3)
    for l, r in enumerate([1.0, 2.0, 3.0]):
        st.record(l, r)
    st.commit(0.5)
    st.record(0, 1.0)                       # EMA fixed point: window == committed
    got = st.commit(0.5)
    assert got == [1.0, 2.0, 3.0]           # layer 0 fixed point; 1, 2 frozen -> retained


def test_commit_errors():
    st = O.MgnState(2)
    with pytest.raises(ValueError):
        st.commit(0.5)                      # zero observations
    st.record(0, 1.0)
    with pytest.raises(ValueError):
        st.commit(1.5)                      # alpha outside [0,1]
    with pytest.raises(FloatingPointError):
        st.record(1, float("nan"))


def test_first_commit_without_probing_is_uniform():
    """SPEC.md:451 (gamma = N_L, T_p = 0): a schedule without probing commits
    its first window before any observation — m = 0, Eq. 3 gives exactly 1/N
    (closed form); a later empty commit is still the SPEC.md:252 usage error,
    and T_p > 0 keeps the error for the first commit too."""
    for normalize in (True, False):
        orc = O.GrassOracle([8, 8, 8, 8, 8], gamma=2, T_p=0, normalize=normalize)
        assert orc.update_probs() == [0.2] * 5
        with pytest.raises(ValueError):
            orc.update_probs()
    with pytest.raises(ValueError):
        O.GrassOracle([8, 8], gamma=1, T_p=1).update_probs()
    st = O.MgnState(3)
    assert st.commit(0.5, empty_first_ok=True) == [0.0, 0.0, 0.0] and st.committed


# ----------------------------------------------------------------- Eq. 3 softmax
def test_softmax_spec_examples(golden):
    for ex in golden("spec_examples.json")["softmax"]:
        p = O.softmax_probs(ex["m"], ex["tau"], ex["normalize"])
        assert p == pytest.approx(ex["p"], rel=0, abs=1e-15), ex["cite"]


def test_softmax_raw_matches_scipy():
    from scipy.special import softmax
    for seed in range(20):
        m = np.random.default_rng(seed).uniform(0, 5, 9)
        for tau in (0.1, 1.0, 7.0):
            assert O.softmax_probs(m, tau, False) == pytest.approx(softmax(m / tau).tolist(), rel=1e-13)


def test_softmax_normalized_matches_scipy_on_max_normalised_input():
    from scipy.special import softmax
    m = np.array([2e-4, 7e-4, 1e-4, 5e-4])
    assert O.softmax_probs(m, 0.5, True) == pytest.approx(softmax(m / m.max() / 0.5).tolist(), rel=1e-13)


def test_softmax_invariants():
    for seed in range(50):
        rng = np.random.default_rng(seed)
        m = rng.uniform(0, 1e-3, rng.integers(1, 41)).tolist()
        tau = float(rng.uniform(0.05, 3))
        p = O.softmax_probs(m, tau, True)
        assert abs(math.fsum(p) - 1.0) <= 1e-12
        assert min(p) > 0
        assert int(np.argmax(p)) == int(np.argmax(m))
        assert O.softmax_probs([x * 37.5 for x in m], tau, True) == pytest.approx(p, rel=1e-12)
    p = O.softmax_probs([0.0, 1.0, 2.0, 3.0], 1e9, False)
    assert max(abs(x - 0.25) for x in p) < 1e-6
    assert O.softmax_probs([0.0, 0.0, 0.0], 1.0, True) == [1 / 3] * 3     # m == 0 -> uniform
    with pytest.raises(ValueError):
        O.softmax_probs([1.0], 0.0)


# -------------------------------------------------------------------- RNG
def test_splitmix64_published_vectors(golden):
    v = golden("splitmix64_vectors.json")
    gamma = int(v["gamma"], 16)
    for k, want in enumerate(v["outputs_from_state_0"]):
        assert O.splitmix64((k * gamma) & O.MASK64) == int(want, 16)


def test_uniform_draws_published_splitmix64_outputs(golden):
    # R7: u(seed, period, k) = (splitmix64(splitmix64(seed) ^ (period*2^16 + k)) >> 11) * 2^-53.
    # With seed = 0 the key is the published output #0; choosing (period, k) so
    # that key ^ (period*2^16 + k) = j*gamma makes the draw the published
    # output #j — its top 53 bits scaled by 2^-53, exactly.
    v = golden("splitmix64_vectors.json")
    gamma = int(v["gamma"], 16)
    outs = [int(x, 16) for x in v["outputs_from_state_0"]]
    key = outs[0]
    for j, out in enumerate(outs):
        ctr = key ^ ((j * gamma) & O.MASK64)
        period, k = ctr >> 16, ctr & 0xFFFF
        assert O.uniform(0, period, k) == (out >> 11) * 2.0 ** -53


def test_uniform_range_and_moments():
    us = [O.uniform(1234, p, k) for p in range(2000) for k in range(10)]
    assert all(0.0 <= u < 1.0 for u in us)
    assert abs(np.mean(us) - 0.5) < 0.01 and abs(np.var(us) - 1 / 12) < 0.005
    assert len(set(us)) == len(us)


# -------------------------------------------------------------- sampler
def test_exact_law_matches_hand_derived_inclusion(golden):
    ex = golden("spec_examples.json")["sampler_law"]
    law = O.sampling_law_exact([Fraction(s) for s in ex["p"]], ex["gamma"])
    assert float(sum(law.values())) == 1.0
    for l in range(4):
        inc = float(sum(pr for k, pr in law.items() if l in k))
        assert inc == pytest.approx(ex["inclusion"][l], abs=1e-14)
    for key, want in ex["pairs_unordered"].items():
        i, j = int(key[0]), int(key[1])
        assert float(law[(i, j)] + law[(j, i)]) == pytest.approx(want, abs=1e-6)


def test_sampler_per_draw_law_on_u_grid():
    # Draw k depends only on u_k; sweeping u over a fine grid recovers each
    # conditional law p_j / (1 - sum of removed) to grid resolution.
    p = [0.4, 0.3, 0.2, 0.1]
    n = 20_000
    first = np.zeros(4)
    for i in range(n):
        first[O.sample_layers(p, 1, u_fn=lambda k, u=(i + 0.5) / n: u)[0]] += 1
    assert first / n == pytest.approx(p, abs=2 / n)
    second = np.zeros(4)
    for i in range(n):
        seq = O.sample_layers(p, 2, u_fn=lambda k, u=(i + 0.5) / n: 0.0 if k == 0 else u)
        assert seq[0] == 0
        second[seq[1]] += 1
    assert second / n == pytest.approx([0, 0.5, 1 / 3, 1 / 6], abs=2 / n)


def test_sampler_monte_carlo_matches_enumeration(golden):
    ex = golden("spec_examples.json")["sampler_law"]
    p = [float(s) for s in ex["p"]]
    cnt = np.zeros(4)
    N = 60_000
    for period in range(N):
        for l in O.sample_layers(p, 2, seed=1234, period=period):
            cnt[l] += 1
    assert cnt / N == pytest.approx(ex["inclusion"], abs=0.01)


def test_torch_multinomial_agrees_with_exact_law(golden):
    # library special case: torch.multinomial(replacement=False) draws the same law
    ex = golden("spec_examples.json")["sampler_law"]
    g = torch.Generator().manual_seed(0)
    p = torch.tensor([float(s) for s in ex["p"]], dtype=torch.float64)
    draws = torch.multinomial(p.expand(200_000, 4), 2, replacement=False, generator=g)
    inc = [(draws == l).any(1).double().mean().item() for l in range(4)]
    assert inc == pytest.approx(ex["inclusion"], abs=0.01)


def test_sampler_special_cases():
    rng = random.Random(0)
    for _ in range(200):
        n = rng.randint(1, 40)
        p = O.softmax_probs([rng.random() for _ in range(n)], 0.3)
        gamma = rng.randint(1, n)
        ids = O.sample_layers(p, gamma, seed=rng.getrandbits(64), period=rng.randint(0, 10**6))
        assert len(ids) == gamma == len(set(ids)) and all(0 <= i < n for i in ids)
    assert sorted(O.sample_layers([0.1, 0.2, 0.7], 3, 5, 9)) == [0, 1, 2]       # gamma = N_L
    assert O.sample_layers([0.1, 0.2, 0.7], 2, 5, 9) == O.sample_layers([0.1, 0.2, 0.7], 2, 5, 9)
    assert O.sample_layers([0.0, 0.0, 0.0], 1, 1, 1) == [2]                     # R = 0 fallback
    one_hot = [1 - 3e-12, 1e-12, 1e-12, 1e-12]
    assert all(O.sample_layers(one_hot, 1, 3, t) == [0] for t in range(500))
    with pytest.raises(ValueError):
        O.sample_layers([0.5, 0.5], 3)


# ----------------------------------------------------------------- AdamW
def test_adamw_closed_form_single_step(golden):
    for ex in golden("spec_examples.json")["adamw"]:
        th, m, v = O.adamw_step(np.float32([ex["theta"]]), np.float32([0]), np.float32([0]),
                                np.float32([ex["g"]]), 1, ex["lr"], weight_decay=ex["wd"])
        # golden is the real-arithmetic value for the decimal inputs; the fp32
        # output may differ by the fp32 rounding of theta0 and of the result.
        assert float(th[0]) == pytest.approx(ex["theta1"], rel=1.5e-7), ex["cite"]
        assert m[0] == np.float32(0.1 * ex["g"]) and v[0] == np.float32(0.001 * ex["g"] ** 2)


def test_adamw_constant_grad_closed_form_every_step():
    # constant g => m_hat = g, v_hat = g^2 => each step dtheta = -lr*g/(|g|+eps) - lr*wd*theta
    lr, wd, eps = 1e-3, 0.1, 1e-8
    g = np.float32([0.5, -2.0, 1e-3])
    th = np.float32([0.3, -0.1, 0.0])
    m = v = np.zeros(3, np.float32)
    for t in range(1, 30):
        want = th.astype(np.float64) * (1 - lr * wd) - lr * g.astype(np.float64) / (np.abs(g) + eps)
        th, m, v = O.adamw_step(th, m, v, g, t, lr, weight_decay=wd, eps=eps)
        assert th == pytest.approx(want.astype(np.float32), rel=2e-6, abs=1e-9)


def test_adamw_zero_grad_no_decay_is_identity_on_theta():
    th0 = np.float32([0.1, -0.2])
    th, m, v = O.adamw_step(th0, np.float32([0.5, 0.5]), np.float32([0.25, 0.25]),
                            np.float32([0, 0]), 3, 0.1)
    assert (m == np.float32(0.45)).all() and (v == np.float32(0.25 * 0.999)).all()
    assert not (th == th0).all()        # m != 0 still moves theta ...
    th, m, v = O.adamw_step(th0, np.zeros(2, np.float32), np.zeros(2, np.float32),
                            np.float32([0, 0]), 1, 0.1)
    assert (th == th0).all() and (m == 0).all() and (v == 0).all()   # ... g = m = 0, wd = 0 does not


def test_adamw_matches_torch_optim_adamw_fp64():
    rng = np.random.default_rng(1)
    n, lr, wd = 1000, 3e-3, 0.05
    th = (rng.standard_normal(n) * 0.02).astype(np.float32)
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    for t in range(1, 6):
        g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
        p = torch.nn.Parameter(torch.from_numpy(th.astype(np.float64)))
        opt = torch.optim.AdamW([p], lr=lr, weight_decay=wd, foreach=False)
        opt.state[p] = {"step": torch.tensor(float(t - 1), dtype=torch.float64),
                        "exp_avg": torch.from_numpy(m.astype(np.float64)),
                        "exp_avg_sq": torch.from_numpy(v.astype(np.float64))}
        p.grad = torch.from_numpy(g.astype(np.float64))
        opt.step()
        th, m, v = O.adamw_step(th, m, v, g, t, lr, weight_decay=wd)
        np.testing.assert_allclose(th, p.detach().numpy(), rtol=2e-7, atol=1e-12)
        np.testing.assert_allclose(m, opt.state[p]["exp_avg"].numpy(), rtol=2e-7, atol=1e-20)
        np.testing.assert_allclose(v, opt.state[p]["exp_avg_sq"].numpy(), rtol=2e-7, atol=1e-25)


# ----------------------------------------------------------------- schedule
def test_schedule_paper_values(golden):
    s = golden("spec_examples.json")["schedule"]
    for t in s["probe_steps"]:
        assert O.schedule_decision(t, s["T_p"], s["T_s"]) == "probe"
    for t in s["resample_steps"]:
        assert "resample" in O.schedule_decision(t, s["T_p"], s["T_s"])
    for t in s["continue_steps"]:
        assert O.schedule_decision(t, s["T_p"], s["T_s"]) == "continue"
    assert O.schedule_decision(200, 150, 25, 50) == "commit+resample"
    assert O.schedule_decision(175, 150, 25, 50) == "resample"


# ------------------------------------------------------- whole-path degeneracy
def test_gamma_equals_NL_degenerates_to_plain_adamw():
    # gamma = N_L updates every layer every step: identical to
    # torch.optim.AdamW over all layers (fp64 library reference).
    rng = np.random.default_rng(5)
    numel = [17, 64, 5]
    lr, wd = 1e-2, 0.01
    orc = O.GrassOracle(numel, gamma=3, weight_decay=wd, seed=9)
    params = [(rng.standard_normal(k) * 0.02).astype(np.float32) for k in numel]
    tparams = [torch.nn.Parameter(torch.from_numpy(p.astype(np.float64))) for p in params]
    opt = torch.optim.AdamW(tparams, lr=lr, weight_decay=wd, foreach=False)
    for step in range(4):
        grads = [(rng.standard_normal(k) * 1e-2).astype(np.float32) for k in numel]
        if step == 0:
            orc.accumulate([0, 1, 2], grads)
            orc.update_probs()
        ids = orc.sample(step)
        assert sorted(ids) == [0, 1, 2]
        orc.step_layers(ids, [params[i] for i in ids], [grads[i] for i in ids], lr)
        for tp, g in zip(tparams, grads):
            tp.grad = torch.from_numpy(g.astype(np.float64))
        opt.step()
        for p, tp in zip(params, tparams):
            np.testing.assert_allclose(p, tp.detach().numpy(), rtol=1e-6, atol=1e-9)
    assert orc.t == [4, 4, 4]


# ----------------------------------------------- R19: always-active groups
def test_always_groups_gamma_equals_NL_is_plain_adamw_over_everything():
    # SPEC.md:145 (embedding / head always trainable, excluded from sampling):
    # with gamma = N_L sampled layers plus the always groups listed every step,
    # every tensor follows torch.optim.AdamW (fp64) -- the always groups too.
    rng = np.random.default_rng(6)
    numel = [17, 64, 5, 40, 9]          # 3 sampled layers + 2 always groups
    lr, wd = 1e-2, 0.01
    orc = O.GrassOracle(numel, gamma=3, weight_decay=wd, seed=9, n_always=2)
    params = [(rng.standard_normal(k) * 0.02).astype(np.float32) for k in numel]
    tparams = [torch.nn.Parameter(torch.from_numpy(p.astype(np.float64))) for p in params]
    opt = torch.optim.AdamW(tparams, lr=lr, weight_decay=wd, foreach=False)
    for step in range(4):
        grads = [(rng.standard_normal(k) * 1e-2).astype(np.float32) for k in numel]
        if step == 0:
            orc.accumulate([0, 1, 2], grads[:3])
            p = orc.update_probs()
            assert len(p) == 5 and p[3:] == [0.0, 0.0] and abs(sum(p) - 1.0) < 1e-12
        ids = orc.sample(step)
        assert sorted(ids) == [0, 1, 2]
        ids = ids + [3, 4]
        orc.step_layers(ids, [params[i] for i in ids], [grads[i] for i in ids], lr)
        for tp, g in zip(tparams, grads):
            tp.grad = torch.from_numpy(g.astype(np.float64))
        opt.step()
        for p_, tp in zip(params, tparams):
            np.testing.assert_allclose(p_, tp.detach().numpy(), rtol=1e-6, atol=1e-9)
    assert orc.t == [4] * 5


def test_always_groups_do_not_touch_mgn_or_sampling():
    # The MGN window, Eq. 3 probabilities and the sampler of a run with always
    # groups equal those of the same run without them (they are invisible to
    # PAPER.md:89-127); the sampler never returns an always id.
    rng = np.random.default_rng(7)
    numel = [33, 10, 50, 21]
    a = O.GrassOracle(numel, gamma=2, seed=3)
    b = O.GrassOracle(numel + [64, 8], gamma=2, seed=3, n_always=2)
    for _ in range(3):
        grads = [(rng.standard_normal(k) * rng.uniform(1e-3, 1)).astype(np.float32) for k in numel + [64, 8]]
        a.accumulate([0, 1, 2, 3], grads[:4])
        b.accumulate([0, 1, 2, 3, 4, 5], grads)
    pa, pb = a.update_probs(), b.update_probs()
    assert pb[:4] == pa and pb[4:] == [0.0, 0.0]
    assert b.last_ss[4] == O.sq_norm(grads[4])
    for period in range(200):
        ids = b.sample(period)
        assert ids == a.sample(period) and max(ids) < 4
    # degenerate sampled probabilities (all zero): the R = 0 fallback takes the
    # last SAMPLED layer, never an always group
    assert b.sample(0, probs=[0.0] * 6) == [3, 2]


# ------------------------------------------------ R17: global-norm clipping
def test_clip_coefficient_matches_torch_clip_grad_norm():
    rng = np.random.default_rng(11)
    for max_norm in (1e-3, 0.05, 1.0, 1e3):
        gs = [rng.standard_normal(k).astype(np.float32) * 0.01 for k in (17, 300, 5)]
        ps = [torch.nn.Parameter(torch.zeros(len(g), dtype=torch.float64)) for g in gs]
        for p, g in zip(ps, gs):
            p.grad = torch.from_numpy(g.astype(np.float64))
        total = torch.nn.utils.clip_grad_norm_(ps, max_norm)
        coef = O.clip_coefficient([O.sq_norm(g) for g in gs], max_norm)
        assert math.sqrt(sum(O.sq_norm(g) for g in gs)) == pytest.approx(float(total), rel=1e-14)
        for p, g in zip(ps, gs):
            np.testing.assert_allclose(p.grad.numpy(), g.astype(np.float64) * coef, rtol=1e-14)
        assert coef <= 1.0 and (coef == 1.0) == (max_norm >= float(total) + 1e-6)


def test_clipped_step_is_torch_clip_then_adamw_and_mgn_sees_raw_norm():
    # R17 + R9: GrassOracle.step_layers(max_grad_norm) == torch clip_grad_norm_ over the
    # call's gradients followed by torch.optim.AdamW (fp64); the MGN window records
    # the RAW (unclipped) norms.
    rng = np.random.default_rng(12)
    numel = [33, 100, 7, 64]
    ids = [3, 1]
    lr, wd, max_norm = 1e-2, 0.01, 0.05
    orc = O.GrassOracle(numel, gamma=2, weight_decay=wd)
    params = [(rng.standard_normal(k) * 0.02).astype(np.float32) for k in numel]
    tp = {l: torch.nn.Parameter(torch.from_numpy(params[l].astype(np.float64))) for l in ids}
    opt = torch.optim.AdamW([tp[l] for l in ids], lr=lr, weight_decay=wd, foreach=False)
    for step in range(3):
        grads = {l: (rng.standard_normal(numel[l]) * 0.05).astype(np.float32) for l in ids}
        orc.step_layers(ids, [params[l] for l in ids], [grads[l] for l in ids], lr, max_grad_norm=max_norm)
        for l in ids:
            tp[l].grad = torch.from_numpy(grads[l].astype(np.float64))
        torch.nn.utils.clip_grad_norm_([tp[l] for l in ids], max_norm)
        opt.step()
        for l in ids:
            np.testing.assert_allclose(params[l], tp[l].detach().numpy(), rtol=1e-6, atol=1e-9)
            assert orc.last_ss[l] == O.sq_norm(grads[l])                     # raw norm
    for l in ids:
        assert orc.mgn.c[l] == 3
    assert orc.mgn.c[0] == orc.mgn.c[2] == 0


# ------------------------------------------------ R18: bf16 mixed precision
def test_bf16_conversions_match_torch():
    rng = np.random.default_rng(4)
    x = np.concatenate([rng.standard_normal(100_000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 100_000),
                        np.float32([0.0, -0.0, np.inf, -np.inf, 1.0, 1.00390625, 1.01171875, 3.4e38])])
    x = x.astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(O.f32_to_bf16(x), want)               # round to nearest even
    back = torch.from_numpy(want.view(np.int16)).view(torch.bfloat16).float().numpy()
    assert np.array_equal(O.bf16_to_f32(want), back)            # exact widening
    assert np.isnan(O.bf16_to_f32(O.f32_to_bf16(np.float32([np.nan])))).all()


def test_adamw_bf16_matches_torch_adamw_on_fp32_master():
    # mixed precision = torch AdamW on an fp32 master fed with the widened
    # bf16 gradient, the bf16 model copy re-rounded from the master each step
    rng = np.random.default_rng(6)
    n, lr, wd = 4000, 1e-3, 0.01
    p_bits = O.f32_to_bf16((rng.standard_normal(n) * 0.02).astype(np.float32))
    master = torch.nn.Parameter(torch.from_numpy(O.bf16_to_f32(p_bits).astype(np.float64)))
    opt = torch.optim.AdamW([master], lr=lr, weight_decay=wd, foreach=False)
    m = v = np.zeros(n, np.float32)
    mw = None
    for t in range(1, 5):
        g_bits = O.f32_to_bf16((rng.standard_normal(n) * 1e-3).astype(np.float32))
        master.grad = torch.from_numpy(O.bf16_to_f32(g_bits).astype(np.float64))
        opt.step()
        mw, m, v, th_bits = O.adamw_step_bf16(mw, m, v, g_bits, t, lr, weight_decay=wd,
                                              theta_bits=p_bits if t == 1 else None)
        # torch keeps an fp64 master, the oracle rounds it to fp32 each step:
        # differences stay at the fp32 ulp of theta (~2e-9)
        np.testing.assert_allclose(mw, master.detach().numpy(), rtol=3e-7, atol=1e-9)
        assert np.array_equal(th_bits, O.f32_to_bf16(mw))
