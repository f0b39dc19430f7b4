"""The device-resident schedule (grass_register_layers /
grass_device_schedule_begin / grass_device_step / grass_device_schedule_end):
the adaptive step with the sampled ids, m, p and the MGN window kept in device
memory (no host round trip between steps) must reproduce the host-driven
schedule (grass_step_layers + grass_update_probs + grass_sample_layers) —
parameters, m, v, t_l, the bf16 master, S / c, m and p — for fp32 / bf16,
with always-active groups, on the every-step schedule and the paper's
T_s / T_u one; a captured step replayed k times equals k eager steps; misuse
is rejected.  The host path is itself checked against the oracle elsewhere
(tests/test_gpu_parity.py), so equality here carries that parity over."""
import numpy as np
import pytest
import torch

import paper_2604_07808_b200 as G
from oracle import grass_oracle as O
from synth import grad_sigmas, layer_grad, layer_params

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _setup(dtype, n_always, T_s, T_u, numel=None, **kw):
    tdt = torch.bfloat16 if dtype == G.DTYPE_BF16 else torch.float32
    numel = numel or [4096 * 5 + 8, 65_536, 4096 * 3, 4096 * 7 + 16, 8192] + [4096 * 2 + 4] * n_always
    nl = len(numel)
    sig = grad_sigmas(nl, 3)
    mk = lambda: G.Grass(numel, gamma=2, T_p=2, T_s=T_s, T_u=T_u, seed=77, weight_decay=0.01, param_dtype=dtype,
                         n_always=n_always, **kw)
    host, dev = mk(), mk()
    base = [layer_params(n, l, device=DEV).to(tdt) for l, n in enumerate(numel)]
    P = [[b.clone() for b in base] for _ in range(2)]
    Gr = [torch.zeros(n, device=DEV, dtype=tdt) for n in numel]     # the registered gradient buffers
    return host, dev, P, Gr, numel, sig, tdt


def _fill(Gr, numel, sig, step, tdt):
    for l, n in enumerate(numel):
        Gr[l].copy_(layer_grad(n, l, sig[l], step=step, device=DEV).to(tdt))


def _same(host, dev, P, numel):
    torch.cuda.synchronize()
    for l in range(len(numel)):
        assert torch.equal(P[0][l], P[1][l]), l
        a, b = host.read_state(l), dev.read_state(l)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2], l
        if host.bf16:
            assert np.array_equal(host.read_master(l), dev.read_master(l)), l
    sa, sb = host.get_mgn(), dev.get_mgn()
    assert sa["S"] == sb["S"] and sa["c"] == sb["c"] and sa["last_ss"] == sb["last_ss"]
    np.testing.assert_allclose(sb["m"], sa["m"], rtol=1e-15, atol=0)
    np.testing.assert_allclose(sb["probs"], sa["probs"], rtol=1e-14, atol=0)


@pytest.mark.parametrize("dtype", [G.DTYPE_FP32, G.DTYPE_BF16])
@pytest.mark.parametrize("T_s,T_u,n_always,alpha", [(1, 1, 0, 0.3), (3, 6, 1, 0.5), (2, 2, 2, 0.8)])
def test_device_schedule_equals_host_schedule(dtype, T_s, T_u, n_always, alpha):
    # alpha != 1/2 in two cases: Eq. 4's two weights are told apart
    host, dev, P, Gr, numel, sig, tdt = _setup(dtype, n_always, T_s, T_u, alpha=alpha)
    nl, ns = len(numel), len(numel) - n_always
    always = list(range(ns, nl))
    T_p, steps, lr = 2, 20, 1e-3
    dev.register_layers(P[1], Gr)
    ids_h = None
    ids_seq = []
    for step in range(steps):
        _fill(Gr, numel, sig, step, tdt)
        d = G.schedule_decision(step, T_p, T_s, T_u)
        if d == G.DECIDE_PROBE:                       # probing: both contexts through the host API
            for c in (host, dev):
                c.mgn_accumulate(list(range(ns)), Gr[:ns])
            continue
        if step == T_p:                               # first adaptive step: commit, then both schedules start
            host.update_probs()
            ids_h = host.sample_layers(0)
            dev.update_probs()
            dev.device_schedule_begin(0)
            period = 0
        layers = ids_h + always
        host.step_layers(layers, [P[0][l] for l in layers], [Gr[l] for l in layers], lr)
        nxt = G.schedule_decision(step + 1, T_p, T_s, T_u)
        commit = nxt == G.DECIDE_COMMIT_RESAMPLE
        resample = nxt in (G.DECIDE_COMMIT_RESAMPLE, G.DECIDE_RESAMPLE)
        dev.device_step(lr, commit=commit, resample=resample)
        if commit:
            host.update_probs()
        if resample:
            period += 1
            ids_h = host.sample_layers(period)
        ids_seq.append(list(ids_h))
        torch.cuda.synchronize()                      # the host step's gradients stay in place until
    ids_d = dev.device_schedule_end()                 # the device step has consumed them
    assert ids_d == ids_h
    assert len({tuple(x) for x in ids_seq}) > 1       # the schedule did resample
    _same(host, dev, P, numel)


@pytest.mark.parametrize("policy", [G.POLICY_STATIC, G.POLICY_UNIFORM])
@pytest.mark.parametrize("normalize", [True, False])
def test_device_schedule_policies_equal_host(policy, normalize):
    """GRASS* (probabilities frozen after the first commit)
    and LISA-uniform, with and without the MGN normalisation of
    Eq. 3: the device commit takes the same branch as grass_update_probs —
    parameters, m, p and the sampled ids equal the host schedule's."""
    host, dev, P, Gr, numel, sig, tdt = _setup(G.DTYPE_FP32, 0, 1, 1, policy=policy, normalize_mgn=normalize,
                                               alpha=0.3)
    nl = len(numel)
    dev.register_layers(P[1], Gr)
    for c in (host, dev):
        _fill(Gr, numel, sig, 0, tdt)
        c.mgn_accumulate(list(range(nl)), Gr)
        c.update_probs()
    ids = host.sample_layers(0)
    dev.device_schedule_begin(0)
    for step in range(1, 8):
        _fill(Gr, numel, sig, step, tdt)
        host.step_layers(ids, [P[0][l] for l in ids], [Gr[l] for l in ids], 1e-3)
        dev.device_step(1e-3)
        host.update_probs()
        ids = host.sample_layers(step)
        torch.cuda.synchronize()
    assert dev.device_schedule_end() == ids
    _same(host, dev, P, numel)
    if policy == G.POLICY_UNIFORM:
        np.testing.assert_array_equal(dev.get_mgn()["probs"], np.full(nl, 1.0 / nl))


def test_device_schedule_commit_and_sampler_against_oracle():
    """The device commit + sampler against the ORACLE directly (not only the
    host path): probe all layers, start the device schedule (ids of period 0
    from the uniform start), one device step with commit + resample — the
    device's probabilities equal the oracle's committed window (probe + the
    update's norms) within the norm tolerance, and its ids are the oracle
    sampler's on those probabilities, bit for bit."""
    numel = [8192, 4096 * 3, 65_536, 4096]
    gr = G.Grass(numel, gamma=2, T_p=1, T_s=1, seed=5)
    orc = O.GrassOracle(numel, gamma=2, seed=5)
    g = [layer_grad(n, l, 10.0 ** (-3 - l % 2), device=DEV) for l, n in enumerate(numel)]
    g_np = [x.cpu().numpy() for x in g]
    p = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    gr.register_layers(p, g)
    gr.mgn_accumulate([0, 1, 2, 3], g)
    orc.accumulate([0, 1, 2, 3], g_np)
    gr.device_schedule_begin(0)
    ids0 = O.sample_layers([0.25] * 4, 2, 5, 0)
    gr.device_step(1e-3, commit=True, resample=True, next_period=9)
    ids = gr.device_schedule_end()
    orc.accumulate(ids0, [g_np[l] for l in ids0])    # the update's norms entered the window
    p_o = orc.update_probs()
    p_d = gr.get_mgn()["probs"]
    np.testing.assert_allclose(p_d, p_o, rtol=1e-5, atol=0)
    assert ids == O.sample_layers(p_d, 2, 5, 9)
    assert gr.read_state(ids0[0])[2] == 1 and gr.read_state(ids0[1])[2] == 1     # the period-0 ids were updated


def test_captured_device_step_replays_equal_eager_steps():
    """One device step (update + commit + resample of the NEXT period, kept on
    the device) captured once and replayed k times == k eager device steps —
    the whole adaptive step as one CUDA graph."""
    host, dev, P, Gr, numel, sig, tdt = _setup(G.DTYPE_FP32, 1, 1, 1)
    eager = dev
    ns = len(numel) - 1
    for c in (host, eager):
        _fill(Gr, numel, sig, 0, tdt)
        c.mgn_accumulate(list(range(ns)), Gr[:ns])
        c.update_probs()
    host.register_layers(P[0], Gr)
    eager.register_layers(P[1], Gr)
    k = 6
    _fill(Gr, numel, sig, 1, tdt)
    for c in (host, eager):
        c.device_schedule_begin(0)
    for _ in range(k):
        eager.device_step(1e-3)
    host.sync()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        host.device_step(1e-3, stream=torch.cuda.current_stream())
    for _ in range(k):
        g.replay()
    assert host.device_schedule_end() == eager.device_schedule_end()
    _same(host, eager, P, numel)


@pytest.mark.parametrize("dtype", [G.DTYPE_FP32, G.DTYPE_BF16])
def test_device_schedule_full_size_layers_equal_host(dtype):
    """At the bench's layer size (a LLaMA-2-7B block, 202,383,360 parameters —
    49,410 tiles, K2 at its 128-CTA launch configuration) over 4 layers, the
    device schedule equals the host one bit for bit after 3 steps with commit
    + resample, and its sampled norm equals the oracle's fp64 norm of the
    same gradient (1e-6)."""
    from synth import MODELS
    n = MODELS["llama2-7b"].layer_numel
    numel = [n] * 4
    tdt = torch.bfloat16 if dtype == G.DTYPE_BF16 else torch.float32
    host = G.Grass(numel, gamma=2, T_p=1, T_s=1, seed=11, param_dtype=dtype)
    dev = G.Grass(numel, gamma=2, T_p=1, T_s=1, seed=11, param_dtype=dtype)
    sig = grad_sigmas(4, 2)
    Gr = [layer_grad(n, l, sig[l], step=0, device=DEV).to(tdt) for l in range(4)]
    Ph = [layer_params(n, l, device=DEV).to(tdt) for l in range(4)]
    Pd = [p.clone() for p in Ph]
    for c in (host, dev):
        c.mgn_accumulate([0, 1, 2, 3], Gr)
        c.update_probs()
    dev.register_layers(Pd, Gr)
    dev.device_schedule_begin(0)
    ids = host.sample_layers(0)
    for k in range(3):
        dev.device_step(3e-5)
        host.step_layers(ids, [Ph[l] for l in ids], [Gr[l] for l in ids], 3e-5)
        host.update_probs()
        ids = host.sample_layers(k + 1)
    assert dev.device_schedule_end() == ids
    torch.cuda.synchronize()
    for l in range(4):
        assert torch.equal(Ph[l], Pd[l]), l
    sa, sb = host.get_mgn(), dev.get_mgn()
    assert sa["last_ss"] == sb["last_ss"] and sa["S"] == sb["S"]
    np.testing.assert_allclose(sb["probs"], sa["probs"], rtol=1e-14, atol=0)   # device exp vs libm exp
    l = ids[0]
    ss = O.sq_norm(Gr[l].float().cpu().numpy().astype(np.float64))
    assert abs(sb["last_ss"][l] - ss) <= 1e-6 * ss


def test_device_schedule_nonfinite_gradient_stops_commits_and_is_reported():
    """A non-finite gradient in a device step: its norm is not
    recorded, the step's commit is skipped and the schedule stops committing,
    and grass_device_schedule_end reports GRASS_E_NONFINITE with the layer —
    m and p stay those of the last good commit."""
    numel = [8192, 4096 * 3, 8192, 4096]
    gr = G.Grass(numel, gamma=2, T_p=1, T_s=1, seed=5)
    g = [layer_grad(n, l, 1e-3, device=DEV) for l, n in enumerate(numel)]
    p = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    gr.register_layers(p, g)
    gr.mgn_accumulate([0, 1, 2, 3], g)
    gr.update_probs()
    before = gr.get_mgn()
    gr.device_schedule_begin(0)
    for x in g:                                        # whichever layers were sampled
        x[3] = float("nan")
    gr.device_step(1e-3)
    gr.device_step(1e-3)                               # a later commit is not taken either
    with pytest.raises(G.GrassError) as e:
        gr.device_schedule_end()
    assert e.value.status == G.binding.E_NONFINITE and "layer" in str(e.value)
    after = gr.get_mgn()
    np.testing.assert_array_equal(after["m"], before["m"])
    np.testing.assert_array_equal(after["probs"], before["probs"])


def test_device_schedule_misuse_rejected():
    numel = [8192, 8192, 4096]
    off = G.Grass(numel, gamma=2, offload=True)
    p = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    g = [layer_grad(n, l, 1e-3, device=DEV) for l, n in enumerate(numel)]
    with pytest.raises(G.GrassError, match="resident"):
        off.register_layers(p, g)
    gr = G.Grass(numel, gamma=2, T_p=0)
    with pytest.raises(G.GrassError, match="register"):
        gr.device_schedule_begin(0)
    with pytest.raises(G.GrassError, match="begin"):
        gr.device_step(1e-3)
    gr.register_layers(p, g)
    gr.device_schedule_begin(0)
    with pytest.raises(G.GrassError, match="device schedule"):
        gr.step_layers([0], [p[0]], [g[0]], 1e-3)
    with pytest.raises(G.GrassError, match="device schedule"):
        gr.update_probs()
    gr.device_step(1e-3)
    gr.device_schedule_end()
    with pytest.raises(G.GrassError):
        G.Grass(numel, gamma=2, max_grad_norm=1.0).register_layers(p, g)
