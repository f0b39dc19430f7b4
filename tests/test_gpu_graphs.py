"""CUDA graphs: grass_step_layers captured once (torch.cuda.graph) and replayed
k times must equal k eager calls bit for bit — parameters, m, v, the device
step counts t_l, the bf16 master initialisation on the first replay, the
clipped update and the MGN window — and the learning rate can come from a
device scalar changed between replays (grass_set_lr_device)."""
import numpy as np
import pytest
import torch

import paper_2604_07808_b200 as G
from synth import layer_grad, layer_params

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _pair(numel, dtype, **kw):
    tdt = torch.bfloat16 if dtype == G.DTYPE_BF16 else torch.float32
    eager = G.Grass(numel, gamma=2, weight_decay=0.01, param_dtype=dtype, **kw)
    graph = G.Grass(numel, gamma=2, weight_decay=0.01, param_dtype=dtype, **kw)
    base = [layer_params(n, l, device=DEV).to(tdt) for l, n in enumerate(numel)]
    grads = [layer_grad(n, l, 1e-3, device=DEV).to(tdt) for l, n in enumerate(numel)]
    return eager, graph, [b.clone() for b in base], [b.clone() for b in base], grads


def _same(eager, graph, pe, pg, ids):
    torch.cuda.synchronize()
    for l in ids:
        assert torch.equal(pe[l], pg[l]), l
        a, b = eager.read_state(l), graph.read_state(l)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2], l
    sa, sb = eager.get_mgn(), graph.get_mgn()
    assert sa["S"] == sb["S"] and sa["c"] == sb["c"] and sa["last_ss"] == sb["last_ss"]


@pytest.mark.parametrize("dtype", [G.DTYPE_FP32, G.DTYPE_BF16])
@pytest.mark.parametrize("clip", [0.0, 1e-3])
def test_captured_step_replays_equal_eager_steps(dtype, clip):
    numel = [4096 * 5 + 8, 65_536, 4096 * 3]
    ids = [2, 0]
    eager, graph, pe, pg, grads = _pair(numel, dtype, max_grad_norm=clip)
    k = 5
    for _ in range(k):
        eager.step_layers(ids, [pe[l] for l in ids], [grads[l] for l in ids], 1e-3)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graph.step_layers(ids, [pg[l] for l in ids], [grads[l] for l in ids], 1e-3,
                          stream=torch.cuda.current_stream())
    for _ in range(k):
        g.replay()
    _same(eager, graph, pe, pg, ids)
    assert graph.read_state(0)[2] == k                     # t advanced on every replay
    if dtype == G.DTYPE_BF16:
        assert np.array_equal(eager.read_master(0), graph.read_master(0))


def test_captured_step_with_device_learning_rate():
    numel = [8192, 4096 * 3 + 4]
    ids = [0, 1]
    eager, graph, pe, pg, grads = _pair(numel, G.DTYPE_FP32)
    lrs = [1e-3, 5e-4, 2e-3, 1e-4]
    lr_t = torch.zeros((), dtype=torch.float32, device=DEV)
    graph.set_lr_device(lr_t)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graph.step_layers(ids, pg, grads, 123.0, stream=torch.cuda.current_stream())  # lr argument ignored
    for lr in lrs:
        eager.step_layers(ids, pe, grads, lr)
        lr_t.fill_(lr)
        g.replay()
    _same(eager, graph, pe, pg, ids)
    graph.set_lr_device(None)


def test_commit_after_replays_sees_every_replay():
    numel = [8192, 8192, 8192]
    gr = G.Grass(numel, gamma=2, T_p=1, T_s=1)
    p = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    g = [layer_grad(n, l, 1e-3, device=DEV) for l, n in enumerate(numel)]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        gr.step_layers([0, 2], [p[0], p[2]], [g[0], g[2]], 1e-3, stream=torch.cuda.current_stream())
    for _ in range(7):
        graph.replay()
    st = gr.get_mgn()                                     # no explicit synchronisation before
    assert st["c"] == [7, 0, 7]
    probs = gr.update_probs()
    assert abs(sum(probs) - 1.0) < 1e-12 and gr.get_mgn()["c"] == [0, 0, 0]   # window consumed


def test_capture_rejected_where_unsupported():
    numel = [8192, 8192]
    p = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    g = [layer_grad(n, l, 1e-3, device=DEV) for l, n in enumerate(numel)]
    off = G.Grass(numel, gamma=2, offload=True, residency=G.RESIDENCY_STEP_PREFETCH)  # fetches every step
    graph = torch.cuda.CUDAGraph()
    with pytest.raises(G.GrassError, match="capture"), pytest.warns(UserWarning):
        with torch.cuda.graph(graph):
            off.step_layers([0, 1], p, g, 1e-3, stream=torch.cuda.current_stream())


def test_captured_p2p_step_replays_equal_eager_steps():
    """The fused P2P data-parallel step (world 1, device barriers whose
    generations advance on the device) captured and replayed == eager."""
    numel = [4096 * 3 + 8, 65_536]
    ids = [1, 0]
    ctxs, P = [], []
    grads = [layer_grad(n, l, 1e-3, device=DEV) for l, n in enumerate(numel)]
    base = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    for _ in range(2):
        c = G.Grass(numel, gamma=2, weight_decay=0.01, dp_mode=G.DP_P2P)
        c.p2p_attach([c.p2p_exchange_block()[0]])
        p = [b.clone() for b in base]
        for l in range(2):
            c.p2p_register_layer(l, [p[l]], [grads[l]])
        ctxs.append(c)
        P.append(p)
    eager, graph = ctxs
    for _ in range(4):
        eager.step_layers(ids, [P[0][l] for l in ids], [grads[l] for l in ids], 1e-3)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graph.step_layers(ids, [P[1][l] for l in ids], [grads[l] for l in ids], 1e-3,
                          stream=torch.cuda.current_stream())
    for _ in range(4):
        g.replay()
    _same(eager, graph, P[0], P[1], ids)


def test_captured_nccl_step_replays_equal_eager_steps():
    """The NCCL data-parallel step (1-rank communicator: reduce-scatter, K2,
    all-gather on the comm stream, fp64 partial all-gather) captured == eager."""
    numel = [4096 * 4, 8192 + 64]
    ids = [0, 1]
    eager, graph, pe, pg, grads = _pair(numel, G.DTYPE_FP32, force_nccl=True)
    for _ in range(3):
        eager.step_layers(ids, pe, grads, 1e-3)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graph.step_layers(ids, pg, grads, 1e-3, stream=torch.cuda.current_stream())
    for _ in range(3):
        g.replay()
    _same(eager, graph, pe, pg, ids)


def test_captured_schedule_period_with_always_group_and_commit():
    """A whole sampling period captured once: the trainable set plus an
    always-active group, replayed T_s times, then a commit — equal to the
    same period run eagerly (MGN, probabilities, states)."""
    numel = [8192] * 4 + [4096 * 3]
    T_s = 5
    ctxs, P = [], []
    base = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    grads = [layer_grad(n, l, 10.0 ** (-3 - (l % 3)), device=DEV) for l, n in enumerate(numel)]
    for _ in range(2):
        c = G.Grass(numel, gamma=2, T_p=1, T_s=T_s, n_always=1, seed=4, weight_decay=0.01)
        c.mgn_accumulate([0, 1, 2, 3], grads[:4])
        c.update_probs()
        ctxs.append(c)
        P.append([b.clone() for b in base])
    eager, graph = ctxs
    ids = eager.sample_layers(0)
    assert ids == graph.sample_layers(0)
    layers = ids + [4]
    for _ in range(T_s):
        eager.step_layers(layers, [P[0][l] for l in layers], [grads[l] for l in layers], 1e-3)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graph.step_layers(layers, [P[1][l] for l in layers], [grads[l] for l in layers], 1e-3,
                          stream=torch.cuda.current_stream())
    for _ in range(T_s):
        g.replay()
    assert eager.update_probs() == graph.update_probs()
    _same(eager, graph, P[0], P[1], layers)
    assert eager.sample_layers(1) == graph.sample_layers(1)


@pytest.mark.parametrize("dtype", [G.DTYPE_FP32, G.DTYPE_BF16])
@pytest.mark.parametrize("overlap", [True, False])
def test_captured_offloaded_step_replays_equal_eager_steps(dtype, overlap):
    """The per-step offload pipeline (fetch -> update -> write-back through the
    chunk ring, copy streams forked into the capture) captured once and
    replayed == eager steps; eager steps after the replays stay identical."""
    numel = [4096 * 9 + 8, 65_536, 4096 * 3]
    ids = [0, 1]
    eager, graph, pe, pg, grads = _pair(numel, dtype, offload=True, overlap=overlap, chunk_elems=8192,
                                        ring_slots=2)
    k = 4
    for _ in range(k):
        eager.step_layers(ids, [pe[l] for l in ids], [grads[l] for l in ids], 1e-3)
    graph.sync()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graph.step_layers(ids, [pg[l] for l in ids], [grads[l] for l in ids], 1e-3,
                          stream=torch.cuda.current_stream())
    for _ in range(k):
        g.replay()
    _same(eager, graph, pe, pg, ids)
    for c, p in ((eager, pe), (graph, pg)):                # eager after replays
        c.step_layers([2, 0], [p[2], p[0]], [grads[2], grads[0]], 1e-3)
    _same(eager, graph, pe, pg, [0, 1, 2])


@pytest.mark.parametrize("residency", ["step", "period"])
def test_offloaded_replays_interleaved_with_eager_steps(residency):
    """capture -> replay -> eager -> replay -> eager -> ... with no host sync in
    between: every eager offloaded call after a capture orders its
    copy streams after the replays already on the caller stream, so no fetch
    overwrites a ring slot a replay still reads and no write-back reads state
    a replay still writes.  Layers of 8 Mi elements (32 MiB per state array)
    keep each replay's copies in flight long enough for a missing fence to
    show; the result must equal the same sequence of eager steps bit for bit."""
    numel = [8 << 20, 8 << 20, 4096 * 3]
    ids = [0, 1]
    kw = dict(offload=True, chunk_elems=1 << 20, ring_slots=2)
    if residency == "period":
        kw.update(residency=G.RESIDENCY_PERIOD, cache_layers=3)
    eager, graph, pe, pg, grads = _pair(numel, G.DTYPE_FP32, **kw)
    if residency == "period":
        for c in (eager, graph):
            c.prefetch_layers(ids)
    graph.sync()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graph.step_layers(ids, [pg[l] for l in ids], [grads[l] for l in ids], 1e-3,
                          stream=torch.cuda.current_stream())
    other = [1, 2] if residency == "step" else [0, 1]   # period: stay within the cached set
    for _ in range(4):
        g.replay()
        eager.step_layers(ids, [pe[l] for l in ids], [grads[l] for l in ids], 1e-3)
        for c, p in ((eager, pe), (graph, pg)):
            c.step_layers(other, [p[l] for l in other], [grads[l] for l in other], 1e-3)
    _same(eager, graph, pe, pg, [0, 1, 2])


def test_captured_nccl_offloaded_step_replays_equal_eager_steps():
    """NCCL data parallelism (1-rank communicator) with per-step offload,
    captured and replayed == eager."""
    numel = [4096 * 6, 8192 + 64]
    ids = [1, 0]
    eager, graph, pe, pg, grads = _pair(numel, G.DTYPE_FP32, force_nccl=True, offload=True, chunk_elems=8192)
    for _ in range(3):
        eager.step_layers(ids, [pe[l] for l in ids], [grads[l] for l in ids], 1e-3)
    graph.sync()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graph.step_layers(ids, [pg[l] for l in ids], [grads[l] for l in ids], 1e-3,
                          stream=torch.cuda.current_stream())
    for _ in range(3):
        g.replay()
    _same(eager, graph, pe, pg, ids)


def test_captured_period_resident_step_replays_equal_eager_steps():
    """Period residency: once the period's layers are cached (prefetched, then
    grass_sync), a captured step is updates in HBM slots only; replays ==
    eager; a step with an uncached layer cannot be captured."""
    numel = [8192 * 3, 8192, 4096 * 5 + 8]
    ids = [2, 0]
    eager, graph, pe, pg, grads = _pair(numel, G.DTYPE_FP32, offload=True, residency=G.RESIDENCY_PERIOD)
    for c in (eager, graph):
        c.prefetch_layers(ids)
    graph.sync()
    with pytest.raises(G.GrassError, match="not cached"), pytest.warns(UserWarning):
        with torch.cuda.graph(torch.cuda.CUDAGraph()):
            graph.step_layers([1], [pg[1]], [grads[1]], 1e-3, stream=torch.cuda.current_stream())
    for _ in range(4):
        eager.step_layers(ids, [pe[l] for l in ids], [grads[l] for l in ids], 1e-3)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graph.step_layers(ids, [pg[l] for l in ids], [grads[l] for l in ids], 1e-3,
                          stream=torch.cuda.current_stream())
    for _ in range(4):
        g.replay()
    _same(eager, graph, pe, pg, ids)
    eager.flush_states()
    graph.flush_states()
    _same(eager, graph, pe, pg, ids)


@pytest.mark.parametrize("mode", ["resident", "offload", "period"])
def test_schedule_graph_mode_equals_eager_schedule(mode):
    """GrassSchedule(graphs=True): one captured update per sampling period,
    replayed on its other steps with eta from a device scalar (a changing
    schedule) — identical to the eager schedule."""
    numel = [8192] * 4 + [4096 * 3]
    kw = {"resident": {}, "offload": dict(offload=True, chunk_elems=8192),
          "period": dict(offload=True, residency=G.RESIDENCY_PERIOD)}[mode]
    T_p, T_s = 2, 3
    runs = []
    for graphs in (False, True):
        gr = G.Grass(numel, gamma=2, T_p=T_p, T_s=T_s, seed=9, n_always=1, weight_decay=0.01, **kw)
        sched = G.GrassSchedule(gr, graphs=graphs)
        P = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
        Gb = [torch.zeros(n, device=DEV) for n in numel]          # persistent gradient buffers
        for step in range(T_p + 3 * T_s):
            layers = sched.begin_step(step)
            for l in layers:
                Gb[l].copy_(layer_grad(numel[l], l, 10.0 ** (-3 - l % 2), step=step, device=DEV))
            sched.end_step(step, [P[l] for l in layers], [Gb[l] for l in layers], 1e-3 * (1 + 0.1 * step))
        gr.sync()
        runs.append((gr, P))
    (ea, pa), (eb, pb) = runs
    _same(ea, eb, pa, pb, list(range(5)))
    assert ea.get_mgn()["m"] == eb.get_mgn()["m"]
