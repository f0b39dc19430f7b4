"""P2P data parallelism (cfg.dp_mode = GRASS_DP_P2P): one fused
kernel reads every rank's gradient over peer memory, sums it in rank order,
updates the rank's element shard and stores theta' into every rank's
parameters; the shard norms are published into every rank's exchange block.

The pool has one GPU, so the multi-rank cases run W contexts ("virtual
ranks") on it with p2p_sync = 0: every buffer is local, the host orders the
ranks' calls (all steps, then every rank's grass_p2p_finish), and no kernel
ever waits on another.  The data path — peer-pointer loads, the rank-order
sum, peer stores, the publication into every rank's gather row and the
rank-order MGN sum — is exactly what runs across GPUs.  The two-process case
does the same through CUDA IPC handles (grass_ipc_export / _import), the
setup real ranks use.  world = 1 with p2p_sync = 1 also runs the device
barrier kernel (trivially satisfied by the rank itself).
"""
import os
import socket

import numpy as np
import pytest
import torch

import paper_2604_07808_b200 as G
from oracle import grass_oracle as O
from dp_tolerance import assert_dp_state_close, dp_sum_bound
from synth import layer_grad, layer_params

pytestmark = pytest.mark.gpu
# GRASS_FUZZ=k multiplies the fuzz seeds (extended runs: profiles/r01_fuzz_extended.txt)
FUZZ = int(os.environ.get("GRASS_FUZZ", "1"))
DEV = "cuda:0"


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _np(t):
    return t.detach().float().cpu().numpy()


def dp_mean(grads):
    """The oracle's DP gradient: the fp64 mean over ranks (O.dp_average, R9),
    and the bound of its fp32 rank-order evaluation (R20, tests/dp_tolerance)."""
    return O.dp_average(grads), dp_sum_bound(grads)


def _mode_kw(mode, chunk=4096):
    return {"resident": {}, "offload": dict(offload=True, chunk_elems=chunk),
            "period": dict(offload=True, residency=G.RESIDENCY_PERIOD)}[mode]


# ------------------------------------------------------------------ world = 1
@pytest.mark.parametrize("dtype", [G.DTYPE_FP32, G.DTYPE_BF16])
@pytest.mark.parametrize("mode", ["resident", "offload", "period"])
def test_p2p_one_rank_bit_identical_to_plain(dtype, mode):
    """world = 1: the P2P kernels (peer-pointer gradient, peer stores, publish +
    device barrier + rank sum) must reproduce the plain path bit for bit."""
    tdt = torch.bfloat16 if dtype == G.DTYPE_BF16 else torch.float32
    numel = [3 * 4096 + 8, 65_536, 4096 + 16]
    kw = dict(gamma=2, weight_decay=0.01, param_dtype=dtype, **_mode_kw(mode))
    ref = G.Grass(numel, **kw)
    p2p = G.Grass(numel, dp_mode=G.DP_P2P, **kw)
    blk, nbytes = p2p.p2p_exchange_block()
    assert nbytes >= 128 + 8 * len(numel)
    p2p.p2p_attach([blk])
    p_ref = [layer_params(n, l, device=DEV).to(tdt) for l, n in enumerate(numel)]
    p_p2p = [p.clone() for p in p_ref]
    g_reg = [torch.zeros(n, device=DEV, dtype=tdt) for n in numel]     # registered gradient buffers
    for l in range(len(numel)):
        p2p.p2p_register_layer(l, [p_p2p[l]], [g_reg[l]])
    for step in range(5):
        ids = [[0, 1], [2, 0], [1, 2], [0, 2], [2, 1]][step]
        for l in ids:
            g_reg[l].copy_(layer_grad(numel[l], l, 1e-3, step=step, device=DEV).to(tdt))
        ref.step_layers(ids, [p_ref[l] for l in ids], [g_reg[l] for l in ids], 1e-3)
        p2p.step_layers(ids, [p_p2p[l] for l in ids], [g_reg[l] for l in ids], 1e-3)
    for l in range(3):
        g_reg[l].copy_(layer_grad(numel[l], l, 1e-3, step=9, device=DEV).to(tdt))
    ref.mgn_accumulate([0, 1, 2], g_reg)
    p2p.mgn_accumulate([0, 1, 2], g_reg)
    ref.sync()
    p2p.sync()
    for l in range(3):
        assert torch.equal(p_ref[l], p_p2p[l]), l
        a, b = ref.read_state(l), p2p.read_state(l)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    sa, sb = ref.get_mgn(), p2p.get_mgn()
    assert sa["S"] == sb["S"] and sa["c"] == sb["c"] and sa["last_ss"] == sb["last_ss"]


def test_p2p_rejects_unregistered_and_misuse():
    numel = [4096, 8192]
    gr = G.Grass(numel, gamma=1, dp_mode=G.DP_P2P)
    p = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    g = [torch.zeros(n, device=DEV) for n in numel]
    with pytest.raises(G.GrassError, match="attach"):
        gr.step_layers([0], [p[0]], [g[0]], 1e-3)
    blk, _ = gr.p2p_exchange_block()
    with pytest.raises(G.GrassError):
        gr.p2p_attach([blk + 256])                      # not its own block
    gr.p2p_attach([blk])
    with pytest.raises(G.GrassError, match="not registered"):
        gr.step_layers([0], [p[0]], [g[0]], 1e-3)
    gr.p2p_register_layer(0, [p[0]], [g[0]])
    other = torch.zeros(4096, device=DEV)
    with pytest.raises(G.GrassError, match="registered"):
        gr.step_layers([0], [p[0]], [other], 1e-3)     # a different gradient buffer
    with pytest.raises(G.GrassError, match="aligned"):
        gr.p2p_register_layer(1, [p[1].data_ptr() + 4], [g[1]])   # misaligned parameters
    with pytest.raises(G.GrassError):
        gr.p2p_finish()                                  # p2p_sync = 1 context
    with pytest.raises(G.GrassError):
        G.Grass(numel, gamma=1, dp_mode=G.DP_P2P, max_grad_norm=1.0)
    with pytest.raises(G.GrassError):
        G.Grass(numel, gamma=1, dp_mode=G.DP_P2P, world=9, rank=0)
    gr.step_layers([0], [p[0]], [g[0]], 1e-3)
    gr.sync()


# --------------------------------------------- W virtual ranks on one GPU
class VirtualRanks:
    """W contexts (rank r of world W, p2p_sync = 0) whose buffers all live on
    this GPU: rank r's parameters P[r][l] and gradients Gr[r][l]."""

    def __init__(self, numel, W, dtype=G.DTYPE_FP32, **kw):
        self.W, self.numel = W, numel
        self.tdt = torch.bfloat16 if dtype == G.DTYPE_BF16 else torch.float32
        self.ctx = [G.Grass(numel, rank=r, world=W, dp_mode=G.DP_P2P, p2p_sync=False,
                            param_dtype=dtype, **kw) for r in range(W)]
        blocks = [c.p2p_exchange_block()[0] for c in self.ctx]
        base = [layer_params(n, l, device=DEV).to(self.tdt) for l, n in enumerate(numel)]
        self.P = [[b.clone() for b in base] for _ in range(W)]
        self.Gr = [[torch.zeros(n, device=DEV, dtype=self.tdt) for n in numel] for _ in range(W)]
        for c in self.ctx:
            c.p2p_attach(blocks)
            for l in range(len(numel)):
                c.p2p_register_layer(l, [self.P[r][l] for r in range(W)], [self.Gr[r][l] for r in range(W)])

    def set_grads(self, ids, step, seed=0):
        for r in range(self.W):
            for l in ids:
                self.Gr[r][l].copy_(layer_grad(self.numel[l], l, 1e-3, step=step, seed=seed, device=DEV,
                                               rank=r).to(self.tdt))

    def step(self, ids, lr):
        for r, c in enumerate(self.ctx):          # every rank's fused kernel, in rank order
            c.step_layers(ids, [self.P[r][l] for l in ids], [self.Gr[r][l] for l in ids], lr)
        for c in self.ctx:                        # then every rank's MGN finish
            c.p2p_finish()

    def probe(self, ids):
        for r, c in enumerate(self.ctx):
            c.mgn_accumulate(ids, [self.Gr[r][l] for l in ids])
        for c in self.ctx:
            c.p2p_finish()


@pytest.mark.parametrize("W", [2, 4, 8])
def test_p2p_virtual_ranks_vs_oracle(W):
    """W ranks: after each step every rank holds the same parameters (bit),
    equal to the oracle's AdamW on the fp64 DP mean (O.dp_average) within the
    1e-5 bars plus the propagated fp32 rank-order summation bound
    (tests/dp_tolerance.py); every rank's MGN is bit-identical and within 1e-6
    of the oracle's norms of the fp64 mean; each rank's m/v are the oracle's
    for its element shard."""
    numel = [8 * W * 1000 + 8 * W * 3, 65_536, 4096 * 3]
    lr = 1e-3
    vr = VirtualRanks(numel, W, gamma=2, weight_decay=0.01)
    orc = O.GrassOracle(numel, gamma=2, weight_decay=0.01)
    theta = [_np(vr.P[0][l]).copy() for l in range(3)]
    for step in range(3):
        ids = [[0, 1], [2, 0], [1, 2]][step]
        vr.set_grads(ids, step)
        gd = {l: dp_mean([_np(vr.Gr[r][l]) for r in range(W)]) for l in ids}
        th_in = {l: theta[l].copy() for l in ids}
        m_in = {l: orc.m[l].copy() for l in ids}
        vr.step(ids, lr)
        torch.cuda.synchronize()
        orc.step_layers(ids, [theta[l] for l in ids], [gd[l][0] for l in ids], float(np.float32(lr)))
        for l in ids:
            got = [_np(vr.P[r][l]) for r in range(W)]
            for r in range(1, W):
                assert np.array_equal(got[0], got[r]), (step, l, r)
            gm, dg = gd[l]
            m_all = np.concatenate([c.read_state(l)[0] for c in vr.ctx])   # rank shards, in order
            v_all = np.concatenate([c.read_state(l)[1] for c in vr.ctx])
            assert all(c.read_state(l)[2] == orc.t[l] for c in vr.ctx)
            assert_dp_state_close(got[0], m_all, v_all, theta[l], orc.m[l], orc.v[l], th_in[l], m_in[l], gm, dg,
                                  orc.t[l], float(np.float32(lr)), where=(W, step, l))
            theta[l][...] = got[0]                 # re-seed the oracle from the GPU
            orc.m[l][...], orc.v[l][...] = m_all, v_all
    vr.set_grads([0, 1, 2], 7)
    vr.probe([0, 1, 2])
    orc.accumulate([0, 1, 2], [O.dp_average([_np(vr.Gr[r][l]) for r in range(W)]) for l in range(3)])
    st = [c.get_mgn() for c in vr.ctx]
    for r in range(1, W):
        assert st[r]["S"] == st[0]["S"] and st[r]["c"] == st[0]["c"] and st[r]["last_ss"] == st[0]["last_ss"]
    for l in range(3):
        assert abs(st[0]["last_ss"][l] - orc.last_ss[l]) <= 1e-6 * orc.last_ss[l]
    assert st[0]["c"] == orc.mgn.c


@pytest.mark.parametrize("dtype", [G.DTYPE_FP32, G.DTYPE_BF16])
def test_p2p_virtual_ranks_offload_and_period_bit_identical(dtype):
    """W = 4 virtual ranks: per-step offload and period residency give the
    resident P2P result bit for bit (parameters, every rank's m/v, MGN)."""
    W = 4
    numel = [8 * W * 2048 + 8 * W, 65_536, 32 * 4096]
    runs = []
    for mode in ("resident", "offload", "period"):
        vr = VirtualRanks(numel, W, dtype=dtype, gamma=2, weight_decay=0.01, **_mode_kw(mode, 8192))
        for step in range(4):
            ids = [[0, 1], [2, 0], [1, 2], [0, 2]][step]
            vr.set_grads(ids, step, seed=3)
            vr.step(ids, 1e-3)
        torch.cuda.synchronize()
        runs.append(vr)
    for vr in runs[1:]:
        for r in range(W):
            for l in range(3):
                assert torch.equal(runs[0].P[r][l], vr.P[r][l])
                a, b = runs[0].ctx[r].read_state(l), vr.ctx[r].read_state(l)
                assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
            assert runs[0].ctx[r].get_mgn()["S"] == vr.ctx[r].get_mgn()["S"]


def test_p2p_virtual_ranks_schedule_always_groups():
    """The full schedule (probe, commit, sample, update) on 2 virtual ranks with
    an always-active group: identical sampled ids and probabilities on both
    ranks, always group updated every adaptive step."""
    W = 2
    numel = [8 * W * 512] * 4 + [8 * W * 100]
    vr = VirtualRanks(numel, W, gamma=2, T_p=2, T_s=2, n_always=1, seed=11)
    for step in range(8):
        d = G.schedule_decision(step, 2, 2)
        if d == G.DECIDE_PROBE:
            vr.set_grads([0, 1, 2, 3], step)
            vr.probe([0, 1, 2, 3])
            continue
        if d == G.DECIDE_COMMIT_RESAMPLE:
            probs = [c.update_probs() for c in vr.ctx]
            assert probs[0] == probs[1] and probs[0][4] == 0.0
        ids = [c.sample_layers((step - 2) // 2) for c in vr.ctx]
        assert ids[0] == ids[1] and 4 not in ids[0]
        ids = ids[0] + [4]
        vr.set_grads(ids, step)
        vr.step(ids, 1e-3)
    torch.cuda.synchronize()
    assert vr.ctx[0].read_state(4)[2] == vr.ctx[1].read_state(4)[2] == 6
    for l in range(5):
        assert torch.equal(vr.P[0][l], vr.P[1][l])


# ------------------------------------------ two processes, CUDA IPC setup
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    numel = [8 * world * 1024 + 8 * world, 65_536]
    gr = G.Grass(numel, gamma=2, rank=rank, world=world, dp_mode=G.DP_P2P, p2p_sync=False,
                 weight_decay=0.01)
    P = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
    Gr = [layer_grad(n, l, 1e-3, step=0, device=DEV, rank=rank) for l, n in enumerate(numel)]
    init = [_np(p).copy() for p in P]
    gr.p2p_setup({l: (P[l], Gr[l]) for l in range(2)})   # IPC handles through the gloo group
    torch.cuda.synchronize()
    dist.barrier()
    gr.step_layers([0, 1], P, Gr, 1e-3)                   # both processes' kernels may overlap:
    torch.cuda.synchronize()                              # neither waits on the other
    dist.barrier()                                        # every rank's publication is done
    gr.p2p_finish()
    gr.sync()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), p0=_np(P[0]), p1=_np(P[1]), i0=init[0], i1=init[1],
             g0=_np(Gr[0]), g1=_np(Gr[1]), S=np.array(gr.get_mgn()["S"]),
             ss=np.array(gr.get_mgn()["last_ss"]))
    dist.barrier()
    dist.destroy_process_group()


def test_p2p_two_processes_ipc(tmp_path):
    import torch.multiprocessing as mp
    W = 2
    mp.spawn(_ipc_worker, args=(W, _free_port(), str(tmp_path)), nprocs=W, join=True)
    r = [np.load(tmp_path / f"r{q}.npz") for q in range(W)]
    numel = [8 * W * 1024 + 8 * W, 65_536]
    for l in range(2):
        assert np.array_equal(r[0][f"p{l}"], r[1][f"p{l}"])   # theta' reached both processes
        gavg, dg = dp_mean([r[q][f"g{l}"] for q in range(W)])
        th0 = r[0][f"i{l}"]
        assert np.array_equal(th0, r[1][f"i{l}"])
        th, m_o, v_o = O.adamw_step(th0, np.zeros_like(th0), np.zeros_like(th0), gavg, 1,
                                    float(np.float32(1e-3)), weight_decay=0.01)
        assert_dp_state_close(r[0][f"p{l}"], m_o, v_o, th, m_o, v_o, th0, 0 * th0, gavg, dg, 1,
                              float(np.float32(1e-3)), where=l)
        assert abs(r[0]["ss"][l] - O.sq_norm(gavg)) <= 1e-6 * O.sq_norm(gavg)
    assert np.array_equal(r[0]["S"], r[1]["S"])


@pytest.mark.parametrize("seed", range(FUZZ * 6))
def test_p2p_fuzz_bit_identical_to_plain_on_the_averaged_gradient(seed):
    """Random world (incl. non-powers of two), ragged layer sizes, random
    active sets and residency modes: the W-rank P2P update of every element
    equals, bit for bit, the single-GPU update fed with the same DP gradient
    formed the way the kernel forms it (fp32 sum in rank order, x fp32(1/W));
    the per-layer norms agree to fp64 summation order (1e-12)."""
    rng = np.random.default_rng(200 + seed)
    W = int(rng.choice([2, 3, 4, 5, 8]))
    nl = int(rng.integers(2, 6))
    numel = [8 * W * int(rng.integers(1, 3000)) for _ in range(nl)]
    mode = ["resident", "offload", "period"][seed % 3]
    kw = dict(gamma=nl, weight_decay=0.01, **_mode_kw(mode, 4096 * int(rng.integers(1, 4))))
    vr = VirtualRanks(numel, W, **kw)
    ref = G.Grass(numel, **{**kw, "offload": False, "residency": 0, "chunk_elems": 0})
    p_ref = [p.clone() for p in vr.P[0]]
    inv = torch.tensor(1.0 / W, dtype=torch.float32, device=DEV)
    for step in range(5):
        ids = [int(x) for x in rng.choice(nl, size=int(rng.integers(1, nl + 1)), replace=False)]
        vr.set_grads(ids, step, seed=seed)
        gavg = []
        for l in ids:
            acc = vr.Gr[0][l].clone()
            for r in range(1, W):
                acc += vr.Gr[r][l]
            gavg.append(acc * inv)
        vr.step(ids, 1e-3)
        ref.step_layers(ids, [p_ref[l] for l in ids], gavg, 1e-3)
    torch.cuda.synchronize()
    for l in range(nl):
        for r in range(W):
            assert torch.equal(vr.P[r][l], p_ref[l]), (W, mode, l, r)
        m_ref, v_ref, t_ref = ref.read_state(l)
        for r, c in enumerate(vr.ctx):
            off, cnt = G.shard_range(numel[l], W, r)
            m, v, t = c.read_state(l)
            assert t == t_ref and np.array_equal(m, m_ref[off:off + cnt]) and np.array_equal(v, v_ref[off:off + cnt])
    s_ref = ref.get_mgn()
    for c in vr.ctx:
        st = c.get_mgn()
        assert st["c"] == s_ref["c"]
        for l in range(nl):
            assert abs(st["S"][l] - s_ref["S"][l]) <= 1e-12 * abs(s_ref["S"][l]) + 1e-300


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_p2p_barrier_protocol_selftest(W):
    """The publication + end barrier + start barrier protocol of the P2P path
    with W ranks emulated as the co-resident CTAs of one cooperative launch:
    after every end barrier each rank holds every rank's row of that round,
    and no rank overwrites a row before every rank has read it."""
    mismatches, timed_out = G.selftest_p2p(W, rounds=2000)
    assert mismatches == 0 and not timed_out


def test_p2p_full_size_7b_layers_four_ranks():
    """LLaMA-2-7B decoder layers (N_p = 202,383,360) on 4 virtual ranks, the
    bench's launch configuration: every rank ends with the same parameters
    (bit), the full-layer norm of the DP gradient is within 1e-6 of the
    oracle's (fp64 DP mean), and AdamW on sampled elements (first/last 4096 +
    100k random) matches the oracle fed with the fp64 DP mean within the bars
    + the propagated rank-order summation bound."""
    from synth import MODELS
    W, n = 4, MODELS["llama2-7b"].layer_numel
    numel = [n, n]
    vr = VirtualRanks(numel, W, gamma=2, weight_decay=0.01)
    rng = np.random.default_rng(1)
    idx = np.unique(np.concatenate([np.arange(4096), n - 1 - np.arange(4096), rng.integers(0, n, 100_000)]))
    ti = torch.from_numpy(idx).to(DEV)
    th_in = [_np(vr.P[0][l][ti]) for l in range(2)]
    vr.set_grads([0, 1], 0)
    vr.step([0, 1], 3e-5)
    torch.cuda.synchronize()
    st = vr.ctx[0].get_mgn()
    for l in range(2):
        for r in range(1, W):
            assert torch.equal(vr.P[0][l], vr.P[r][l])
        gavg, dg = dp_mean([_np(vr.Gr[r][l]) for r in range(W)])
        ss = O.sq_norm(gavg)
        assert abs(st["last_ss"][l] - ss) <= 1e-6 * ss
        g_s = gavg[idx]
        th_o, m_o, v_o = O.adamw_step(th_in[l], np.zeros_like(g_s), np.zeros_like(g_s), g_s, 1,
                                      float(np.float32(3e-5)), weight_decay=0.01)
        got = _np(vr.P[0][l][ti])
        m_all = np.concatenate([c.read_state(l)[0] for c in vr.ctx])   # rank shards, in order
        v_all = np.concatenate([c.read_state(l)[1] for c in vr.ctx])
        assert_dp_state_close(got, m_all[idx], v_all[idx], th_o, m_o, v_o, th_in[l], 0 * g_s, g_s, dg[idx], 1,
                              float(np.float32(3e-5)), where=l)


@pytest.mark.parametrize("path", ["nccl", "p2p"])
def test_debug_check_world1(path):
    """debug_check: grass_update_probs all-gathers a hash of the MGN and the
    probabilities (NCCL, or the P2P exchange blocks + end barrier) and compares
    them — at world 1 the path runs and agrees with itself."""
    numel = [4096 * 3, 8192]
    kw = dict(gamma=1, T_p=1, T_s=1, debug_check=True)
    gr = (G.Grass(numel, force_nccl=True, **kw) if path == "nccl"
          else G.Grass(numel, dp_mode=G.DP_P2P, **kw))
    g = [layer_grad(n, l, 1e-3, device=DEV) for l, n in enumerate(numel)]
    if path == "p2p":
        gr.p2p_attach([gr.p2p_exchange_block()[0]])
        p = [layer_params(n, l, device=DEV) for l, n in enumerate(numel)]
        for l in range(2):
            gr.p2p_register_layer(l, [p[l]], [g[l]])
    before = gr.launch_count
    gr.mgn_accumulate([0, 1], g)
    probs = gr.update_probs()
    assert abs(sum(probs) - 1.0) < 1e-12
    assert gr.launch_count >= before + 2      # the norm launches plus the check's collective
    plain = G.Grass(numel, **{k: v for k, v in kw.items() if k != "debug_check"})
    plain.mgn_accumulate([0, 1], g)
    assert plain.update_probs() == probs


def test_p2p_checkpoint_roundtrip_virtual_ranks(tmp_path):
    """Every virtual rank writes its checkpoint; fresh P2P contexts restored from
    them continue bit-identically to the uninterrupted run."""
    W = 2
    numel = [8 * W * 700, 8 * W * 1300]
    vr = VirtualRanks(numel, W, gamma=2, weight_decay=0.01)
    for step in range(2):
        vr.set_grads([0, 1], step)
        vr.step([0, 1], 1e-3)
    torch.cuda.synchronize()
    for r, c in enumerate(vr.ctx):
        c.save_state(str(tmp_path / f"r{r}"))
    snap = [[p.clone() for p in vr.P[r]] for r in range(W)]
    vr2 = VirtualRanks(numel, W, gamma=2, weight_decay=0.01)
    for r, c in enumerate(vr2.ctx):
        c.load_state(str(tmp_path / f"r{r}"))
        for l in range(2):
            vr2.P[r][l].copy_(snap[r][l])
    for step in range(2, 4):
        for v in (vr, vr2):
            v.set_grads([0, 1], step)
            v.step([0, 1], 1e-3)
    torch.cuda.synchronize()
    for r in range(W):
        for l in range(2):
            assert torch.equal(vr.P[r][l], vr2.P[r][l])
            a, b = vr.ctx[r].read_state(l), vr2.ctx[r].read_state(l)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2] == 4
