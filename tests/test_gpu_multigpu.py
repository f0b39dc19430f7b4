"""Data parallelism across REAL GPUs (DESIGN §10/§13): runs when
>= 2 GPUs are visible (skipped on the 1-GPU pool; the W = 1 case of the same
harness runs everywhere and checks the harness itself).

For W in {2, 4, 8} (as many as are visible), both data paths — NCCL (grouped
send/recv of the gradient slices + the update kernel's fp32 rank-order sum +
ncclAllGather of theta) and P2P (one fused kernel over CUDA-IPC-mapped peer
memory with device barriers, p2p_sync = 1) — and both dtypes:
  * every rank ends with bit-identical parameters, MGN window, probabilities
    and sampled ids;
  * NCCL and P2P agree bit for bit (the same fp32 rank-order arithmetic, R20);
  * against the oracle fed with the fp64 DP mean (O.dp_average): norms within
    1e-6, theta / m / v within the DESIGN §6 bars plus the propagated fp32
    summation bound (tests/dp_tolerance.py), after every step;
  * P2P records the NVLink bytes per rank (8 B x gamma N_p (W-1)/W).
Two launch styles: one process per GPU (torch.multiprocessing, NCCL process
group, CUDA IPC for P2P), and W threads of ONE process, one per GPU (peer
access enabled; the device barriers then cross real GPUs in one process).
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch

import paper_2604_07808_b200 as G
from dp_tolerance import assert_dp_state_close, dp_sum_bound
from oracle import grass_oracle as O
from synth import layer_grad, layer_params

pytestmark = pytest.mark.gpu
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
WORLDS = [w for w in (2, 4, 8) if w <= NGPU]
multigpu = pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs (the pool has 1)")
LR, WD = 1e-3, 0.01
STEPS = [[0, 1], [2, 0], [1, 2]]


def _numel(W):
    return [8 * W * 3000 + 8 * W * 5, 65_536, 4096 * 3]      # divisible by 8W: bf16 shards


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _f32(t):
    return t.detach().float().cpu().numpy()


def run_rank(rank, W, mode, dtype, ctx_kw, setup):
    """One rank's workload: 3 steps of grass_step_layers, a probing pass,
    commit, sample.  `setup(ctx, params, grads)` wires the data path (P2P
    attach / register).  Returns per-step snapshots as numpy."""
    dev = torch.device("cuda", torch.cuda.current_device())
    tdt = torch.bfloat16 if dtype == G.DTYPE_BF16 else torch.float32
    numel = _numel(W)
    ctx = G.Grass(numel, gamma=2, T_p=1, T_s=1, weight_decay=WD, param_dtype=dtype, rank=rank, world=W,
                  device=dev.index, dp_mode=mode, **ctx_kw)
    params = [layer_params(n, l, device=dev).to(tdt) for l, n in enumerate(numel)]
    grads = [torch.zeros(n, device=dev, dtype=tdt) for n in numel]
    setup(ctx, params, grads)
    out = {"steps": []}
    for step, ids in enumerate(STEPS):
        for l in ids:
            grads[l].copy_(layer_grad(numel[l], l, 1e-3, step=step, device=dev, rank=rank).to(tdt))
        torch.cuda.synchronize()
        ctx.step_layers(ids, [params[l] for l in ids], [grads[l] for l in ids], LR)
        ctx.sync()
        snap = {"ids": ids, "params": {l: _f32(params[l]) for l in ids},
                "grads": {l: _f32(grads[l]) for l in ids},
                "m": {l: ctx.read_state(l)[0] for l in ids}, "v": {l: ctx.read_state(l)[1] for l in ids},
                "t": {l: ctx.read_state(l)[2] for l in ids}}
        if dtype == G.DTYPE_BF16:
            snap["master"] = {l: ctx.read_master(l) for l in ids}
        out["steps"].append(snap)
    for l in range(3):
        grads[l].copy_(layer_grad(numel[l], l, 1e-3, step=7, device=dev, rank=rank).to(tdt))
    torch.cuda.synchronize()
    ctx.mgn_accumulate([0, 1, 2], grads)
    st = ctx.get_mgn()
    out["probe_grads"] = [_f32(g) for g in grads]
    out["S"], out["c"], out["last_ss"] = st["S"], st["c"], st["last_ss"]
    out["probs"] = ctx.update_probs()
    out["ids"] = ctx.sample_layers(0)
    out["shards"] = [ctx.shard(l) for l in range(3)]
    out["init_params"] = [_f32(layer_params(n, l, device=dev).to(tdt)) for l, n in enumerate(numel)]
    ctx.close()
    return out


# --------------------------------------------------- one process per GPU
def _proc_worker(rank, W, port, mode, dtype, out_dir):
    import pickle

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=W, device_id=torch.device("cuda", rank))

    def setup(ctx, params, grads):
        if mode == G.DP_P2P:
            ctx.p2p_setup({l: (params[l], grads[l]) for l in range(3)})   # CUDA IPC over the group
            torch.cuda.synchronize()
            dist.barrier()
    out = run_rank(rank, W, mode, dtype, {}, setup)
    with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)
    dist.barrier()
    dist.destroy_process_group()


def _run_processes(W, mode, dtype, tmp_path):
    import pickle

    import torch.multiprocessing as mp
    d = tmp_path / f"{mode}_{dtype}"
    d.mkdir()
    mp.spawn(_proc_worker, args=(W, _free_port(), mode, dtype, str(d)), nprocs=W, join=True)
    return [pickle.load(open(d / f"r{r}.pkl", "rb")) for r in range(W)]


# --------------------------------------------------- W threads of one process
def _run_threads(W, mode, dtype):
    for a in range(W):
        for b in range(W):
            if a != b:
                G.enable_peer_access(a, b)
    nid = G.nccl_unique_id() if mode == G.DP_NCCL and W > 1 else None
    ctxs, bufs, outs, errs = [None] * W, [None] * W, [None] * W, []
    created = threading.Barrier(W)

    def setup_for(rank):
        def setup(ctx, params, grads):
            ctxs[rank] = ctx
            bufs[rank] = (params, grads)
            created.wait()                               # every rank's buffers exist
            if mode == G.DP_P2P:
                ctx.p2p_attach([ctxs[q].p2p_exchange_block()[0] for q in range(W)])
                for l in range(3):
                    ctx.p2p_register_layer(l, [bufs[q][0][l] for q in range(W)], [bufs[q][1][l] for q in range(W)])
            created.wait()
        return setup

    def body(rank):
        try:
            torch.cuda.set_device(rank)
            kw = {"nccl_id": nid} if nid is not None else ({"force_nccl": True} if mode == G.DP_NCCL else {})
            outs[rank] = run_rank(rank, W, mode, dtype, kw, setup_for(rank))
        except BaseException as ex:  # surfaced below
            errs.append(repr(ex))
            created.abort()
    th = [threading.Thread(target=body, args=(r,)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return outs


# ------------------------------------------------------------------- checks
def check_against_oracle(res, W, dtype):
    """res: per-rank results.  Cross-rank identity + oracle parity."""
    numel = _numel(W)
    for r in range(1, W):
        assert res[r]["S"] == res[0]["S"] and res[r]["c"] == res[0]["c"] and res[r]["last_ss"] == res[0]["last_ss"]
        assert res[r]["probs"] == res[0]["probs"] and res[r]["ids"] == res[0]["ids"]
        for k, snap in enumerate(res[r]["steps"]):
            for l in snap["ids"]:
                assert np.array_equal(snap["params"][l], res[0]["steps"][k]["params"][l]), (r, k, l)
    orc = O.GrassOracle(numel, gamma=2, weight_decay=WD)
    theta = [res[0]["init_params"][l].astype(np.float32).copy() for l in range(3)]
    bf16 = dtype == G.DTYPE_BF16
    for k, ids in enumerate(STEPS):
        for l in ids:
            gr = [res[r]["steps"][k]["grads"][l] for r in range(W)]
            gmean, dg = O.dp_average(gr), dp_sum_bound(gr)
            th_in = theta[l].copy()
            m_in, v_in = orc.m[l].copy(), orc.v[l].copy()
            t = orc.t[l] + 1
            th_o, m_o, v_o = O.adamw_step(th_in, m_in, v_in, gmean, t, float(np.float32(LR)), weight_decay=WD)
            orc.t[l] = t
            m_all = np.concatenate([res[r]["steps"][k]["m"][l] for r in range(W)])
            v_all = np.concatenate([res[r]["steps"][k]["v"][l] for r in range(W)])
            got = (np.concatenate([res[r]["steps"][k]["master"][l] for r in range(W)]) if bf16
                   else res[0]["steps"][k]["params"][l])
            assert_dp_state_close(got, m_all, v_all, th_o, m_o, v_o, th_in, m_in, gmean, dg, t,
                                  float(np.float32(LR)), where=(W, k, l))
            if bf16:   # the bf16 model copy is RNE(master') on every rank
                assert np.array_equal(O.bf16_to_f32(O.f32_to_bf16(got)), res[0]["steps"][k]["params"][l])
            assert all(res[r]["steps"][k]["t"][l] == t for r in range(W))
            theta[l][...] = got                                # re-seed the oracle from the GPU
            orc.m[l][...], orc.v[l][...] = m_all, v_all
    for l in range(3):
        ss = O.sq_norm(O.dp_average([res[r]["probe_grads"][l] for r in range(W)]))
        assert abs(res[0]["last_ss"][l] - ss) <= 1e-6 * ss, (l, res[0]["last_ss"][l], ss)


def check_paths_identical(a, b, W):
    """NCCL and P2P: the same bits (theta, states, MGN, probabilities, ids)."""
    for r in range(W):
        assert a[r]["S"] == b[r]["S"] and a[r]["last_ss"] == b[r]["last_ss"] and a[r]["probs"] == b[r]["probs"]
        for k in range(len(STEPS)):
            for key in ("params", "m", "v"):
                for l in STEPS[k]:
                    assert np.array_equal(a[r]["steps"][k][key][l], b[r]["steps"][k][key][l]), (r, k, key, l)


def nvlink_bytes_per_rank(W, dtype):
    esz = 2 if dtype == G.DTYPE_BF16 else 4
    numel = _numel(W)
    per_step = [sum(numel[l] for l in ids) for ids in STEPS]
    return [2 * esz * n * (W - 1) // W for n in per_step]


# -------------------------------------------------------------------- tests
@multigpu
@pytest.mark.parametrize("W", WORLDS)
@pytest.mark.parametrize("dtype", [G.DTYPE_FP32, G.DTYPE_BF16])
def test_multigpu_processes_nccl_and_p2p_vs_oracle(W, dtype, tmp_path):
    res = {mode: _run_processes(W, mode, dtype, tmp_path) for mode in (G.DP_NCCL, G.DP_P2P)}
    for mode in res:
        check_against_oracle(res[mode], W, dtype)
    check_paths_identical(res[G.DP_NCCL], res[G.DP_P2P], W)
    rec = os.environ.get("GRASS_RECORD_DIR")
    if rec:
        import json
        os.makedirs(rec, exist_ok=True)
        with open(os.path.join(rec, f"multigpu_W{W}_dtype{dtype}.json"), "w") as f:
            json.dump({"W": W, "dtype": dtype, "p2p_nvlink_bytes_per_rank_per_step": nvlink_bytes_per_rank(W, dtype),
                       "ok": True}, f)


@multigpu
@pytest.mark.parametrize("W", WORLDS)
@pytest.mark.parametrize("mode", [G.DP_NCCL, G.DP_P2P])
def test_multigpu_threads_one_process_vs_oracle(W, mode):
    """W contexts on W devices in one process, one thread each: the P2P device
    barriers and peer loads / stores cross real GPUs."""
    res = _run_threads(W, mode, G.DTYPE_FP32)
    check_against_oracle(res, W, G.DTYPE_FP32)


@pytest.mark.parametrize("mode", [G.DP_NCCL, G.DP_P2P])
def test_multigpu_harness_world1(mode):
    """The harness above at W = 1 on one GPU (runs on the pool): the same
    workload, oracle checks and NCCL / P2P identity."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    res = _run_threads(1, mode, G.DTYPE_FP32)
    check_against_oracle(res, 1, G.DTYPE_FP32)
    if mode == G.DP_P2P:
        other = _run_threads(1, G.DP_NCCL, G.DTYPE_FP32)
        check_paths_identical(other, res, 1)
