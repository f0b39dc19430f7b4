"""World-size-2 CPU tests (gloo) of the data-parallel decomposition that
libgrass runs over NCCL when world > 1 (include/grass.h, grass_step_layers):

  N1  exchange of each active layer's gradient slices (rank r sends slice q to
      rank q: point-to-point send / recv, as the library's grouped ncclSend /
      ncclRecv), then the W slices of the shard summed in ascending rank order
      in fp32 and x fp32(1/W) (what the update kernel does, reading R20)
  a1  fp64 squared norm of the shard, N3 all-gather of the shard partials,
      fixed ascending-rank sum -> identical ss_l on every rank
  a5  AdamW on the shard with this rank's m/v slice
  N2  all-gather of the parameter shards
  a3/a4 probabilities and sampled ids identical on every rank

The shard plan and the sampler are the LIBRARY's host functions
(grass_shard_range, grass_sample_from_probs); the arithmetic on each shard is
the oracle's, and the result must equal the oracle run on the full,
DP-averaged gradient — the statement the GPU path implements.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2604_07808_b200 as G
        from oracle import grass_oracle as O
        from synth import grad_sigmas, layer_grad, layer_params

        numel = [4096 * 3, 8 * 1000, 4096 + 8 * 7]          # all divisible by 4*world
        sig = grad_sigmas(3, 0)
        lr, wd, seed = 1e-3, 0.01, 1234
        ids = [2, 0]
        out = {}
        # --- every rank holds full params (replicas) and its own local grads
        params = [layer_params(numel[l], l).numpy() for l in range(3)]
        local = [layer_grad(numel[l], l, sig[l], rank=rank).numpy() for l in range(3)]
        shard_ss, new_params = [], {}
        for j, l in enumerate(sorted(ids)):
            off, cnt = G.shard_range(numel[l], world, rank)
            # N1: exchange — slice q of this rank's gradient to rank q, every
            # rank's slice of this shard received into slot q (own: a copy)
            slots = [None] * world
            reqs = []
            for peer in range(world):
                if peer == rank:
                    slots[peer] = torch.from_numpy(local[l][off:off + cnt].copy())
                    continue
                slots[peer] = torch.empty(cnt)
                reqs.append(dist.isend(torch.from_numpy(local[l][peer * cnt:(peer + 1) * cnt].copy()), dst=peer))
                reqs.append(dist.irecv(slots[peer], src=peer))
            for rq in reqs:
                rq.wait()
            # the kernel's sum: ascending rank order in fp32, then x fp32(1/W)
            acc = slots[0].clone()
            for peer in range(1, world):
                acc = acc + slots[peer]
            g_shard = (acc * torch.tensor(1.0 / world, dtype=torch.float32)).numpy()
            shard_ss.append(O.sq_norm(g_shard))
            th, m, v = O.adamw_step(params[l][off:off + cnt], np.zeros(cnt, np.float32),
                                    np.zeros(cnt, np.float32), g_shard, 1, lr, weight_decay=wd)
            # N2: all-gather of the parameter shards
            parts = [torch.empty(cnt) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(th))
            new_params[l] = torch.cat(parts).numpy()
        # N3: all-gather shard partials, ascending-rank sum
        ss_all = [torch.zeros(len(ids), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(ss_all, torch.tensor(shard_ss, dtype=torch.float64))
        ss = [float(sum(ss_all[r][j] for r in range(world))) for j in range(len(ids))]
        out["ss"] = ss
        out["params"] = {l: new_params[l] for l in new_params}
        out["local"] = {l: local[l] for l in ids}
        # identical MGN -> identical probs -> identical ids on every rank
        m = [O.rms_norm(x, numel[l]) for x, l in zip(ss, sorted(ids))] + [1e-4]
        p = G.softmax_probs(m, 1.0, True)
        out["probs"] = p
        out["ids"] = G.sample_from_probs(p, 2, seed, 7)
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


def test_dp_sharded_decomposition_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in res[r], res[r].get("error")

    sys.path.insert(0, ROOT)
    from oracle import grass_oracle as O
    from synth import grad_sigmas, layer_grad, layer_params
    numel = [4096 * 3, 8 * 1000, 4096 + 8 * 7]
    sig = grad_sigmas(3, 0)
    from dp_tolerance import assert_dp_state_close, dp_sum_bound
    for j, l in enumerate([0, 2]):
        # the oracle on the full DP-averaged gradient (fp64 mean, R9 / R20)
        per_rank = [layer_grad(numel[l], l, sig[l], rank=r).numpy() for r in range(world)]
        for r in range(world):
            np.testing.assert_array_equal(res[r]["local"][l], per_rank[r])
        g, dg = O.dp_average(per_rank), dp_sum_bound(per_rank)
        ss_full = O.sq_norm(g)
        for r in range(world):
            assert res[r]["ss"][j] == pytest.approx(ss_full, rel=1e-6)
        assert res[0]["ss"] == res[1]["ss"]                  # bit-identical across ranks
        th0 = layer_params(numel[l], l).numpy()
        z = np.zeros(numel[l], np.float32)
        th, m1, v1 = O.adamw_step(th0, z, z, g, 1, 1e-3, weight_decay=0.01)
        for r in range(world):
            np.testing.assert_array_equal(res[r]["params"][l], res[0]["params"][l])
            assert_dp_state_close(res[r]["params"][l], m1, v1, th, m1, v1, th0, z, g, dg, 1, 1e-3)
    assert res[0]["probs"] == res[1]["probs"]
    assert res[0]["ids"] == res[1]["ids"]


@pytest.mark.slow
def test_bench_reference_arm_under_torchrun_world2():
    """The driver's N>1 launch of the reference arm: rank 0 prints one JSON
    line, the other rank exits 0 without work."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
