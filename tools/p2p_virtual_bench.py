"""The P2P fused kernel (f2) with W "virtual ranks" on ONE GPU (p2p_sync = 0,
every rank's buffers local): each rank's call reads W gradient slices of its
element shard, updates it, and stores theta' into W parameter buffers — the
same kernel and access pattern as across GPUs, with HBM standing in for
NVLink.  Reports each rank's call time and its HBM bytes / time, i.e. whether
the gradient ring keeps the kernel at the memory roofline as W grows (over
NVLink the same kernel is then link-bound).

    python tools/p2p_virtual_bench.py      # on the GPU box; prints JSON
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_07808_b200 as G  # noqa: E402
from synth import MODELS, layer_grad, layer_params  # noqa: E402


def run(W, n, gamma=2, reps=5):
    numel = [n] * gamma
    ctx = [G.Grass(numel, gamma=gamma, rank=r, world=W, dp_mode=G.DP_P2P, p2p_sync=False) for r in range(W)]
    blocks = [c.p2p_exchange_block()[0] for c in ctx]
    P = [[layer_params(n, l, device="cuda") for l in range(gamma)] for _ in range(W)]
    Gr = [[layer_grad(n, l, 1e-3, device="cuda", rank=r) for l in range(gamma)] for r in range(W)]
    for c in ctx:
        c.p2p_attach(blocks)
        for l in range(gamma):
            c.p2p_register_layer(l, [P[r][l] for r in range(W)], [Gr[r][l] for r in range(W)])
    ids = list(range(gamma))
    times = []
    for it in range(reps + 1):
        evs = []
        for r, c in enumerate(ctx):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            c.step_layers(ids, P[r], Gr[r], 1e-3)
            e1.record()
            evs.append((e0, e1))
        for c in ctx:
            c.p2p_finish()
        torch.cuda.synchronize()
        if it:
            times.append(sum(a.elapsed_time(b) for a, b in evs) / W)
    for c in ctx:
        c.close()
    ms = min(times)
    shard = gamma * n // W
    bytes_per_rank = shard * (4 * W + 4 + 8 + 8 + 4 * W)   # W grad slices + theta + m,v in/out + W theta' stores
    return {"world": W, "call_ms_per_rank": ms, "bytes_per_rank": bytes_per_rank,
            "GBps_per_rank": bytes_per_rank / (ms / 1e3) / 1e9}


def main():
    n = MODELS["llama2-7b"].layer_numel
    print(json.dumps([run(W, n) for W in (1, 2, 4, 8)], indent=1))


if __name__ == "__main__":
    main()
