"""Sweep the offload pipeline's chunk size and ring depth (step residency) on
a 4-layer LLaMA-2-7B-shaped stack, gamma = 2; prints ms/step and link GB/s."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_07808_b200 as G  # noqa: E402
from synth import MODELS, layer_grad, layer_params  # noqa: E402

n = MODELS["llama2-7b"].layer_numel
dev = "cuda:0"
params = [layer_params(n, l, device=dev) for l in range(4)]
grads = [layer_grad(n, l, 1e-4, device=dev) for l in range(4)]
s = torch.cuda.Stream()
res = {}
for chunk_mi in (2, 4, 8, 16, 32):
    for slots in (2, 3, 4):
        ctx = G.Grass([n] * 4, gamma=2, offload=True, chunk_elems=chunk_mi << 20, ring_slots=slots)
        ids = [0, 1]
        for _ in range(2):
            ctx.step_layers(ids, [params[l] for l in ids], [grads[l] for l in ids], 1e-4, stream=s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        K = 5
        for k in range(K):
            ids = [[0, 1], [2, 3]][k % 2]
            ctx.step_layers(ids, [params[l] for l in ids], [grads[l] for l in ids], 1e-4, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        res[f"chunk{chunk_mi}Mi_slots{slots}"] = {"ms": ms, "GBps_per_dir": 8 * 2 * n / ms / 1e6}
        print(chunk_mi, slots, res[f"chunk{chunk_mi}Mi_slots{slots}"], flush=True)
        del ctx
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "offload_sweep.json"), "w"), indent=1)
