"""e2e leg (configs[1] with the step's gradients in pinned host memory,
streamed through the context's gradient ring) as a function of the ring's
chunk size: fill / drain of the H2D pipeline vs per-chunk launch overhead.
    python tools/e2e_chunk_sweep.py     # -> stdout JSON
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_07808_b200 as G  # noqa: E402
from synth import MODELS, grad_sigmas, layer_grad, layer_params  # noqa: E402

shape = MODELS["llama2-7b"]
n, NL = shape.layer_numel, shape.n_layers
dev = torch.device("cuda", 0)
sig = grad_sigmas(NL, 0)
ids = [3, 17]
params = {l: layer_params(n, l, device=dev, norm_numel=shape.norm_numel) for l in ids}
host_g = [layer_grad(n, l, sig[l]).pin_memory() for l in ids]
s = torch.cuda.Stream(device=dev)
res = {}
for chunk_mi in (16, 8, 4, 2, 1):
    ctx = G.Grass([n] * NL, gamma=2, T_p=1, T_s=1, chunk_elems=chunk_mi << 20, ring_slots=3)
    for _ in range(2):
        ctx.step_layers(ids, [params[l] for l in ids], host_g, 3e-5, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    K = 8
    for _ in range(K):
        ctx.step_layers(ids, [params[l] for l in ids], host_g, 3e-5, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    res[f"{chunk_mi}Mi"] = {"ms_per_step": round(ms, 3), "h2d_GBps": round(2 * n * 4 / ms / 1e6, 1)}
    print(chunk_mi, res[f"{chunk_mi}Mi"], flush=True)
    ctx.close()
print(json.dumps(res))
