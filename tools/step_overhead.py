"""Where the every-step-resample loop spends its non-kernel time: host time of
each call (perf_counter) and the GPU gap between consecutive steps' kernels.
    python tools/step_overhead.py
"""
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_07808_b200 as G  # noqa: E402
from synth import MODELS, grad_sigmas, layer_grad, layer_params  # noqa: E402

shape = MODELS["llama2-7b"]
n, NL = shape.layer_numel, shape.n_layers
dev = torch.device("cuda", 0)
sig = grad_sigmas(NL, 0)
params = [layer_params(n, l, device=dev) for l in range(NL)]
grads = [layer_grad(n, l, sig[l], device=dev) for l in range(NL)]
s = torch.cuda.Stream(device=dev)
ctx = G.Grass([n] * NL, gamma=2, T_p=1, T_s=1, T_u=1, seed=1234)
ctx.mgn_accumulate(list(range(NL)), grads, stream=s)
ctx.update_probs()
ids = ctx.sample_layers(0)
rec = {"step_layers_host_us": [], "update_probs_host_us": [], "sample_host_us": [], "step_total_us": []}
ev = []
for k in range(40):
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    ctx.step_layers(ids, [params[l] for l in ids], [grads[l] for l in ids], 3e-5, stream=s)
    e1.record(s)
    t1 = time.perf_counter()
    ctx.update_probs()
    t2 = time.perf_counter()
    ids = ctx.sample_layers(k + 1)
    t3 = time.perf_counter()
    if k >= 5:
        rec["step_layers_host_us"].append((t1 - t0) * 1e6)
        rec["update_probs_host_us"].append((t2 - t1) * 1e6)
        rec["sample_host_us"].append((t3 - t2) * 1e6)
        rec["step_total_us"].append((t3 - t0) * 1e6)
        ev.append((e0, e1))
torch.cuda.synchronize()
kern = [a.elapsed_time(b) * 1e3 for a, b in ev]
gaps = [ev[i][1].elapsed_time(ev[i + 1][0]) * 1e3 for i in range(len(ev) - 1)]
out = {k: round(statistics.median(v), 1) for k, v in rec.items()}
out["gpu_step_us"] = round(statistics.median(kern), 1)
out["gpu_gap_between_steps_us"] = round(statistics.median(gaps), 1)
print(json.dumps(out))
