"""configs[1] device-resident steps (grass_device_step), eager and graph-replayed,
for ncu launch lists:  ncu --metrics gpu__time_duration.sum python tools/device_step_profile.py"""
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
params = [layer_params(n, l, device=dev) for l in range(NL)]
grads = [layer_grad(n, l, sig[l], device=dev) for l in range(NL)]
s = torch.cuda.Stream(device=dev)
ctx = G.Grass([n] * NL, gamma=2, T_p=1, T_s=1, T_u=1, seed=1234)
ctx.mgn_accumulate(list(range(NL)), grads, stream=s)
ctx.update_probs()
ctx.register_layers(params, grads)
ctx.device_schedule_begin(0, stream=s)
for _ in range(5):
    ctx.device_step(3e-5, stream=s)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
e[0].record(s)
for _ in range(20):
    ctx.device_step(3e-5, stream=s)
e[1].record(s)
ctx.sync()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        ctx.device_step(3e-5, stream=s)
e[2].record(s)
with torch.cuda.stream(s):
    for _ in range(20):
        g.replay()
e[3].record(s)
torch.cuda.synchronize()
print(f"eager {e[0].elapsed_time(e[1]) / 20:.4f} ms/step, graph {e[2].elapsed_time(e[3]) / 20:.4f} ms/step")
print("ids", ctx.device_schedule_end())
