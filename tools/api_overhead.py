"""Host-side cost of the C-ABI calls on tiny layers (GPU time negligible)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_07808_b200 as G  # noqa: E402

dev = "cuda:0"
gr = G.Grass([4096] * 32, gamma=2, T_p=1, T_s=1)
p = [torch.zeros(4096, device=dev) for _ in range(32)]
g = [torch.ones(4096, device=dev) * 1e-3 for _ in range(32)]
gr.mgn_accumulate(list(range(32)), g)
gr.update_probs()
ids = gr.sample_layers(0)
s = torch.cuda.current_stream()
res = {}
def step():
    gr.step_layers(ids, [p[l] for l in ids], [g[l] for l in ids], 1e-3)


def step_commit():
    step()
    gr.update_probs()


for name, fn in (("step_layers", step), ("step_plus_update_probs", step_commit),
                 ("sample_layers", lambda: gr.sample_layers(7))):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(2000):
        fn()
    res[name + "_us"] = (time.perf_counter() - t) / 2000 * 1e6
    torch.cuda.synchronize()
# the full loop: step + commit + resample, GPU-timed
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for k in range(2000):
    gr.step_layers(ids, [p[l] for l in ids], [g[l] for l in ids], 1e-3)
    gr.update_probs()
    ids = gr.sample_layers(k)
e1.record()
torch.cuda.synchronize()
res["loop_us_per_step"] = e0.elapsed_time(e1) / 2000 * 1e3

# the same small update (2 layers x 4096) eager vs one captured CUDA graph
# replayed: launch-bound regime, where graphs pay off
ids = [3, 17]
gs = torch.cuda.Stream()
def eager_steps(n):
    for _ in range(n):
        gr.step_layers(ids, [p[l] for l in ids], [g[l] for l in ids], 1e-3, stream=gs)
with torch.cuda.stream(gs):
    eager_steps(50)
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(gs):
    eager_steps(2000)
torch.cuda.synchronize()
res["eager_step_us_wall"] = (time.perf_counter() - t) / 2000 * 1e6
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    gr.step_layers(ids, [p[l] for l in ids], [g[l] for l in ids], 1e-3, stream=torch.cuda.current_stream())
for _ in range(50):
    graph.replay()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(2000):
    graph.replay()
torch.cuda.synchronize()
res["graph_replay_step_us_wall"] = (time.perf_counter() - t) / 2000 * 1e6
print(json.dumps(res, indent=1))
