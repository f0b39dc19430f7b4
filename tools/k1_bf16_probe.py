"""bf16 probing pass (K1, 2 B/param) over the LLaMA-2-7B stack, for ncu:
    python tools/k1_bf16_probe.py            # prints ms per pass
    ncu --set full -k regex:grass_stream_kernel -s 2 -c 1 python tools/k1_bf16_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_07808_b200 as G  # noqa: E402
from synth import MODELS, layer_grad  # noqa: E402

shape = MODELS["llama2-7b"]
n, NL = shape.layer_numel, shape.n_layers
ctx = G.Grass([n] * NL, gamma=2, param_dtype=G.DTYPE_BF16)
g = [layer_grad(n, l, 1e-3, device="cuda").to(torch.bfloat16) for l in range(NL)]
ids = list(range(NL))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(4):
    if i == 3:
        e0.record()
    ctx.mgn_accumulate(ids, g)
e1.record()
torch.cuda.synchronize()
print(f"bf16 probe {e0.elapsed_time(e1):.3f} ms, {2 * n * NL / e0.elapsed_time(e1) / 1e6:.0f} GB/s")
ctx.close()
