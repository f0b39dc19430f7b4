"""Small end-to-end exercise of every kernel variant and path, for
compute-sanitizer (one tool per run): K1/K2 fp32 + bf16, ragged tails, offload
(step + period), 1-rank NCCL path, clipping."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_07808_b200 as G  # noqa: E402
from synth import layer_grad, layer_params  # noqa: E402

dev = "cuda:0"
numel = [4096 * 6 + 3, 65_536 + 8, 5, 4096 * 25]
for dtype in (G.DTYPE_FP32, G.DTYPE_BF16):
    tdt = torch.float32 if dtype == G.DTYPE_FP32 else torch.bfloat16
    for kw in ({}, {"offload": True, "chunk_elems": 8192},
               {"offload": True, "chunk_elems": 8192, "residency": G.RESIDENCY_PERIOD},
               {"force_nccl": True} if dtype == G.DTYPE_FP32 else {"max_grad_norm": 1e-3},
               {"max_grad_norm": 1e-3}):
        n = [x + (x % 8 and 8 - x % 8) for x in numel] if kw.get("force_nccl") else numel
        gr = G.Grass(n, gamma=2, param_dtype=dtype, **kw)
        p = [layer_params(k, l, device=dev).to(tdt) for l, k in enumerate(n)]
        gr.mgn_accumulate([0, 1, 2, 3], [layer_grad(k, l, 1e-3, device=dev).to(tdt) for l, k in enumerate(n)])
        gr.update_probs()
        for step, ids in enumerate([[0, 1], [2, 3], [3, 1], [0, 2]]):
            gr.step_layers(ids, [p[l] for l in ids], [layer_grad(n[l], l, 1e-3, step=step, device=dev).to(tdt)
                                                       for l in ids], 1e-3)
        gr.sync()
        gr.close()
torch.cuda.synchronize()
print("sanitize case ok")
