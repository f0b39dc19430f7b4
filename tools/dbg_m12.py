import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2604_07808_b200 as G
from synth import layer_grad, layer_params
from oracle import grass_oracle as O
print("lib", G.binding.LIB_PATH)
for dtype in (G.DTYPE_FP32, G.DTYPE_BF16):
    tdt = torch.bfloat16 if dtype == G.DTYPE_BF16 else torch.float32
    numel = [4096 * 12 * 5, 4096 * 12 * 3 + 4096 * 7 + 13, 4096 * 6 * 4 + 5, 3]
    gr = G.Grass(numel, gamma=4, param_dtype=dtype)
    grads = [layer_grad(n, l, 10.0 ** (-l), device="cuda").to(tdt) for l, n in enumerate(numel)]
    gr.mgn_accumulate(list(range(4)), grads)
    k1 = gr.get_mgn()["last_ss"]
    params = [layer_params(n, l, device="cuda").to(tdt) for l, n in enumerate(numel)]
    gr.step_layers([3, 1, 0, 2], [params[3], params[1], params[0], params[2]], [grads[3], grads[1], grads[0], grads[2]], 1e-4)
    k2 = gr.get_mgn()["last_ss"]
    print(dtype, [repr(x) for x in k1], [repr(x) for x in k2], k1 == k2)
    print("exact", [repr(O.sq_norm(g.float().cpu().numpy().astype(np.float64))) for g in grads])
