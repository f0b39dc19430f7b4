"""Profiling driver for the P2P fused kernel at world 1 (LLaMA-2-7B layers,
gamma = 2): a few grass_step_layers calls on a GRASS_DP_P2P context, for
    ncu --set full -k regex:grass_stream_kernel -c 2 python tools/p2p_profile.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_07808_b200 as G  # noqa: E402
from synth import MODELS, layer_grad, layer_params  # noqa: E402

n_p = MODELS["llama2-7b"].layer_numel
ctx = G.Grass([n_p] * 2, gamma=2, T_p=1, T_s=1, T_u=1, dp_mode=G.DP_P2P)
ctx.p2p_attach([ctx.p2p_exchange_block()[0]])
P = [layer_params(n_p, l, device="cuda") for l in range(2)]
Gr = [layer_grad(n_p, l, 1e-3, device="cuda") for l in range(2)]
for l in range(2):
    ctx.p2p_register_layer(l, [P[l]], [Gr[l]])
for _ in range(4):
    ctx.step_layers([0, 1], P, Gr, 3e-5)
ctx.sync()
print("ok")
