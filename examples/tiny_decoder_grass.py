"""Training a tiny decoder-only transformer with GRASS through libgrass.

What the caller does (the library's boundary, include/grass.h), here through
paper_2604_07808_b200.GrassBlocks:
  * each decoder block's parameters live in ONE flat fp32 buffer (the
    parameters are views into it), and so do their gradients;
  * the schedule (GrassSchedule) says which blocks need gradients; the other
    blocks are frozen (requires_grad False);
  * after backward, the flat gradient buffers go to the library: probing
    steps only record the Eq. 2 norms, later steps run the fused norm + AdamW
    of the trainable blocks (optimizer states offloaded to pinned host memory
    with period residency);
  * the embeddings and the output head are always trainable (LISA convention,
    SPEC.md:145): one more flat buffer, registered as an always-active group
    (n_always = 1, DESIGN R19) — never sampled, updated by the same fused
    kernel every adaptive step, its m/v kept in HBM.

    python examples/tiny_decoder_grass.py
"""
from __future__ import annotations

import os
import sys

import torch
import torch.nn as nn

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_07808_b200 as G  # noqa: E402


class Block(nn.Module):
    def __init__(self, d, heads):
        super().__init__()
        self.n1 = nn.LayerNorm(d)
        self.attn = nn.MultiheadAttention(d, heads, batch_first=True)
        self.n2 = nn.LayerNorm(d)
        self.mlp = nn.Sequential(nn.Linear(d, 4 * d), nn.GELU(), nn.Linear(4 * d, d))

    def forward(self, x, mask):
        h = self.n1(x)
        x = x + self.attn(h, h, h, attn_mask=mask, need_weights=False)[0]
        return x + self.mlp(self.n2(x))


class TinyDecoder(nn.Module):
    def __init__(self, vocab=256, d=128, heads=4, layers=6, ctx=64):
        super().__init__()
        self.emb = nn.Embedding(vocab, d)
        self.pos = nn.Parameter(torch.zeros(ctx, d))
        self.blocks = nn.ModuleList(Block(d, heads) for _ in range(layers))
        self.head = nn.Linear(d, vocab)

    def forward(self, idx):
        t = idx.shape[1]
        mask = torch.triu(torch.full((t, t), float("-inf"), device=idx.device), 1)
        x = self.emb(idx) + self.pos[:t]
        for b in self.blocks:
            x = b(x, mask)
        return self.head(x)


def train(steps=60, T_p=5, T_s=5, gamma=2, seed=0, device="cuda", log=True, dtype=torch.float32,
          graphs=False, step_graphs=False):
    """graphs: the library update of each period is one captured CUDA graph;
    step_graphs: the whole step (forward, backward, update) is, through
    GrassBlocks.train_step."""
    torch.manual_seed(seed)
    model = TinyDecoder().to(device=device, dtype=dtype)   # bf16: fp32 master + m + v in libgrass
    gb = G.GrassBlocks(model.blocks, always=[[model.emb.weight, model.pos, *model.head.parameters()]],
                       gamma=gamma, T_p=T_p, T_s=T_s, seed=seed, offload=True,
                       residency=G.RESIDENCY_PERIOD, graphs=graphs, step_graphs=step_graphs)
    # a learnable synthetic task: predict the next token of a fixed random walk
    data = torch.cumsum(torch.randint(-2, 3, (64, 65), generator=torch.Generator().manual_seed(seed)), 1) % 256
    data = data.to(device)
    losses = []
    def loss_fn():                     # reads the static batch `data`
        logits = model(data[:, :-1])
        return nn.functional.cross_entropy(logits.float().reshape(-1, 256), data[:, 1:].reshape(-1))

    for step in range(steps):
        if step_graphs:
            loss = gb.train_step(step, loss_fn, lr=1e-3)
            ids = gb.layers
        else:
            ids = gb.begin_step(step)      # freezes the blocks that are not trained this step
            loss = loss_fn()
            loss.backward()
            # probing steps only record norms: no parameter update
            gb.end_step(step, lr=1e-3)
            gb.zero_grad()
        losses.append(float(loss.detach()))
        if log and step % 10 == 0:
            print(f"step {step:3d} loss {losses[-1]:.4f} trainable {ids if step >= T_p else 'none (probe)'}")
    gb.grass.sync()
    return losses


if __name__ == "__main__":
    train()
