"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

Holds NONE of the method's arithmetic (no norms, no softmax, no sampling, no
AdamW): only layer shapes and seeded random tensors, so both the oracle and the
CUDA path can be fed the same inputs.  Recipe:

* Layout: one flat fp32 buffer per decoder block, HF LLaMA order
  q, k, v, o, gate, up, down, input_norm, post_attention_norm.
* theta ~ N(0, 0.02^2) (SPEC.md:148 init std), the two RMSNorm weights = 1.0.
* g_l ~ N(0, sigma_l^2), sigma_l log-uniform in [1e-5, 1e-3] per layer, drawn
  from the data seed (per-layer MGN spread like PAPER.md:96 / Fig. 1).
* m = v = 0 at t = 0 (fresh optimizer state).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_ff: int

    @property
    def pieces(self):
        d, hd = self.d_model, self.d_model // self.n_heads
        kv = self.n_kv_heads * hd
        return [("q", d * d), ("k", d * kv), ("v", d * kv), ("o", d * d),
                ("gate", d * self.d_ff), ("up", d * self.d_ff), ("down", self.d_ff * d),
                ("input_norm", d), ("post_attention_norm", d)]

    @property
    def layer_numel(self) -> int:
        return sum(n for _, n in self.pieces)

    @property
    def norm_numel(self) -> int:
        return 2 * self.d_model


MODELS = {
    "llama2-7b": ModelShape("llama2-7b", 32, 4096, 32, 32, 11008),
    "llama3-8b": ModelShape("llama3-8b", 32, 4096, 32, 8, 14336),
    "llama2-13b": ModelShape("llama2-13b", 40, 5120, 40, 40, 13824),
    # a small stack with the same block layout: bench.py's legs exercised in seconds (tests/test_gpu_bench.py)
    "tiny-bench": ModelShape("tiny-bench", 8, 256, 4, 4, 688),
}

TINY_NUMEL = 65_536
TINY_LAYERS = 4


def _gen(device, *key) -> torch.Generator:
    s = 0
    for k in key:
        s = (s * 1_000_003 + int(k) + 1) & ((1 << 63) - 1)
    g = torch.Generator(device=device)
    g.manual_seed(s)
    return g


def grad_sigmas(n_layers: int, seed: int = 0):
    """Per-layer gradient std, log-uniform in [1e-5, 1e-3]."""
    g = _gen("cpu", seed, 7, n_layers)
    u = torch.rand(n_layers, generator=g, dtype=torch.float64)
    return [10.0 ** (-5.0 + 2.0 * float(x)) for x in u]


def layer_params(numel: int, layer: int, seed: int = 0, device="cpu", norm_numel: int = 0):
    """theta ~ N(0, 0.02^2), trailing `norm_numel` entries (RMSNorm weights) = 1."""
    g = _gen(device, seed, 1, layer)
    t = torch.randn(numel, generator=g, device=device, dtype=torch.float32)
    t.mul_(0.02)
    if norm_numel:
        t[numel - norm_numel:] = 1.0
    return t


def layer_grad(numel: int, layer: int, sigma: float, step: int = 0, seed: int = 0,
               device="cpu", rank: int = 0):
    g = _gen(device, seed, 2, layer, step, rank)
    t = torch.randn(numel, generator=g, device=device, dtype=torch.float32)
    t.mul_(sigma)
    return t


def integer_grad(numel: int, layer: int, lo: int = -3, hi: int = 3, seed: int = 0, device="cpu"):
    """Integer-valued gradients: their squared norm is an exact integer."""
    g = _gen(device, seed, 3, layer)
    return torch.randint(lo, hi + 1, (numel,), generator=g, device=device).to(torch.float32)


def random_probs(n: int, seed: int):
    g = _gen("cpu", seed, 4, n)
    x = torch.rand(n, generator=g, dtype=torch.float64) + 1e-3
    x = x / x.sum()
    return [float(v) for v in x]


def random_mgn(n: int, seed: int):
    g = _gen("cpu", seed, 5, n)
    return [float(v) for v in (torch.rand(n, generator=g, dtype=torch.float64) * 1e-3)]


def tiny_numels():
    return [TINY_NUMEL] * TINY_LAYERS


def human_bytes(b: float) -> str:
    for u in ("B", "KB", "MB", "GB", "TB"):
        if abs(b) < 1000:
            return f"{b:.2f} {u}"
        b /= 1000
    return f"{b:.2f} PB"


__all__ = ["ModelShape", "MODELS", "grad_sigmas", "layer_params", "layer_grad",
           "integer_grad", "random_probs", "random_mgn", "tiny_numels", "TINY_NUMEL",
           "TINY_LAYERS", "human_bytes"]
