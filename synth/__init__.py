"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no amax, scale, codec, reduction or
Adam): only tensor shapes and random numbers.  It is the one module that both the
CUDA path's callers and the oracle's callers import (task rule ③).

Shapes — the synthetic gradient sets of SURVEY.md §8(d): GPT models of PAPER.md
Table 1 (d/L = 768/12, 4096/32, 5120/40, 12288/96), RoPE so no position
table, Megatron-style bias + LayerNorm layout, tied embedding with the
vocabulary padded to V = 50304 (an assumption; the paper does not state V).

Values — per (step, tensor, rank):
    g = a_t * (rho * z_common + sqrt(1 - rho^2) * z_rank),   z ~ Student-t(nu = 3)
with a_t log-uniform in [1e-6, 1e-2] per tensor ("typically small gradient values",
P:166) and rho = 0.5 cross-rank correlation, so post-scaling sums overflow
and the auto-scaling factor mu is exercised.  Heavy tails make
amax/rms >> 1 as real gradients do.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Tuple

import torch

VOCAB_PADDED = 50304

GPT_CONFIGS = {
    # name: (d_model, n_layers)   PAPER.md Table 1
    "gpt-125m": (768, 12),
    "gpt-7b": (4096, 32),
    "gpt-13b": (5120, 40),
    "gpt-175b": (12288, 96),
}


@dataclass(frozen=True)
class TensorSpec:
    name: str
    shape: Tuple[int, ...]

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n


def gpt_gradient_set(model: str, n_layers: int | None = None) -> List[TensorSpec]:
    """Per-parameter gradient tensors of a Megatron-style GPT.

    ``n_layers`` overrides the layer count (used for GPT-175B per-layer slices).
    Order: tied embedding, then per layer ln1.{w,b}, qkv.{w,b}, proj.{w,b},
    ln2.{w,b}, fc1.{w,b}, fc2.{w,b}, then the final LayerNorm lnf.{w,b}.
    """
    d, L = GPT_CONFIGS[model]
    if n_layers is not None:
        L = n_layers
    specs = [TensorSpec("emb.w", (VOCAB_PADDED, d))]
    for l in range(L):
        p = f"layer{l}."
        specs += [
            TensorSpec(p + "ln1.w", (d,)), TensorSpec(p + "ln1.b", (d,)),
            TensorSpec(p + "qkv.w", (3 * d, d)), TensorSpec(p + "qkv.b", (3 * d,)),
            TensorSpec(p + "proj.w", (d, d)), TensorSpec(p + "proj.b", (d,)),
            TensorSpec(p + "ln2.w", (d,)), TensorSpec(p + "ln2.b", (d,)),
            TensorSpec(p + "fc1.w", (4 * d, d)), TensorSpec(p + "fc1.b", (4 * d,)),
            TensorSpec(p + "fc2.w", (d, 4 * d)), TensorSpec(p + "fc2.b", (d,)),
        ]
    specs += [TensorSpec("lnf.w", (d,)), TensorSpec("lnf.b", (d,))]
    return specs


def square_set(n: int = 4096) -> List[TensorSpec]:
    """Config C1: one n x n fp32 gradient tensor (BASELINE.json configs[0])."""
    return [TensorSpec("w", (n, n))]


# ---------------------------------------------------------------- seeds
SEED_BASE = 0x5EED0000


def common_seed(step: int, t: int) -> int:
    return SEED_BASE + 1000003 * step + 1009 * t


def rank_seed(step: int, t: int, rank: int) -> int:
    return common_seed(step, t) + 7919 * (rank + 1)


def amplitude(t: int, lo: float = 1e-6, hi: float = 1e-2) -> float:
    """a_t, log-uniform in [lo, hi], a function of the tensor index only."""
    g = torch.Generator(device="cpu")
    g.manual_seed(0xA11CE + 31 * t)
    u = torch.rand((), generator=g, dtype=torch.float64).item()
    return math.exp(math.log(lo) + u * (math.log(hi) - math.log(lo)))


def _student_t3(n: int, seed: int, device) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn((4, n), generator=g, device=device, dtype=torch.float32)
    chi2 = x[1] * x[1] + x[2] * x[2] + x[3] * x[3]
    return x[0] / torch.sqrt(chi2 / 3.0)


def fill_gradient(out: torch.Tensor, step: int, t: int, rank: int, rho: float = 0.5,
                  amp: float | None = None) -> torch.Tensor:
    """Write the synthetic gradient of (step, tensor t, rank) into ``out`` (fp32 or bf16)."""
    n = out.numel()
    dev = out.device
    a = amplitude(t) if amp is None else amp
    zc = _student_t3(n, common_seed(step, t), dev)
    zr = _student_t3(n, rank_seed(step, t, rank), dev)
    g = a * (rho * zc + math.sqrt(1.0 - rho * rho) * zr)
    out.view(-1).copy_(g.to(out.dtype))
    return out


def fill_weights(out: torch.Tensor, t: int, std: float = 0.02) -> torch.Tensor:
    """Initial FP32 master weights: N(0, std^2) for every tensor (GPT-style init)."""
    g = torch.Generator(device=out.device)
    g.manual_seed(0x3E1647 + 131 * t)
    w = torch.randn(out.numel(), generator=g, device=out.device, dtype=torch.float32) * std
    out.view(-1).copy_(w.to(out.dtype))
    return out


def uniform_codes(n: int, seed: int, device="cpu") -> torch.Tensor:
    """Random bytes (e.g. pre-quantized FP8 codes for a collective sweep)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randint(0, 256, (n,), generator=g, device=device, dtype=torch.uint8)
