"""Synthetic workloads the FSDP runtime is measured on (BASELINE.json configs).

GPT-style decoder (GPT-2 layout: learned positions, pre-LN blocks with
biases, tied LM head).  The root unit holds wte/wpe/ln_f (tied head inside
one unit, so no SharedParameterError); every Block is a unit
(transformer-block auto-wrap).  Shapes reproduce SURVEY §8:
  tiny     d=256  L=2  V=1024  S=128  -> root psi 295,424, block psi 789,760
  gpt1.3b  d=2048 L=24 V=50304 S=2048 -> N = 1,315,819,520, block 50,358,272
  gpt30b   d=7168 L=48 V=50304 S=2048 -> N = 29,974,755,328, block 616,655,872
Model compute (GEMMs, attention) is ordinary torch (cuBLAS / SDPA): the
FSDP hot path this repo builds is everything around it.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn as nn
import torch.nn.functional as F


@dataclass(frozen=True)
class GPTConfig:
    name: str
    d: int
    layers: int
    vocab: int
    seq: int
    heads: int

    @property
    def block_params(self) -> int:
        return 12 * self.d * self.d + 13 * self.d

    @property
    def root_params(self) -> int:
        return (self.vocab + self.seq) * self.d + 2 * self.d

    @property
    def n_params(self) -> int:
        return self.layers * self.block_params + self.root_params

    def flops_per_token(self, seq: int | None = None) -> float:
        """6·N_nonembed + 12·L·d·S + 6·V·d (fwd+bwd); `seq`
        overrides S for samples run at a shorter sequence length."""
        s = self.seq if seq is None else seq
        return (6.0 * self.layers * self.block_params + 12.0 * self.layers * self.d * s
                + 6.0 * self.vocab * self.d)


CONFIGS = {
    "tiny": GPTConfig("tiny", 256, 2, 1024, 128, 4),
    "gpt1.3b": GPTConfig("gpt1.3b", 2048, 24, 50304, 2048, 16),
    "gpt30b": GPTConfig("gpt30b", 7168, 48, 50304, 2048, 56),
    # depth-reduced same-width variants (single-GPU references)
    "gpt1.3b-l4": GPTConfig("gpt1.3b-l4", 2048, 4, 50304, 2048, 16),
}


class Attention(nn.Module):
    def __init__(self, d: int, heads: int):
        super().__init__()
        self.c_attn = nn.Linear(d, 3 * d)
        self.c_proj = nn.Linear(d, d)
        self.heads = heads

    def forward(self, x):
        b, s, d = x.shape
        q, k, v = self.c_attn(x).split(d, dim=2)
        h = self.heads
        q = q.view(b, s, h, d // h).transpose(1, 2)
        k = k.view(b, s, h, d // h).transpose(1, 2)
        v = v.view(b, s, h, d // h).transpose(1, 2)
        y = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        return self.c_proj(y.transpose(1, 2).reshape(b, s, d))


class MLP(nn.Module):
    def __init__(self, d: int):
        super().__init__()
        self.c_fc = nn.Linear(d, 4 * d)
        self.c_proj = nn.Linear(4 * d, d)

    def forward(self, x):
        return self.c_proj(F.gelu(self.c_fc(x), approximate="tanh"))


class Block(nn.Module):
    def __init__(self, d: int, heads: int):
        super().__init__()
        self.ln_1 = nn.LayerNorm(d)
        self.attn = Attention(d, heads)
        self.ln_2 = nn.LayerNorm(d)
        self.mlp = MLP(d)

    def forward(self, x):
        x = x + self.attn(self.ln_1(x))
        return x + self.mlp(self.ln_2(x))


class GPT(nn.Module):
    def __init__(self, cfg: GPTConfig):
        super().__init__()
        self.cfg = cfg
        self.wte = nn.Embedding(cfg.vocab, cfg.d)
        self.wpe = nn.Embedding(cfg.seq, cfg.d)
        self.h = nn.ModuleList([Block(cfg.d, cfg.heads) for _ in range(cfg.layers)])
        self.ln_f = nn.LayerNorm(cfg.d)

    def forward(self, idx, targets=None):
        b, s = idx.shape
        pos = torch.arange(s, device=idx.device)
        x = self.wte(idx) + self.wpe(pos)
        for blk in self.h:
            x = blk(x)
        x = self.ln_f(x)
        logits = F.linear(x, self.wte.weight)           # tied head
        if targets is None:
            return logits
        return F.cross_entropy(logits.float().view(-1, logits.size(-1)), targets.view(-1))


def init_gpt_(model: GPT, seed: int = 0) -> GPT:
    """GPT-2 style init (normal 0.02, scaled residual projections)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    L = model.cfg.layers
    for name, p in model.named_parameters():
        with torch.no_grad():
            if name.endswith("bias"):
                p.zero_()
            elif "ln" in name:
                p.fill_(1.0)
            else:
                std = 0.02 / math.sqrt(2 * L) if name.endswith("c_proj.weight") else 0.02
                p.copy_(torch.randn(p.shape, generator=g) * std)
    return model


def param_init_fn(module: nn.Module) -> None:
    """Deferred (meta-device) per-module init used for models too large to
    build unsharded: deterministic, device-side."""
    with torch.no_grad():
        for name, p in module.named_parameters(recurse=False):
            if name == "bias":
                p.zero_()
            elif isinstance(module, nn.LayerNorm):
                p.fill_(1.0)
            else:
                p.normal_(0.0, 0.02)


def synthetic_batch(cfg: GPTConfig, batch: int, seed: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    """Token ids uniform over [0, V) from a fixed seed."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randint(0, cfg.vocab, (batch, cfg.seq), generator=g)
    y = torch.randint(0, cfg.vocab, (batch, cfg.seq), generator=g)
    return x.to(device), y.to(device)
