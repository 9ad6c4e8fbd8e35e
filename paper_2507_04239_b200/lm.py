"""A GPT-2-small-geometry language model with power attention (BASELINE
configs[4]: 12 layers, width 768, 12 heads of d=64, MLP x4, ~124M parameters
with the 50257-token embedding tied to the LM head; geometry of the reference's
dense_transformer_params, flops.py:92-94, and the 124M GPT-2 of PAPER.md:240).

Every attention layer is `power_full` (p=2, chunk 1024, log-gated, bf16 on the
tcgen05 kernels).  The dense layers (projections, MLP, LM head) are plain
torch modules and run on cuBLAS under bf16 autocast: they are outside the
power-attention path this package implements.  Data parallelism uses torch
DistributedDataParallel (bucketed NCCL all-reduce overlapped with the
backward); the attention op itself is local to each GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn as nn
import torch.nn.functional as F


@dataclass(frozen=True)
class LMConfig:
    vocab: int = 50257
    width: int = 768
    layers: int = 12
    heads: int = 12
    mlp_ratio: int = 4
    p: int = 2
    chunk: int = 1024
    gate_bias: float = 4.0   # sigmoid(4) = 0.982: a ~55-token half-life at init

    @property
    def head_dim(self) -> int:
        return self.width // self.heads

    @property
    def padded_vocab(self) -> int:
        """Embedding / LM-head rows: the vocabulary rounded up to a multiple of 64
        so the head GEMMs run on the aligned cuBLAS kernels (50257 -> 50304; the
        padded logits are never targets)."""
        return (self.vocab + 63) // 64 * 64


def non_embedding_params(cfg: LMConfig) -> int:
    """(4 + 2 mlp_ratio) width^2 layers (reference flops.py:92-94)."""
    return (4 + 2 * cfg.mlp_ratio) * cfg.width ** 2 * cfg.layers


class PowerAttentionBlock(nn.Module):
    """Pre-norm power-attention sublayer: q, k, v projections, a per-head gate
    (log g = logsigmoid(x w_g + b_g)), power_full, output projection."""

    def __init__(self, cfg: LMConfig, attn_fn=None):
        super().__init__()
        self.cfg = cfg
        self.norm = nn.LayerNorm(cfg.width)
        # separate projections: q, k, v come out contiguous in [b, t, h, d], the
        # layout power_full reads in place (a fused qkv would need three copies)
        self.q = nn.Linear(cfg.width, cfg.width, bias=False)
        self.k = nn.Linear(cfg.width, cfg.width, bias=False)
        self.v = nn.Linear(cfg.width, cfg.width, bias=False)
        self.gate = nn.Linear(cfg.width, cfg.heads)
        self.proj = nn.Linear(cfg.width, cfg.width, bias=False)
        self.attn_fn = attn_fn

    def forward(self, x):
        cfg = self.cfg
        b, t, _ = x.shape
        h = self.norm(x)
        q, k, v = (proj(h).view(b, t, cfg.heads, cfg.head_dim) for proj in (self.q, self.k, self.v))
        log_g = F.logsigmoid(self.gate(h).float())
        if self.attn_fn is None:
            from .power import power_full

            y = power_full(q, k, v, log_g, p=cfg.p, chunk_size=cfg.chunk)
        else:
            y = self.attn_fn(q, k, v, log_g, cfg.p, cfg.chunk)
        return x + self.proj(y.reshape(b, t, cfg.width))


class MLPBlock(nn.Module):
    def __init__(self, cfg: LMConfig):
        super().__init__()
        self.norm = nn.LayerNorm(cfg.width)
        self.up = nn.Linear(cfg.width, cfg.mlp_ratio * cfg.width)
        self.down = nn.Linear(cfg.mlp_ratio * cfg.width, cfg.width)

    def forward(self, x):
        return x + self.down(F.gelu(self.up(self.norm(x)), approximate="tanh"))


class PowerLM(nn.Module):
    """Token ids [b, t] -> next-token logits [b, t, vocab]; no positional
    embedding (the gates give the model its notion of recency)."""

    def __init__(self, cfg: LMConfig = LMConfig(), attn_fn=None):
        super().__init__()
        self.cfg = cfg
        self.embed = nn.Embedding(cfg.padded_vocab, cfg.width)
        self.blocks = nn.ModuleList()
        for _ in range(cfg.layers):
            self.blocks.append(PowerAttentionBlock(cfg, attn_fn))
            self.blocks.append(MLPBlock(cfg))
        self.norm = nn.LayerNorm(cfg.width)
        self.apply(self._init)
        for blk in self.blocks:
            if isinstance(blk, PowerAttentionBlock):
                nn.init.constant_(blk.gate.bias, cfg.gate_bias)

    @staticmethod
    def _init(m):
        if isinstance(m, nn.Linear):
            nn.init.normal_(m.weight, std=0.02)
            if m.bias is not None:
                nn.init.zeros_(m.bias)
        elif isinstance(m, nn.Embedding):
            nn.init.normal_(m.weight, std=0.02)

    def forward(self, tokens):
        x = self.embed(tokens)
        for blk in self.blocks:
            x = blk(x)
        return F.linear(self.norm(x), self.embed.weight)   # LM head tied to the embedding



def lm_loss(model, tokens, targets):
    """Mean next-token cross-entropy; `model` may be DDP-wrapped.  The logits stay
    in the autocast dtype (the softmax accumulates in fp32 inside the kernel)."""
    logits = model(tokens)
    return F.cross_entropy(logits.view(-1, logits.shape[-1]), targets.reshape(-1))


def train_step(model, opt, tokens, targets, autocast=True):
    """One optimizer step: forward, loss, backward (DDP all-reduce overlapped
    when `model` is wrapped), AdamW update.  Returns the loss tensor."""
    with torch.autocast(device_type=tokens.device.type, dtype=torch.bfloat16, enabled=autocast):
        loss = lm_loss(model, tokens, targets)
    loss.backward()
    opt.step()
    opt.zero_grad(set_to_none=True)
    return loss.detach()


def attention_flops(cfg: LMConfig, t: int, b: int = 1) -> float:
    """Algorithmic FLOPs of the attention ops of one fwd+bwd step (SURVEY 8d
    convention: contractions only, bwd = 2 fwd)."""
    import math

    d = cfg.head_dim
    D = math.comb(d + cfg.p - 1, cfg.p)
    c = min(cfg.chunk, t)
    n = t // c
    intra = n * c * (c + 1) // 2 * 2 * d
    state = (2 * t - c) * D * d
    return 3 * 2 * b * cfg.heads * cfg.layers * (intra + state)


def weight_flops(cfg: LMConfig, tokens: int) -> float:
    """6 N tokens for the dense weights (non-embedding + the tied LM head)."""
    return 6.0 * (non_embedding_params(cfg) + cfg.padded_vocab * cfg.width) * tokens
