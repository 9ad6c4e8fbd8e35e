"""Reference-shaped types and the attention form (reference attention.py).

Only the power mechanism is on the CUDA path (SURVEY §2 rows 2b are out of
scope); other mechanisms raise InvalidSpec."""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from ._convert import back, to_dev
from .errors import InvalidSpec, NonFiniteInput, OddPowerWithNormalize, ShapeMismatch
from .expansions import ExpansionSpec


class Mechanism(str, Enum):
    EXP = "exp"
    WINDOW = "window"
    LINEAR = "linear"
    POWER = "power"


def _np(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


@dataclass
class SequenceBatch:
    """q, k [b, t, h, d]; v [b, t, h, e]; gates [b, t, h] in [0, 1] or None
    (attention.py:45-103).  Arrays may be numpy or torch tensors."""

    q: object
    k: object
    v: object
    gates: object = None

    def __post_init__(self):
        for name in ("q", "k", "v"):
            a = getattr(self, name)
            if a.ndim != 4:
                raise ShapeMismatch(f"{name} must be [b, t, h, feature], got {tuple(a.shape)}")
            finite = torch.isfinite(a).all().item() if isinstance(a, torch.Tensor) else np.isfinite(a).all()
            if not finite:
                raise NonFiniteInput(f"{name} contains non-finite values")
        if tuple(self.k.shape) != tuple(self.q.shape):
            raise ShapeMismatch(f"k shape {tuple(self.k.shape)} != q shape {tuple(self.q.shape)}")
        if tuple(self.v.shape[:3]) != tuple(self.q.shape[:3]):
            raise ShapeMismatch("v disagrees with q on [b, t, h]")
        if self.gates is not None:
            g = self.gates
            if tuple(g.shape) != tuple(self.q.shape[:3]):
                raise ShapeMismatch(f"gates shape {tuple(g.shape)} != [b, t, h]")
            gn = _np(g)
            if not np.isfinite(gn).all():
                raise NonFiniteInput("gates contain non-finite values")
            if (gn < 0).any() or (gn > 1).any():
                raise InvalidSpec("gates must lie in [0, 1]")

    b = property(lambda s: s.q.shape[0])
    t = property(lambda s: s.q.shape[1])
    h = property(lambda s: s.q.shape[2])
    d = property(lambda s: s.q.shape[3])
    v_dim = property(lambda s: s.v.shape[3])

    @property
    def on_host(self) -> bool:
        return not isinstance(self.q, torch.Tensor)


@dataclass(frozen=True)
class AttentionConfig:
    """attention.py:106-171 (power / linear mechanisms carry a SPOW spec)."""

    mechanism: Mechanism
    expansion: ExpansionSpec | None = None
    window: int | None = None
    chunk_size: int | None = None
    scale: float | None = None
    normalize: bool = False
    use_log_space: bool = False
    epsilon: float | None = None

    def __post_init__(self):
        object.__setattr__(self, "mechanism", Mechanism(self.mechanism))
        if self.mechanism in (Mechanism.LINEAR, Mechanism.POWER) and self.expansion is None:
            raise InvalidSpec(f"{self.mechanism.value} mechanism needs an ExpansionSpec")
        if self.mechanism is Mechanism.POWER:
            if self.normalize and self.p % 2:
                raise OddPowerWithNormalize(f"normalization needs positive scores: p={self.p} must be even")
            if self.use_log_space and self.p % 2:
                raise InvalidSpec(f"log-space scoring needs even p, got p={self.p}")
        if self.chunk_size is not None and self.chunk_size < 1:
            raise InvalidSpec(f"chunk_size must be >= 1, got {self.chunk_size}")

    @property
    def p(self) -> int:
        if self.expansion is None:
            raise InvalidSpec(f"{self.mechanism.value} mechanism has no power degree")
        return self.expansion.p

    def scale_for(self, d: int) -> float:
        return 1.0 / math.sqrt(d) if self.scale is None else self.scale

    @classmethod
    def power(cls, expansion: ExpansionSpec, **kw) -> "AttentionConfig":
        return cls(Mechanism.POWER, expansion=expansion, **kw)


@dataclass
class AttentionOutput:
    """y [b, t, h, e]; rowsum [b, t, h] (attention.py:174-179)."""

    y: object
    rowsum: object = None


def run_power(batch: SequenceBatch, cfg: AttentionConfig, chunk: int | None) -> AttentionOutput:
    """Shared body of the attention and chunked forms: one power_full call."""
    from .power import power_full_with_rowsum

    if cfg.mechanism is not Mechanism.POWER:
        raise InvalidSpec(f"only the power mechanism runs on the CUDA path, got {cfg.mechanism.value}")
    # every expansion kind gives <phi(x), phi(y)> = (x . y)^p (expansions.py:3-5):
    # the output does not depend on the kind
    spec = cfg.expansion
    if spec.d != batch.d:
        raise ShapeMismatch(f"spec.d={spec.d} but q has d={batch.d}")
    host = batch.on_host
    np_dt = np.result_type(_np(batch.q).dtype, _np(batch.v).dtype) if host else None
    src_dt = batch.q.dtype if not host else None
    tdt = torch.float32 if host or src_dt == torch.float64 else src_dt
    q, k, v = (to_dev(x, tdt) for x in (batch.q, batch.k, batch.v))
    lg = None if batch.gates is None else torch.log(to_dev(batch.gates, torch.float32))
    y, rs = power_full_with_rowsum(q, k, v, lg, p=spec.p, chunk_size=chunk, scale=cfg.scale,
                                   normalize=cfg.normalize, check_denominator="sync")
    if not host and src_dt == torch.float64:
        y = y.to(torch.float64)
    return AttentionOutput(back(y, host, np_dt), back(rs, host, np_dt))


def power_attention_form(batch: SequenceBatch, cfg: AttentionConfig) -> AttentionOutput:
    """Quadratic form (attention.py:273-309): one chunk spanning the sequence."""
    if cfg.use_log_space:
        return run_log_space(batch, cfg)
    return run_power(batch, cfg, None)


def run_log_space(batch: SequenceBatch, cfg: AttentionConfig) -> AttentionOutput:
    """attention.py:289-305: the stabilised scores p*log(|s|+eps) + log-decay,
    row-max shifted (pa_power_logspace_fwd).  f64 inputs compute in f64, f32 in
    f32, half types in f32; eps = cfg.epsilon_for(dtype) (attention.py:152-155)."""
    from .power import power_logspace_forward

    if cfg.mechanism is not Mechanism.POWER:
        raise InvalidSpec(f"only the power mechanism runs on the CUDA path, got {cfg.mechanism.value}")
    # every expansion kind gives <phi(x), phi(y)> = (x . y)^p (expansions.py:3-5):
    # the output does not depend on the kind
    spec = cfg.expansion
    if spec.d != batch.d:
        raise ShapeMismatch(f"spec.d={spec.d} but q has d={batch.d}")
    host = batch.on_host
    if host:
        np_dt = np.result_type(_np(batch.q).dtype, _np(batch.v).dtype)
        tdt = torch.float64 if np_dt == np.float64 else torch.float32
    else:
        np_dt = None
        tdt = torch.float64 if batch.q.dtype == torch.float64 else torch.float32
    q, k, v = (to_dev(x, tdt) for x in (batch.q, batch.k, batch.v))
    lg = None
    if batch.gates is not None:
        g = to_dev(batch.gates, tdt)
        lg = torch.log(g)  # -inf for zero gates: handled exactly by the kernel
    eps = cfg.epsilon if cfg.epsilon is not None else (1e-12 if tdt == torch.float64 else 1e-7)
    y, rs = power_logspace_forward(q, k, v, lg, p=spec.p, scale=cfg.scale, normalize=cfg.normalize,
                                   eps=eps)
    if not host and batch.q.dtype not in (torch.float32, torch.float64):
        y = y.to(batch.q.dtype)
    return AttentionOutput(back(y, host, np_dt), back(rs, host, np_dt))


def attention(batch: SequenceBatch, cfg: AttentionConfig) -> AttentionOutput:
    """attention.py:341-343 for the power mechanism."""
    return power_attention_form(batch, cfg)
