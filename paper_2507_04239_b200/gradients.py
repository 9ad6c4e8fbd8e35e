"""vjp_chunked with the reference's signature (gradients.py:361-483), computed
by the CUDA backward of power_full.  dgates = dlog_g / g (gate gradients need
strictly positive gates, as in the reference gradients.py:9-10)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._convert import back, to_dev
from .attention import AttentionConfig, Mechanism, SequenceBatch
from .errors import InvalidSpec, ShapeMismatch


@dataclass
class GradBundle:
    dq: object
    dk: object
    dv: object
    dgates: object = None


def vjp_chunked(batch: SequenceBatch, cfg: AttentionConfig, plan, upstream) -> GradBundle:
    from .power import power_full

    if cfg.mechanism is not Mechanism.POWER:
        raise InvalidSpec("only the power mechanism has a CUDA backward")
    spec = cfg.expansion   # outputs (and so gradients) do not depend on the kind
    host = batch.on_host
    chunk = None if plan is None else plan.c
    if plan is None and cfg.chunk_size is not None:
        chunk = cfg.chunk_size
    dt = torch.float32 if host or batch.q.dtype == torch.float64 else batch.q.dtype
    q, k, v = (to_dev(x, dt).detach().requires_grad_(True) for x in (batch.q, batch.k, batch.v))
    lg = None
    if batch.gates is not None:
        g = to_dev(batch.gates, torch.float32)
        lg = torch.log(g).detach().requires_grad_(True)
    up = to_dev(upstream, dt)
    if tuple(up.shape) != tuple(batch.v.shape):
        raise ShapeMismatch(f"upstream must match y {tuple(batch.v.shape)}, got {tuple(up.shape)}")
    y = power_full(q, k, v, lg, p=spec.p, chunk_size=chunk, scale=cfg.scale, normalize=cfg.normalize,
                   check_denominator="sync")
    grads = torch.autograd.grad(y, [q, k, v] + ([lg] if lg is not None else []), up)
    dg = None if lg is None else grads[3] / torch.exp(lg.detach())
    f64 = np.float64 if host else None
    return GradBundle(back(grads[0], host, f64), back(grads[1], host, f64), back(grads[2], host, f64),
                      back(dg, host, f64))
