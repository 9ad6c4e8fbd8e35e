"""Chunked form and per-chunk operators with the reference's names and argument
meaning (reference chunked.py).  The pipeline itself runs in the CUDA library
(one pa_power_full_fwd call); the per-chunk ops bind the C ABI one by one."""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from .attention import (AttentionConfig, AttentionOutput, Mechanism, SequenceBatch,
                        power_attention_form, run_power)
from .errors import InvalidSpec, ShapeMismatch, StateTooLarge, ZeroDenominator
from .expansions import ExpansionSpec, expansion_dim
from .kernels import discumsum_kernel, query_state_kernel, update_state_kernel

DEFAULT_STATE_BUDGET = 2**31


def _xp(x):
    return torch if isinstance(x, torch.Tensor) else np


@dataclass
class ChunkState:
    """[D, e] state and [D] key_sum of one stream (chunked.py:40-63)."""

    s: object
    key_sum: object
    spec: ExpansionSpec

    def __post_init__(self):
        dim = expansion_dim(self.spec)
        if self.s.ndim != 2 or self.s.shape[0] != dim:
            raise ShapeMismatch(f"state must be [D={dim}, v], got {tuple(self.s.shape)}")
        if tuple(self.key_sum.shape) != (dim,):
            raise ShapeMismatch(f"key_sum must be [D={dim}], got {tuple(self.key_sum.shape)}")

    @classmethod
    def zeros(cls, spec, v_dim, dtype=np.float64):
        dim = expansion_dim(spec)
        return cls(np.zeros((dim, v_dim), dtype=dtype), np.zeros(dim, dtype=dtype), spec)


@dataclass(frozen=True)
class ChunkPlan:
    """ceil(t/c) chunks, the last possibly short (chunked.py:66-86)."""

    t: int
    c: int

    def __post_init__(self):
        if self.t < 1 or self.c < 1:
            raise InvalidSpec(f"need t >= 1 and c >= 1, got t={self.t}, c={self.c}")

    @property
    def n_chunks(self) -> int:
        return -(-self.t // self.c)

    @property
    def last_chunk_len(self) -> int:
        return self.t - (self.n_chunks - 1) * self.c

    def bounds(self):
        return [(s, min(s + self.c, self.t)) for s in range(0, self.t, self.c)]


def _suffix_products(g):
    xp = _xp(g)
    out = xp.ones_like(g)
    if g.shape[-1] > 1:
        rev = xp.flip(g, (-1,)) if xp is torch else g[..., ::-1]
        cp = xp.cumprod(rev, -1) if xp is torch else np.cumprod(rev, axis=-1)
        cp = xp.flip(cp, (-1,)) if xp is torch else cp[..., ::-1]
        out[..., :-1] = cp[..., 1:]
    return out


def _prefix_products(g):
    return torch.cumprod(g, -1) if isinstance(g, torch.Tensor) else np.cumprod(g, axis=-1)


def check_state_budget(spec, v_dim, streams, itemsize, budget):
    dim = expansion_dim(spec)
    nbytes = dim * (v_dim + 1) * streams * itemsize
    if nbytes > budget:
        raise StateTooLarge(f"state of {nbytes} bytes (D={dim}, v={v_dim}, streams={streams}) "
                            f"exceeds the budget of {budget} bytes")
    return dim


def update_state(spec, k_chunk, v_chunk, gates_chunk=None, backend=None):
    """(ChunkState, lam) for one stream's chunk (chunked.py:123-153)."""
    if k_chunk.ndim != 2 or v_chunk.ndim != 2 or k_chunk.shape[0] != v_chunk.shape[0]:
        raise ShapeMismatch(f"chunk arrays must be [c, d]/[c, v], got {tuple(k_chunk.shape)}, {tuple(v_chunk.shape)}")
    if k_chunk.shape[1] != spec.d:
        raise ShapeMismatch(f"keys have dim {k_chunk.shape[1]}, spec.d={spec.d}")
    if gates_chunk is None:
        decay, lam = None, 1.0
    else:
        if tuple(gates_chunk.shape) != (k_chunk.shape[0],):
            raise ShapeMismatch(f"gates must be [c], got {tuple(gates_chunk.shape)}")
        decay = _suffix_products(gates_chunk)[None]
        lam = float(gates_chunk.prod())
    s, ks = update_state_kernel(k_chunk[None], v_chunk[None], decay, spec, backend=backend)
    return ChunkState(s[0], ks[0], spec), lam


def discumsum(values, lambdas):
    """Discounted cumulative sum along axis 0 on the device, bit-exact with the
    sequential loop (chunked.py:156-176)."""
    return discumsum_kernel(values, lambdas)


def discumsum_states(states, lambdas):
    if not states:
        return []
    xp = _xp(states[0].s)
    spec = states[0].spec
    s = discumsum(xp.stack([st.s for st in states]), lambdas)
    ks = discumsum(xp.stack([st.key_sum for st in states]), lambdas)
    return [ChunkState(s[k], ks[k], spec) for k in range(len(states))]


def query_state(state, q_chunk, y_attn=None, zeta=None, gates_prefix=None, scale=None,
                normalize=False, backend=None):
    """chunked.py:189-232: combine the carried state with the intra-chunk output."""
    if q_chunk.ndim != 2 or q_chunk.shape[1] != state.spec.d:
        raise ShapeMismatch(f"queries must be [c, d={state.spec.d}], got {tuple(q_chunk.shape)}")
    c = q_chunk.shape[0]
    if scale is None:
        scale = 1.0 / math.sqrt(state.spec.d)
    ys, den = query_state_kernel(scale * q_chunk[None], state.s[None], state.key_sum[None],
                                 state.spec, backend=backend)
    ys, den = ys[0], den[0]
    if gates_prefix is not None:
        if tuple(gates_prefix.shape) != (c,):
            raise ShapeMismatch(f"gates_prefix must be [c], got {tuple(gates_prefix.shape)}")
        ys = ys * gates_prefix[:, None]
        den = den * gates_prefix
    out = ys if y_attn is None else y_attn + ys
    if normalize:
        total = den if zeta is None else zeta + den
        if bool((total <= 0).any()):
            raise ZeroDenominator("zeta + phi(q) . key_sum is not positive (odd degree or all-zero inputs?)")
        out = out / total[:, None]
    return out


def chunked_power_attention(batch: SequenceBatch, cfg: AttentionConfig, plan: ChunkPlan | None = None,
                            state_budget: int = DEFAULT_STATE_BUDGET, backend=None, op_timer=None):
    """chunked.py:287-413 as one CUDA pipeline call.  op_timer (if given)
    accumulates wall ns of the whole fused pipeline under "power_full".

    cfg.use_log_space: the reference threads it into the intra-chunk config
    (chunked.py:323, 336 -> attention.py:289-305); that call runs the
    reference's operator loop on the GPU operators instead (_chunked_log_space:
    the stabilised intra-chunk kernel per chunk, update_state / discumsum /
    query_state kernels), so the eps of p log(|s| + eps) enters as it does in
    the reference."""
    if cfg.mechanism not in (Mechanism.POWER, Mechanism.LINEAR) or cfg.expansion is None:
        raise InvalidSpec(f"{cfg.mechanism.value} mechanism has no feature expansion")
    spec = cfg.expansion
    if plan is None:
        if cfg.chunk_size is None:
            raise InvalidSpec("chunked form needs a ChunkPlan or cfg.chunk_size")
        plan = ChunkPlan(batch.t, cfg.chunk_size)
    if plan.t != batch.t:
        raise ShapeMismatch(f"plan is for t={plan.t}, batch has t={batch.t}")
    itemsize = batch.q.element_size() if isinstance(batch.q, torch.Tensor) else np.asarray(batch.q).dtype.itemsize
    check_state_budget(spec, batch.v_dim, batch.b * batch.h, itemsize, state_budget)
    t0 = time.perf_counter_ns()
    out = _chunked_log_space(batch, cfg, plan, backend) if cfg.use_log_space else run_power(batch, cfg, plan.c)
    if op_timer is not None:
        if isinstance(out.y, torch.Tensor):
            torch.cuda.synchronize()
        op_timer["power_full"] = op_timer.get("power_full", 0) + time.perf_counter_ns() - t0
    return out


def _chunked_log_space(batch: SequenceBatch, cfg: AttentionConfig, plan: ChunkPlan, backend=None):
    """The reference's chunked loop (chunked.py:315-395) with the log-space
    intra-chunk form: per chunk the stabilised attention form (unnormalized,
    pa_power_logspace_fwd) and the state contribution (update_state kernel),
    then the discounted cumsum over chunks and the query of the carried state,
    combined and optionally normalized.  numpy in, numpy out; torch stays on
    the device."""
    from dataclasses import replace

    spec = cfg.expansion
    xp = _xp(batch.q)
    b, t, h = batch.b, batch.t, batch.h
    e, S = batch.v_dim, batch.b * batch.h
    scale = cfg.scale_for(batch.d)
    intra_cfg = replace(cfg, normalize=False, chunk_size=None)

    def streams(x):   # [b, c, h, ...] -> [b*h, c, ...]
        x = xp.swapaxes(x, 1, 2)
        return x.reshape(S, *x.shape[2:])

    bounds = plan.bounds()
    y_attn, zetas, contribs, key_contribs, prefixes, lams = [], [], [], [], [], []
    for start, stop in bounds:
        gk = None if batch.gates is None else batch.gates[:, start:stop]
        sub = SequenceBatch(batch.q[:, start:stop], batch.k[:, start:stop], batch.v[:, start:stop], gk)
        intra = power_attention_form(sub, intra_cfg)
        y_attn.append(intra.y)
        zetas.append(intra.rowsum)
        if gk is None:
            decay = prefix = lam = None
        else:
            g_s = streams(gk[..., None])[..., 0]                      # [S, c]
            decay, prefix = _suffix_products(g_s), _prefix_products(g_s)
            lam = g_s.prod(-1) if xp is torch else np.prod(g_s, axis=-1)
        prefixes.append(prefix)
        lams.append(lam)
        s_k, g_k = update_state_kernel(streams(batch.k[:, start:stop]), streams(batch.v[:, start:stop]), decay,
                                       spec, backend=backend)
        contribs.append(s_k)
        key_contribs.append(g_k)
    n = len(bounds)
    if n > 1:
        if batch.gates is None:
            trans = xp.ones((n - 1, S), dtype=contribs[0].dtype) if xp is np else \
                torch.ones(n - 1, S, dtype=contribs[0].dtype, device=contribs[0].device)
        else:
            trans = xp.stack([lams[k] for k in range(1, n)])
        acc = discumsum(xp.stack(contribs), trans)
        key_acc = discumsum(xp.stack(key_contribs), trans)
    else:
        acc, key_acc = xp.stack(contribs), xp.stack(key_contribs)
    ys, rss = [], []
    for k, (start, stop) in enumerate(bounds):
        c = stop - start
        yk, rk = y_attn[k], zetas[k]
        if k > 0:
            qk = streams(scale * batch.q[:, start:stop])
            yq, den = query_state_kernel(qk, acc[k - 1], key_acc[k - 1], spec, backend=backend)
            if prefixes[k] is not None:
                yq = yq * prefixes[k][..., None]
                den = den * prefixes[k]
            yk = yk + xp.swapaxes(yq.reshape(b, h, c, e), 1, 2)
            rk = rk + xp.swapaxes(den.reshape(b, h, c), 1, 2)
        ys.append(yk)
        rss.append(rk)
    cat = (lambda xs: torch.cat(xs, 1)) if xp is torch else (lambda xs: np.concatenate(xs, 1))
    y, rowsum = cat(ys), cat(rss)
    if cfg.normalize:
        if bool((rowsum <= 0).any()):
            raise ZeroDenominator("zeta + phi(q) . key_sum is not positive; cannot normalize")
        y = y / rowsum[..., None]
    return AttentionOutput(y, rowsum)


def power_attention(batch, cfg, form="attention", plan=None, backend=None, op_timer=None):
    """chunked.py:461-476 (the recurrent form is an oracle-only form)."""
    if form == "attention":
        return power_attention_form(batch, cfg)
    if form == "chunked":
        return chunked_power_attention(batch, cfg, plan, backend=backend, op_timer=op_timer)
    if form == "recurrent":
        # the recurrent form equals the chunked form with c = 1 (test_chunked.py:245-249)
        return chunked_power_attention(batch, cfg, ChunkPlan(batch.t, 1))
    raise InvalidSpec(f"form must be attention, recurrent, or chunked, got {form!r}")


def stream_chunk(state, q_chunk, k_chunk, v_chunk, gates_chunk, cfg, backend=None):
    """One constant-memory streaming step (chunked.py:416-458)."""
    spec = cfg.expansion
    xp = _xp(q_chunk)
    if state is None:
        z = (torch.zeros if xp is torch else np.zeros)
        dim = expansion_dim(spec)
        kw = dict(dtype=v_chunk.dtype, device=v_chunk.device) if xp is torch else dict(dtype=np.result_type(q_chunk, v_chunk))
        state = ChunkState(z((dim, v_chunk.shape[1]), **kw), z((dim,), **kw), spec)
    sub = SequenceBatch(q_chunk[None, :, None, :], k_chunk[None, :, None, :], v_chunk[None, :, None, :],
                        None if gates_chunk is None else gates_chunk[None, :, None])
    from dataclasses import replace
    intra = run_power(sub, replace(cfg, normalize=False, chunk_size=None), None)
    prefix = None if gates_chunk is None else _prefix_products(gates_chunk)
    y = query_state(state, q_chunk, y_attn=intra.y[0, :, 0, :], zeta=intra.rowsum[0, :, 0],
                    gates_prefix=prefix, scale=cfg.scale_for(q_chunk.shape[1]), normalize=cfg.normalize)
    contrib, lam = update_state(spec, k_chunk, v_chunk, gates_chunk)
    return y, ChunkState(lam * state.s + contrib.s, lam * state.key_sum + contrib.key_sum, spec)
