"""power_full: the north-star operator (chunked power attention with log-gates)
as a torch autograd op over the C ABI.

Semantics (reference chunked.py:287-413 with g = exp(log_G); attention form
when chunk_size is None or >= t, reference test_chunked.py:239-243):

    y[i] = sum_{j <= i} exp(L_i - L_j) (scale * q_i . k_j)^p v_j      (unnormalized)
    y[i] /= sum_{j <= i} exp(L_i - L_j) (scale * q_i . k_j)^p          (normalize=True)

with L the cumulative sum of log_G over time.  Gradients: dQ, dK, dV and
dlog_G = g * dgates (reference gradients.py:361-483).
"""

from __future__ import annotations

import collections
import ctypes
import math
import os
import threading
import warnings

import torch

from . import _lib
from .errors import InvalidSpec, OddPowerWithNormalize, ShapeMismatch, ZeroDenominator

_DTYPES = {torch.float32: _lib.PA_F32, torch.bfloat16: _lib.PA_BF16, torch.float16: _lib.PA_F16}


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0")


def make_problem(Q, V, p, chunk_size, scale, normalize, gated, deterministic=None, strict=None) -> _lib.PaProblem:
    """The pa_problem of a call.  scale=None means 1/sqrt(d); any other value
    (zero and negative included) is used as given, like the reference's
    scale_for (attention.py:149-150)."""
    b, t, h, d = Q.shape
    e = V.shape[-1]
    c = t if chunk_size is None else min(int(chunk_size), t)
    det = _env_flag("PA_DETERMINISTIC") if deterministic is None else bool(deterministic)
    strict = _env_flag("PA_STRICT_TC") if strict is None else bool(strict)
    flags = (_lib.PA_FLAG_DETERMINISTIC if det else 0) | (_lib.PA_FLAG_STRICT_TC if strict else 0)
    has_scale = scale is not None
    return _lib.PaProblem(b, t, h, d, e, int(p), c, int(bool(normalize)), _DTYPES[Q.dtype], int(bool(gated)),
                          int(has_scale), flags, float(scale) if has_scale else 0.0)


_warned = set()


def _route(pr) -> bool:
    """True when the problem runs on the tensor-core kernels.  Raises the
    reference's error class for an invalid problem (make_geo's own code) and
    warns once per shape when a 16-bit problem drops to the fp32 CUDA-core
    kernels (PA_STRICT_TC=1 / strict=True turns that into an error)."""
    rc = _lib.load().pa_uses_tensor_cores(ctypes.byref(pr))
    if rc < 0:
        _lib.check(-rc, "power_full")
    if rc == 0 and pr.dtype != _lib.PA_F32:
        key = (pr.p, pr.d, pr.e, pr.chunk, pr.t % max(pr.chunk, 1), pr.dtype)
        if key not in _warned:
            _warned.add(key)
            warnings.warn(
                f"power_full: p={pr.p} d={pr.d} e={pr.e} chunk={pr.chunk} t={pr.t} dtype={pr.dtype} is outside the "
                "tcgen05 tensor-core kernels (bf16, p=2, d=e=64, chunk a multiple of 128 up to 1024, t a multiple "
                "of the chunk); running the fp32 CUDA-core kernels", RuntimeWarning, stacklevel=4)
    return rc >= 1


def _validate(Q, K, V, log_G, p, chunk_size, normalize):
    for name, x in (("Q", Q), ("K", K), ("V", V)):
        if not isinstance(x, torch.Tensor) or x.dim() != 4:
            raise ShapeMismatch(f"{name} must be a [b, t, h, feature] tensor")
        if not x.is_cuda:
            raise InvalidSpec(f"{name} must be a CUDA tensor (this package has no CPU path)")
    if K.shape != Q.shape:
        raise ShapeMismatch(f"K shape {tuple(K.shape)} != Q shape {tuple(Q.shape)}")
    if V.shape[:3] != Q.shape[:3]:
        raise ShapeMismatch(f"V shape {tuple(V.shape)} disagrees with Q on [b, t, h]")
    if K.device != Q.device or V.device != Q.device or (log_G is not None and log_G.device != Q.device):
        raise InvalidSpec("Q, K, V and log_G must live on one CUDA device")
    if Q.dtype not in _DTYPES or K.dtype != Q.dtype or V.dtype != Q.dtype:
        raise InvalidSpec("Q, K, V must share one dtype among float32, bfloat16, float16")
    if log_G is not None and tuple(log_G.shape) != tuple(Q.shape[:3]):
        raise ShapeMismatch(f"log_G shape {tuple(log_G.shape)} != [b, t, h] {tuple(Q.shape[:3])}")
    if chunk_size is not None and int(chunk_size) < 1:
        raise InvalidSpec(f"chunk_size must be >= 1, got {chunk_size}")
    if p < 1:
        raise InvalidSpec(f"power degree must be >= 1, got {p}")
    if normalize and p % 2:
        # reference attention.py:133-139
        raise OddPowerWithNormalize(f"normalize=True needs an even power degree, got p={p}")


# ---------------------------------------------------------------- zero denominators
# The reference raises ZeroDenominator from the forward (chunked.py:392-395).
# "sync" reads the device flag right away (a stream synchronisation);
# "deferred" copies it asynchronously into pinned memory and raises from the
# next power_full call (or check_denominators()) once the copy has landed, so a
# training loop never stalls on it.
_pending = threading.local()


def _pending_list():
    if not hasattr(_pending, "q"):
        _pending.q = collections.deque()
    return _pending.q


def check_denominators(block: bool = True) -> None:
    """Raise ZeroDenominator if a deferred check of an earlier normalized
    forward found a non-positive score sum (block=True waits for the copies)."""
    q = _pending_list()
    while q:
        ev, flag = q[0]
        if not block and not ev.query():
            return
        ev.synchronize()
        q.popleft()
        if int(flag.item()):
            q.clear()
            raise ZeroDenominator("zeta + phi(q) . key_sum is not positive; cannot normalize")


def _check_mode(check_den):
    if check_den in (True, "sync"):
        return "sync"
    if check_den in (False, None, "off"):
        return "off"
    if check_den == "deferred":
        return "deferred"
    raise InvalidSpec(f"check_denominator must be True/'sync', 'deferred' or False, got {check_den!r}")


class _PowerFull(torch.autograd.Function):
    @staticmethod
    def forward(ctx, Q, K, V, log_G, p, chunk_size, scale, normalize, check_den, want_rowsum, det, strict):
        lib = _lib.load()
        Q, K, V = Q.contiguous(), K.contiguous(), V.contiguous()
        lg = None if log_G is None else log_G.detach().to(torch.float32).contiguous()
        pr = make_problem(Q, V, p, chunk_size, scale, normalize, lg is not None, det, strict)
        _route(pr)
        wsb = lib.pa_fwd_workspace_bytes(ctypes.byref(pr))
        ws = torch.empty(wsb, dtype=torch.uint8, device=Q.device)
        y = torch.empty(*Q.shape[:3], V.shape[-1], dtype=Q.dtype, device=Q.device)
        # the score sum costs extra MMAs; only produce it when it is consumed
        need_rs = bool(normalize or want_rowsum)
        rowsum = torch.empty(*Q.shape[:3] if need_rs else (0,), dtype=torch.float32, device=Q.device)
        st = _stream(Q.device)
        _lib.check(lib.pa_power_full_fwd(ctypes.byref(pr), _ptr(Q), _ptr(K), _ptr(V), _ptr(lg),
                                         _ptr(y), _ptr(rowsum if need_rs else None), _ptr(ws), wsb, st),
                   "power_full forward")
        mode = _check_mode(check_den)
        if normalize and mode == "sync":
            cnt = ctypes.c_int32(0)
            _lib.check(lib.pa_fwd_zero_denominators(ctypes.byref(pr), _ptr(ws), st, ctypes.byref(cnt)),
                       "zero-denominator check")
            if cnt.value:
                raise ZeroDenominator("zeta + phi(q) . key_sum is not positive; cannot normalize")
        elif normalize and mode == "deferred":
            # both workspace layouts keep the flag in their first 4 bytes
            flag = torch.empty(1, dtype=torch.int32, pin_memory=True)
            flag.copy_(ws[:4].view(torch.int32), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(Q.device))
            _pending_list().append((ev, flag))
        ctx.pr = pr
        ctx.has_lg = lg is not None
        ctx.save_for_backward(Q, K, V, lg if lg is not None else torch.empty(0, device=Q.device),
                              y, rowsum, ws)
        ctx.mark_non_differentiable(rowsum)
        return y, rowsum

    @staticmethod
    def backward(ctx, dy, _drowsum):
        lib = _lib.load()
        Q, K, V, lg, y, rowsum, ws = ctx.saved_tensors
        lg = lg if ctx.has_lg else None
        pr = ctx.pr
        with torch.cuda.device(Q.device):
            check_denominators(block=False)
            dy = dy.contiguous().to(Q.dtype)
            bb = lib.pa_bwd_workspace_bytes(ctypes.byref(pr))
            bws = torch.empty(bb, dtype=torch.uint8, device=Q.device)
            dQ = torch.empty_like(Q)
            dK = torch.empty_like(K)
            dV = torch.empty_like(V)
            dlg = torch.empty_like(lg) if lg is not None else None
            _lib.check(lib.pa_power_full_bwd(ctypes.byref(pr), _ptr(Q), _ptr(K), _ptr(V), _ptr(lg),
                                             _ptr(y), _ptr(rowsum if rowsum.numel() else None), _ptr(dy),
                                             _ptr(dQ), _ptr(dK), _ptr(dV), _ptr(dlg), _ptr(ws), _ptr(bws), bb,
                                             _stream(Q.device)), "power_full backward")
        return dQ, dK, dV, dlg, None, None, None, None, None, None, None, None


def power_full_with_rowsum(Q, K, V, log_G=None, *, p=2, chunk_size=None, scale=None,
                           normalize=False, check_denominator="deferred", deterministic=None, strict=None,
                           _want_rowsum=True):
    """(y, rowsum): rowsum is the reference AttentionOutput.rowsum
    (unnormalized score sum zeta + phi(q).key_sum, chunked.py:390)."""
    _validate(Q, K, V, log_G, p, chunk_size, normalize)
    with torch.cuda.device(Q.device):
        check_denominators(block=False)
        return _PowerFull.apply(Q, K, V, log_G, int(p), chunk_size, scale, bool(normalize), check_denominator,
                                bool(_want_rowsum), deterministic, strict)


def power_full(Q, K, V, log_G=None, *, p=2, chunk_size=None, scale=None, normalize=False,
               check_denominator="deferred", deterministic=None, strict=None):
    """Chunked power attention on CUDA.  Q, K [b, t, h, d]; V [b, t, h, e];
    log_G [b, t, h] (log of gates in (0, 1]; None = ungated).  Returns y
    [b, t, h, e] in Q's dtype.  Zero gates (log_G = -inf) are clamped to
    log g = -80 inside the kernels.

    check_denominator (normalize=True): "deferred" (default) raises
    ZeroDenominator from a later call once the asynchronous flag read lands
    (see check_denominators); True/"sync" raises from this call (synchronises
    the stream); False skips the check.  deterministic=True (or
    PA_DETERMINISTIC=1) fixes the tensor-core summation order so repeated calls
    are bit-identical; strict=True (or PA_STRICT_TC=1) raises InvalidSpec
    instead of running a 16-bit problem on the fp32 CUDA-core kernels."""
    return power_full_with_rowsum(Q, K, V, log_G, p=p, chunk_size=chunk_size, scale=scale,
                                  normalize=normalize, check_denominator=check_denominator,
                                  deterministic=deterministic, strict=strict, _want_rowsum=False)[0]


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)


_LS_DTYPES = {torch.float32: _lib.PA_F32, torch.float64: _lib.PA_F64}


def power_logspace_forward(Q, K, V, log_G=None, *, p=2, scale=None, normalize=False, eps=None):
    """Stabilised attention form (reference attention.py:289-305, use_log_space):
    forward only, through pa_power_logspace_fwd.  Q, K, V, log_G share one dtype
    (float32 or float64); log_G may hold -inf for zero gates.  eps defaults to
    the reference's DEFAULT_EPSILON (1e-7 f32, 1e-12 f64, attention.py:42).
    Returns (y, rowsum).  Gradients of the log-space form are those of the
    direct form (reference SPEC.md:325): use power_full / vjp_chunked."""
    for name, x in (("Q", Q), ("K", K), ("V", V)):
        if not isinstance(x, torch.Tensor) or x.dim() != 4:
            raise ShapeMismatch(f"{name} must be a [b, t, h, feature] tensor")
        if not x.is_cuda:
            raise InvalidSpec(f"{name} must be a CUDA tensor (this package has no CPU path)")
    if Q.dtype not in _LS_DTYPES or K.dtype != Q.dtype or V.dtype != Q.dtype:
        raise InvalidSpec("log-space form: Q, K, V must share float32 or float64")
    if K.shape != Q.shape or V.shape[:3] != Q.shape[:3]:
        raise ShapeMismatch("log-space form: Q, K, V disagree on [b, t, h, d]")
    if p % 2:
        raise InvalidSpec(f"log-space scoring needs even p, got p={p}")
    if eps is None:
        eps = 1e-7 if Q.dtype == torch.float32 else 1e-12
    lib = _lib.load()
    Q, K, V = Q.contiguous(), K.contiguous(), V.contiguous()
    lg = None if log_G is None else log_G.detach().to(Q.dtype).contiguous()
    if lg is not None and tuple(lg.shape) != tuple(Q.shape[:3]):
        raise ShapeMismatch(f"log_G shape {tuple(lg.shape)} != [b, t, h] {tuple(Q.shape[:3])}")
    b, t, h, d = Q.shape
    pr = _lib.PaProblem(b, t, h, d, V.shape[-1], int(p), t, int(bool(normalize)), _LS_DTYPES[Q.dtype],
                        int(lg is not None), int(scale is not None), 0, float(scale) if scale is not None else 0.0)
    y = torch.empty_like(V)
    rowsum = torch.empty(Q.shape[:3], dtype=Q.dtype, device=Q.device)
    with torch.cuda.device(Q.device):
        rc = lib.pa_power_logspace_fwd(ctypes.byref(pr), float(eps), _ptr(Q), _ptr(K), _ptr(V), _ptr(lg),
                                       _ptr(y), _ptr(rowsum), _stream(Q.device))
    _lib.check(rc, "pa_power_logspace_fwd")
    return y, rowsum
