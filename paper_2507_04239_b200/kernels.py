"""The reference's plugin boundary (kernels.py:55-110) bound to the C ABI.

There is one backend, "cuda"; the reference's "compiled"/"python" names
resolve to it so reference-style callers keep working."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._convert import back, to_dev
from .errors import InvalidSpec, ShapeMismatch
from .expansions import ExpansionKind, ExpansionSpec, expansion_dim, monomial_table

VALID_BACKENDS = ("auto", "cuda", "compiled")


def available_backends() -> tuple[str, ...]:
    return ("cuda",)


def resolve_backend(backend: str | None = None) -> str:
    name = "auto" if backend is None else backend
    if name not in VALID_BACKENDS:
        raise InvalidSpec(f"backend must be one of {VALID_BACKENDS}, got {name!r}")
    return "cuda"


def _prep(arrs, host):
    dt = torch.float64 if any((a is not None) and (
        (isinstance(a, np.ndarray) and a.dtype == np.float64) or
        (isinstance(a, torch.Tensor) and a.dtype == torch.float64)) for a in arrs) else torch.float32
    return [None if a is None else to_dev(a, dt).contiguous() for a in arrs], dt


def _p(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_DEV_TABLES: dict = {}


def _device_table(spec: ExpansionSpec, device):
    """The kind's monomial table on the device (uploaded once per spec/device)."""
    key = (spec, str(device))
    if key not in _DEV_TABLES:
        idx, w = monomial_table(spec)
        _DEV_TABLES[key] = (torch.from_numpy(np.ascontiguousarray(idx)).to(device),
                            torch.from_numpy(np.ascontiguousarray(w)).to(device))
    return _DEV_TABLES[key]


def update_state_kernel(k_chunk, v_chunk, decay, spec: ExpansionSpec, backend=None):
    """(state [n, D, e], key_sum [n, D]) from k [n, c, d], v [n, c, e], decay [n, c]|None."""
    resolve_backend(backend)
    host = not isinstance(k_chunk, torch.Tensor)
    (k, v, w), dt = _prep([k_chunk, v_chunk, decay], host)
    if k.dim() != 3 or v.dim() != 3 or k.shape[:2] != v.shape[:2] or k.shape[2] != spec.d:
        raise ShapeMismatch(f"need k [n, c, d={spec.d}] and v [n, c, e], got {tuple(k.shape)}, {tuple(v.shape)}")
    n, c, d = k.shape
    e = v.shape[2]
    D = expansion_dim(spec)
    state = torch.empty(n, D, e, dtype=dt, device=k.device)
    ks = torch.empty(n, D, dtype=dt, device=k.device)
    code = _lib.PA_F64 if dt == torch.float64 else _lib.PA_F32
    lib = _lib.load()
    with torch.cuda.device(k.device):
        if spec.kind is ExpansionKind.SPOW:
            rc = lib.pa_update_state(n, c, d, e, spec.p, code, _p(k), _p(v), _p(w), _p(state), _p(ks), 0,
                                     _stream())
        else:
            ti, tw = _device_table(spec, k.device)
            rc = lib.pa_update_state_table(n, c, d, e, spec.p, D, code, _p(k), _p(v), _p(w), _p(ti), _p(tw),
                                           _p(state), _p(ks), 0, _stream())
    _lib.check(rc, "update_state")
    return back(state, host), back(ks, host)


def query_state_kernel(q_chunk, state, key_sum, spec: ExpansionSpec, backend=None):
    """(y [n, c, e], denom [n, c]) from pre-scaled q [n, c, d], state [n, D, e], key_sum [n, D]."""
    resolve_backend(backend)
    host = not isinstance(q_chunk, torch.Tensor)
    (q, st, ks), dt = _prep([q_chunk, state, key_sum], host)
    n, c, d = q.shape
    e = st.shape[2]
    if d != spec.d or st.shape[1] != expansion_dim(spec) or ks.shape != st.shape[:2]:
        raise ShapeMismatch("query_state_kernel shapes disagree with the spec")
    y = torch.empty(n, c, e, dtype=dt, device=q.device)
    den = torch.empty(n, c, dtype=dt, device=q.device)
    code = _lib.PA_F64 if dt == torch.float64 else _lib.PA_F32
    lib = _lib.load()
    with torch.cuda.device(q.device):
        if spec.kind is ExpansionKind.SPOW:
            rc = lib.pa_query_state(n, c, d, e, spec.p, code, _p(q), _p(st), _p(ks), _p(y), _p(den), 0,
                                    _stream())
        else:
            ti, tw = _device_table(spec, q.device)
            rc = lib.pa_query_state_table(n, c, d, e, spec.p, st.shape[1], code, _p(q), _p(st), _p(ks), _p(ti),
                                          _p(tw), _p(y), _p(den), 0, _stream())
    _lib.check(rc, "query_state")
    return back(y, host), back(den, host)


def discumsum_kernel(values, lambdas):
    """out[0] = values[0]; out[k] = lambdas[k-1] * out[k-1] + values[k] on the
    device (chunked.py:156-176); lambdas [n-1] or [n-1, L] per leading slice."""
    host = not isinstance(values, torch.Tensor)
    (vals, lams), dt = _prep([values, lambdas], host)
    n = vals.shape[0]
    if lams.shape[0] not in (max(n - 1, 0), n):
        raise ShapeMismatch(f"need {n - 1} transition decays, got {lams.shape[0]}")
    if bool((lams < 0).any()) or bool((lams > 1).any()):
        raise InvalidSpec("decays must lie in [0, 1]")
    lams = lams[: max(n - 1, 0)]
    rest = tuple(vals.shape[1:])
    total = int(np.prod(rest)) if rest else 1
    if n > 1 and lams.dim() == 1:
        lam2, L = lams.reshape(n - 1, 1), 1
    elif n > 1:
        lead = tuple(lams.shape[1:]) + (1,) * (len(rest) - lams.dim() + 1)
        try:
            lam2 = torch.broadcast_to(lams.reshape(n - 1, *lead), (n - 1, *rest)).reshape(n - 1, -1)
        except RuntimeError as exc:
            raise ShapeMismatch(f"lambdas {tuple(lams.shape)} do not broadcast over {rest}") from exc
        L = total
    else:
        lam2, L = None, 1
    out = torch.empty_like(vals)
    code = _lib.PA_F64 if dt == torch.float64 else _lib.PA_F32
    lam2 = lam2.contiguous() if lam2 is not None else torch.zeros(1, dtype=dt, device=vals.device)
    with torch.cuda.device(vals.device):
        rc = _lib.load().pa_discumsum(n, L, total // L, code, _p(vals), _p(lam2), _p(out), _stream())
    _lib.check(rc, "discumsum")
    return back(out, host)
