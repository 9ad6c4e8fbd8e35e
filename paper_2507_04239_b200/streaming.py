"""Batched streaming on the tensor cores: every (batch, head) stream keeps a
resident slot-form state on the GPU and consumes its sequence step by step.

The reference's `stream_chunk` (chunked.py:416-458) is one stream and one
chunk at a time on the host; feeding chunks in order reproduces the chunked
form with constant memory.  `stream_step` does the same for all b*h streams at
once through the sequence-parallel kernels of the C ABI, which are exactly a
"chunks against an incoming state" operation:

    y        = pa_sp_fwd_finish(step, carry = state)        (query + intra + combine)
    end      = pa_sp_fwd_local(step)                        (the step's own end state)
    state'   = pa_sp_combine(state, end) = Lambda_step state + end

A step may hold any number of tokens: it is cut into chunks of `chunk_size`
(a multiple of 128 up to 1024; default min(1024, the step rounded up to 128))
and the tail is zero-padded (zero keys and values, log-gate 0: nothing reaches
the state or the real tokens' outputs; padded outputs are dropped).  The chunk
grid does not change the result (the chunked form is chunk-size independent,
reference test_chunked.py:278-285).  Path: bf16 (fp16 inputs are converted),
p = 2, d = e = 64 -- the north-star shape.

The state is the kernels' slot form: fp32 [b, h, 2304 slots, 80] with the SPOW
weight omega folded in (pa_tc_common.cuh).  `to_chunk_states` / `from_chunk_states`
convert to and from the reference's ChunkState ([D, e] state and [D] key_sum
per stream, chunked.py:40-63).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _lib
from .errors import InvalidSpec, ShapeMismatch
from .power import _ptr, _stream, make_problem

SLOTS, COLS, HD = 2304, 80, 64


@lru_cache(maxsize=None)
def _slot_features():
    """slot -> (a, b) of the block order (pa_tc_common.cuh make_blk_tab) and the
    NDMI feature index of (min, max) (reference expansions.py:106-123)."""
    al, be = [], []
    for b_ in range(8):
        for a_ in range(2 * b_ + 2):
            al.append(a_)
            be.append(b_)
    f = np.arange(SLOTS)
    a = 4 * np.asarray(al)[f >> 5] + ((f >> 3) & 3)
    b = 8 * np.asarray(be)[f >> 5] + (f & 7)
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    # NDMI index of (lo, hi), lexicographic over lo <= hi
    feat = lo * HD - lo * (lo - 1) // 2 + (hi - lo)
    live = a <= b
    omega = np.where(a == b, 1.0, 2.0)
    return feat[live], np.nonzero(live)[0], omega[live]


@dataclass
class StreamState:
    """Slot-form states of b x h streams after `chunks` chunks of history."""

    data: torch.Tensor          # fp32 [b * h * 2304 * 80] (flat, the ABI's carry layout)
    b: int
    h: int
    chunks: int = 0

    @classmethod
    def empty(cls, b: int, h: int, device) -> "StreamState":
        return cls(torch.zeros(b * h * SLOTS * COLS, dtype=torch.float32, device=device), b, h, 0)

    def to_chunk_states(self):
        """(s [b, h, D, 64], key_sum [b, h, D]) float64 numpy in the reference's
        ChunkState layout (D = 2080 SPOW features, weights w_f = sqrt(omega_f))."""
        feat, slots, omega = _slot_features()
        st = self.data.view(self.b, self.h, SLOTS, COLS).double().cpu().numpy()
        D = HD * (HD + 1) // 2
        s = np.zeros((self.b, self.h, D, HD))
        ks = np.zeros((self.b, self.h, D))
        w = np.sqrt(omega)
        s[:, :, feat, :] = st[:, :, slots, :HD] / w[:, None]
        ks[:, :, feat] = st[:, :, slots, HD] / w
        return s, ks

    @classmethod
    def from_chunk_states(cls, s, key_sum, chunks: int, device) -> "StreamState":
        """Inverse of to_chunk_states (duplicate slots stay zero)."""
        feat, slots, omega = _slot_features()
        s = np.asarray(s, dtype=np.float64)
        key_sum = np.asarray(key_sum, dtype=np.float64)
        b, h = s.shape[:2]
        st = np.zeros((b, h, SLOTS, COLS))
        w = np.sqrt(omega)
        st[:, :, slots, :HD] = s[:, :, feat, :] * w[:, None]
        st[:, :, slots, HD] = key_sum[:, :, feat] * w
        return cls(torch.tensor(st.reshape(-1), dtype=torch.float32, device=device), b, h, int(chunks))


def _check(Q, K, V, log_G, p):
    if Q.dim() != 4 or K.shape != Q.shape or V.shape[:3] != Q.shape[:3]:
        raise ShapeMismatch("q, k, v must be [b, t, h, 64] with equal b, t, h")
    if int(p) != 2 or Q.shape[-1] != HD or V.shape[-1] != HD:
        raise InvalidSpec("stream_step runs the tensor-core path: p = 2, d = e = 64")
    if not Q.is_cuda:
        raise InvalidSpec("stream_step needs CUDA tensors")
    if log_G is not None and tuple(log_G.shape) != tuple(Q.shape[:3]):
        raise ShapeMismatch("log_g must be [b, t, h]")


def stream_step(state: StreamState | None, Q, K, V, log_G=None, *, p: int = 2, chunk_size: int | None = None,
                scale: float | None = None, normalize: bool = False):
    """Consume one step of tokens [b, t_step, h, 64] for every stream against
    `state` (None = empty history).  Returns (y [b, t_step, h, 64], new state);
    feeding a sequence step by step reproduces power_full on the whole of it."""
    _check(Q, K, V, log_G, p)
    b, t, h, _ = Q.shape
    dev = Q.device
    if state is None:
        state = StreamState.empty(b, h, dev)
    if (state.b, state.h) != (b, h) or state.data.device != dev:
        raise ShapeMismatch("the state belongs to other streams")
    c = int(chunk_size) if chunk_size is not None else min(1024, (t + 127) // 128 * 128)
    if c % 128 or c > 1024 or c < 128:
        raise InvalidSpec("stream_step chunk_size must be a multiple of 128 up to 1024")
    tp = (t + c - 1) // c * c
    dt = torch.bfloat16

    def pad(x, fill=0.0):
        x = x.to(dt) if x.dtype != torch.float32 else x
        if tp == t:
            return x.contiguous()
        shape = list(x.shape)
        shape[1] = tp
        out = torch.full(shape, fill, dtype=x.dtype, device=dev)
        out[:, :t] = x
        return out

    q, k, v = pad(Q), pad(K), pad(V)
    lg = None if log_G is None else pad(log_G.detach().to(torch.float32))
    n = tp // c
    pr = make_problem(q, v, p, c, scale, normalize, lg is not None)
    pr.flags |= _lib.PA_FLAG_KEY_SUM   # the state always carries key_sum (ChunkState.key_sum)
    sp = _lib.PaSpPart(state.chunks, state.chunks + n)
    lib = _lib.load()
    st = _stream(dev)
    with torch.cuda.device(dev):
        wsb = lib.pa_fwd_workspace_bytes(ctypes.byref(pr))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        end = torch.empty_like(state.data)
        _lib.check(lib.pa_sp_fwd_local(ctypes.byref(pr), ctypes.byref(sp), _ptr(q), _ptr(k), _ptr(v), _ptr(lg),
                                       _ptr(ws), wsb, _ptr(end), st), "stream step (local)")
        y = torch.empty(b, tp, h, HD, dtype=dt, device=dev)
        rs = torch.empty(b, tp, h, dtype=torch.float32, device=dev) if normalize else None
        carry = state.data if state.chunks > 0 else None
        _lib.check(lib.pa_sp_fwd_finish(ctypes.byref(pr), ctypes.byref(sp), _ptr(q), _ptr(k), _ptr(v), _ptr(lg),
                                        _ptr(y), _ptr(rs), _ptr(ws), wsb, _ptr(carry), st), "stream step (finish)")
        if state.chunks > 0:
            new = torch.empty_like(end)
            _lib.check(lib.pa_sp_combine(ctypes.byref(pr), ctypes.byref(sp), _ptr(ws), _ptr(state.data), _ptr(end),
                                         _ptr(new), st), "stream step (combine)")
        else:
            new = end
    y = y[:, :t]
    if Q.dtype != dt:
        y = y.to(Q.dtype)
    return y, StreamState(new, b, h, state.chunks + n)
