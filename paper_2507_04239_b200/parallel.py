"""Sequence parallelism for power_full (BASELINE configs[3]).

A long sequence is split into contiguous chunk ranges, one per rank (one
process per GPU).  The chunk-state recurrence of the reference
(discumsum, chunked.py:156-176 / 356-367: A_k = lambda_k A_{k-1} + S_k) is a
linear recurrence with the associative combine
(l1, S1) o (l2, S2) = (l1 l2, l2 S1 + S2), so the only cross-rank dependency is
one D x (e+1) state per stream per rank boundary:

  forward   local:   every rank builds its chunk states from a zero carry and
                     reports its end state E_r (pa_sp_fwd_local)
            chain:   C_0 = 0, C_{r+1} = exp(L_r) C_r + E_r, passed rank to rank
                     with NCCL point-to-point (pa_sp_combine; L_r = sum of the
                     rank's chunk log-decays)
            finish:  discumsum from C_r, then attention + state query
                     (pa_sp_fwd_finish)
  backward  local:   cotangent P_r of the incoming state from a zero end-state
                     cotangent (pa_sp_bwd_local)
            chain:   H_{R-1} = 0, H_{r-1} = exp(L_r) H_r + P_r, passed backwards
            finish:  reverse discumsum from H_r and every gradient kernel
                     (pa_sp_bwd_finish)

The local phases run concurrently on all ranks; the chains move
b*h*2304*80*4 bytes per hop (11.8 MB for b=1, h=16) and do one elementwise
kernel per hop.  `emulate_ranks` runs the same protocol for R virtual ranks in
one process (one GPU) -- the parity tests use it.
"""

from __future__ import annotations

import ctypes
import math
from typing import Callable, Optional

import torch

from . import _lib
from .errors import InvalidSpec
from .power import _DTYPES, _ptr, _stream, _validate, make_problem


class SpPartition:
    """This rank's slice of the sequence: chunks [chunk0, chunk0 + local_chunks) of nchunks."""

    def __init__(self, rank: int, world: int, t_total: int, chunk: int):
        if t_total % chunk:
            raise InvalidSpec(f"sequence length {t_total} must be a multiple of the chunk size {chunk}")
        n = t_total // chunk
        if n % world:
            raise InvalidSpec(f"{n} chunks do not split evenly over {world} ranks")
        self.rank, self.world, self.chunk = rank, world, chunk
        self.nchunks = n
        self.local_chunks = n // world
        self.chunk0 = rank * self.local_chunks
        self.t0 = self.chunk0 * chunk
        self.t_local = self.local_chunks * chunk

    def part(self) -> _lib.PaSpPart:
        return _lib.PaSpPart(self.chunk0, self.nchunks)


# ---------------------------------------------------------------- carry chains
def _peer(group, rank: int) -> int:
    """Global rank of group rank `rank` (dist.send/recv take global ranks even
    when a group is given)."""
    import torch.distributed as dist

    return rank if group is None else dist.get_global_rank(group, rank)


def _host_staged(group) -> bool:
    """gloo moves CPU tensors only: carries are staged through host memory."""
    import torch.distributed as dist

    return dist.get_backend(group) == "gloo"


def _send(x: torch.Tensor, dst: int, group) -> None:
    import torch.distributed as dist

    dist.send(x.cpu() if (x.is_cuda and _host_staged(group)) else x, dst=dst, group=group)


def _recv(like: torch.Tensor, src: int, group) -> torch.Tensor:
    import torch.distributed as dist

    if like.is_cuda and _host_staged(group):
        buf = torch.empty(like.shape, dtype=like.dtype)
        dist.recv(buf, src=src, group=group)
        return buf.to(like.device)
    buf = torch.empty_like(like)
    dist.recv(buf, src=src, group=group)
    return buf


def chain_forward(local: torch.Tensor, combine: Callable[[Optional[torch.Tensor], torch.Tensor], torch.Tensor],
                  rank: int, world: int, group=None) -> Optional[torch.Tensor]:
    """Exclusive left-to-right scan of the per-rank local results over ranks.
    Returns the incoming carry of this rank (None on rank 0).  One receive from
    rank-1 and one send to rank+1 (torch.distributed point-to-point); `rank`
    and `world` are positions inside `group`."""
    import torch.distributed as dist

    carry = None
    if rank > 0:
        carry = _recv(local, _peer(group, rank - 1), group)
    if rank < world - 1:
        _send(combine(carry, local).contiguous(), _peer(group, rank + 1), group)
    return carry


def chain_backward(local: torch.Tensor, combine: Callable[[Optional[torch.Tensor], torch.Tensor], torch.Tensor],
                   rank: int, world: int, group=None) -> Optional[torch.Tensor]:
    """The same scan right to left (cotangents flow from later ranks)."""
    import torch.distributed as dist

    carry = None
    if rank < world - 1:
        carry = _recv(local, _peer(group, rank + 1), group)
    if rank > 0:
        _send(combine(carry, local).contiguous(), _peer(group, rank - 1), group)
    return carry


# ---------------------------------------------------------------- per-rank kernels
class _Rank:
    """One rank's buffers and the C ABI calls of the protocol."""

    def __init__(self, Q, K, V, lg, p, chunk, scale, normalize, part: SpPartition):
        self.Q, self.K, self.V, self.lg = Q, K, V, lg
        self.pr = make_problem(Q, V, p, chunk, scale, normalize, lg is not None)
        self.sp = part.part()
        self.part = part
        lib = _lib.load()
        self.lib = lib
        dev = Q.device
        self.nfl = lib.pa_sp_state_floats(ctypes.byref(self.pr))
        self.wsb = lib.pa_fwd_workspace_bytes(ctypes.byref(self.pr))
        self.ws = torch.empty(self.wsb, dtype=torch.uint8, device=dev)
        self.normalize = normalize

    def state(self):
        return torch.zeros(self.nfl, dtype=torch.float32, device=self.Q.device)

    def combine(self, carry, local):
        out = torch.empty_like(local)
        _lib.check(self.lib.pa_sp_combine(ctypes.byref(self.pr), ctypes.byref(self.sp), _ptr(self.ws),
                                          _ptr(carry), _ptr(local), _ptr(out), _stream(self.Q.device)),
                   "sp combine")
        return out

    def fwd_local(self):
        end = self.state()
        _lib.check(self.lib.pa_sp_fwd_local(ctypes.byref(self.pr), ctypes.byref(self.sp), _ptr(self.Q),
                                            _ptr(self.K), _ptr(self.V), _ptr(self.lg), _ptr(self.ws), self.wsb,
                                            _ptr(end), _stream(self.Q.device)), "sp forward (local)")
        return end

    def fwd_finish(self, carry, want_rowsum):
        Q, V = self.Q, self.V
        y = torch.empty(*Q.shape[:3], V.shape[-1], dtype=Q.dtype, device=Q.device)
        # keep a detached alias only: holding the autograd output here would make a
        # reference cycle (output -> grad_fn -> ctx -> this object) and delay freeing
        self.y = y.detach()
        need_rs = bool(self.normalize or want_rowsum)
        self.rowsum = torch.empty(*Q.shape[:3] if need_rs else (0,), dtype=torch.float32, device=Q.device)
        _lib.check(self.lib.pa_sp_fwd_finish(ctypes.byref(self.pr), ctypes.byref(self.sp), _ptr(Q), _ptr(self.K),
                                             _ptr(V), _ptr(self.lg), _ptr(self.y),
                                             _ptr(self.rowsum if need_rs else None), _ptr(self.ws), self.wsb,
                                             _ptr(carry), _stream(Q.device)), "sp forward (finish)")
        return y

    def bwd_local(self, dy):
        lib = self.lib
        self.dy = dy.contiguous().to(self.Q.dtype)
        self.bwb = lib.pa_bwd_workspace_bytes(ctypes.byref(self.pr))
        self.bws = torch.empty(self.bwb, dtype=torch.uint8, device=self.Q.device)
        pre = self.state()
        rs = self.rowsum if self.rowsum.numel() else None
        _lib.check(lib.pa_sp_bwd_local(ctypes.byref(self.pr), ctypes.byref(self.sp), _ptr(self.Q), _ptr(self.K),
                                       _ptr(self.V), _ptr(self.lg), _ptr(self.y), _ptr(rs), _ptr(self.dy),
                                       _ptr(self.ws), _ptr(self.bws), self.bwb, _ptr(pre),
                                       _stream(self.Q.device)), "sp backward (local)")
        return pre

    def bwd_finish(self, carry):
        Q, K, V, lg = self.Q, self.K, self.V, self.lg
        dQ, dK, dV = torch.empty_like(Q), torch.empty_like(K), torch.empty_like(V)
        dlg = torch.empty_like(lg) if lg is not None else None
        rs = self.rowsum if self.rowsum.numel() else None
        _lib.check(self.lib.pa_sp_bwd_finish(ctypes.byref(self.pr), ctypes.byref(self.sp), _ptr(Q), _ptr(K),
                                             _ptr(V), _ptr(lg), _ptr(self.y), _ptr(rs), _ptr(self.dy), _ptr(dQ),
                                             _ptr(dK), _ptr(dV), _ptr(dlg), _ptr(self.ws), _ptr(self.bws),
                                             self.bwb, _ptr(carry), _stream(Q.device)), "sp backward (finish)")
        return dQ, dK, dV, dlg


def _prep(Q, K, V, log_G):
    Q, K, V = Q.contiguous(), K.contiguous(), V.contiguous()
    lg = None if log_G is None else log_G.detach().to(torch.float32).contiguous()
    return Q, K, V, lg


class _PowerFullSP(torch.autograd.Function):
    @staticmethod
    def forward(ctx, Q, K, V, log_G, p, chunk, scale, normalize, t_total, group, rank, world):
        Q, K, V, lg = _prep(Q, K, V, log_G)
        part = SpPartition(rank, world, t_total, chunk)
        r = _Rank(Q, K, V, lg, p, chunk, scale, normalize, part)
        end = r.fwd_local()
        carry = chain_forward(end, r.combine, rank, world, group)
        y = r.fwd_finish(carry, False)
        ctx.r, ctx.group, ctx.has_lg = r, group, lg is not None
        ctx.rank, ctx.world = rank, world
        return y

    @staticmethod
    def backward(ctx, dy):
        r = ctx.r
        with torch.cuda.device(r.Q.device):
            pre = r.bwd_local(dy)
            carry = chain_backward(pre, r.combine, ctx.rank, ctx.world, ctx.group)
            dQ, dK, dV, dlg = r.bwd_finish(carry)
        return dQ, dK, dV, dlg, None, None, None, None, None, None, None, None


def power_full_sp(Q, K, V, log_G=None, *, p=2, chunk_size, scale=None, normalize=False, group=None):
    """power_full over a sequence split across the ranks of `group` (one GPU per
    rank): Q, K, V, log_G hold this rank's contiguous token range
    [rank * t_local, (rank + 1) * t_local) of a sequence of world * t_local tokens.
    Returns this rank's slice of y; the backward returns this rank's gradients."""
    import torch.distributed as dist

    _validate(Q, K, V, log_G, p, chunk_size, normalize)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    t_total = Q.shape[1] * world
    with torch.cuda.device(Q.device):
        return _PowerFullSP.apply(Q, K, V, log_G, int(p), int(chunk_size), scale, bool(normalize), t_total,
                                  group, rank, world)


def emulate_ranks(Q, K, V, log_G, *, ranks: int, p=2, chunk_size, scale=None, normalize=False, dy=None):
    """Run the sequence-parallel protocol for `ranks` virtual ranks in this
    process (slices of the full [b, t, h, .] tensors, carries handed over in
    memory instead of NCCL).  Returns y (and the gradients when dy is given),
    concatenated over the sequence -- they must equal power_full's."""
    _validate(Q, K, V, log_G, p, chunk_size, normalize)
    t = Q.shape[1]
    if t % ranks:
        raise InvalidSpec("t must split evenly over the virtual ranks")
    tl = t // ranks
    Q, K, V, lg = _prep(Q, K, V, log_G)
    rk = []
    for r in range(ranks):
        sl = slice(r * tl, (r + 1) * tl)
        part = SpPartition(r, ranks, t, int(chunk_size))
        rk.append(_Rank(Q[:, sl].contiguous(), K[:, sl].contiguous(), V[:, sl].contiguous(),
                        None if lg is None else lg[:, sl].contiguous(), int(p), int(chunk_size), scale,
                        bool(normalize), part))
    ends = [r.fwd_local() for r in rk]
    carries = [None]
    for r in range(ranks - 1):
        carries.append(rk[r].combine(carries[r], ends[r]))
    ys = [rk[r].fwd_finish(carries[r], False) for r in range(ranks)]
    y = torch.cat(ys, dim=1)
    if dy is None:
        return y
    pres = [rk[r].bwd_local(dy[:, r * tl:(r + 1) * tl]) for r in range(ranks)]
    cots = [None] * ranks
    for r in range(ranks - 1, 0, -1):
        cots[r - 1] = rk[r].combine(cots[r], pres[r])
    grads = [rk[r].bwd_finish(cots[r]) for r in range(ranks)]
    out = [torch.cat([g[i] for g in grads], dim=1) for i in range(3)]
    dlg = torch.cat([g[3] for g in grads], dim=1) if lg is not None else None
    return y, out[0], out[1], out[2], dlg


def chunk_count(t: int, chunk: int) -> int:
    return math.ceil(t / chunk)
