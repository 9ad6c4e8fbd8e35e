"""CPU oracle for chunked power attention -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's algorithm for
the hot path (``/root/reference/pkg/src/power_attention``).  It exists so the
CUDA path can be checked against the reference semantics on machines where the
reference itself is not importable (the GPU box).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may import it; the product package never does.

Parity of this restatement is pinned against the real reference by
``tests/golden/make_golden.py`` (fixtures in ``tests/golden/*.npz``) and by
``tests/test_oracle.py``.

Layout conventions follow the reference: q, k are [b, t, h, d], v is
[b, t, h, e] (``e`` = value width, the reference's ``v``), gates [b, t, h] with
raw gate values in [0, 1].  Internally everything is reshaped to per-stream
arrays [S, t, x] with S = b*h streams (reference chunked.py:282-284 flattens the
same way).
"""

from __future__ import annotations

import math
from functools import lru_cache
from itertools import combinations_with_replacement

import numpy as np

__all__ = [
    "ndmi_table",
    "expansion_table",
    "feature_dim",
    "phi",
    "phi_vjp",
    "chunk_bounds",
    "intra_chunk",
    "update_state",
    "discumsum",
    "discumsum_vjp",
    "query_state",
    "chunked_forward",
    "chunked_backward",
    "attention_forward",
    "power_full",
    "power_full_vjp",
    "max_rel_error",
    "generate_inputs",
]


# --------------------------------------------------------------------------
# metric (reference checks.py:26-31, tests/conftest.py:7-11)
# --------------------------------------------------------------------------
def max_rel_error(a, b) -> float:
    """max |a-b| / max(1, |a|, |b|), elementwise then max."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    scale = np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
    return float((np.abs(a - b) / scale).max())


def generate_inputs(b, t, h, d, e, seed=0, dtype=np.float64, gating=False):
    """Same generator and draw order as reference inputs.py:20-35 (Philox)."""
    rng = np.random.Generator(np.random.Philox(seed))
    q = rng.uniform(-1.0, 1.0, (b, t, h, d)).astype(dtype)
    k = rng.uniform(-1.0, 1.0, (b, t, h, d)).astype(dtype)
    v = rng.uniform(-1.0, 1.0, (b, t, h, e)).astype(dtype)
    g = rng.uniform(0.9, 1.0, (b, t, h)).astype(dtype) if gating else None
    return q, k, v, g


# --------------------------------------------------------------------------
# SPOW feature map (reference expansions.py)
# --------------------------------------------------------------------------
def feature_dim(p: int, d: int) -> int:
    """D = C(d+p-1, p) (expansions.py:87-99, SPOW branch)."""
    return math.comb(d + p - 1, p)


@lru_cache(maxsize=None)
def ndmi_table(p: int, d: int):
    """(idx [D, p] int32, w [D] float64): non-decreasing multi-indices in
    lexicographic order (expansions.py:106-123) with sqrt-multinomial weights
    sqrt(p! / prod(hist!)) (expansions.py:149-163, table 171-198)."""
    rows = list(combinations_with_replacement(range(d), p))
    idx = np.array(rows, dtype=np.int32).reshape(len(rows), p)
    w = np.empty(len(rows))
    for r, row in enumerate(rows):
        denom = 1
        for val in set(row):
            denom *= math.factorial(row.count(val))
        w[r] = math.sqrt(math.factorial(p) / denom)
    idx.setflags(write=False)
    w.setflags(write=False)
    return idx, w


def expansion_table(kind: str, p: int, d: int, d_tile=None):
    """(idx, w) of the three expansion kinds (expansions.py:171-198):
    spow = ndmi_table; tpow = every ordered tuple, first index slowest
    (_cartesian_indices 166-168), weight 1; tspow = for each NDMI over the
    d/d_tile tiles (weight w_T) the dense d_tile^p block of tile offsets, every
    entry weighted w_T (188-194)."""
    if kind == "spow":
        return ndmi_table(p, d)
    if kind == "tpow":
        idx = np.indices((d,) * p).reshape(p, -1).T.astype(np.int32)
        return idx, np.ones(idx.shape[0])
    tiles, tw = ndmi_table(p, d // d_tile)
    offs = np.indices((d_tile,) * p).reshape(p, -1).T
    idx = (tiles[:, None, :].astype(np.int64) * d_tile + offs[None]).reshape(-1, p).astype(np.int32)
    return idx, np.repeat(tw, d_tile ** p)


def table_update_state(k, v, decay, idx, w):
    """update_state with an explicit monomial table (_reference.py:16-33):
    state[s] = sum_j decay_j phi(k_j) (x) v_j, key_sum[s] = sum_j decay_j phi(k_j)."""
    ph = np.take(k, idx[:, 0], axis=-1) * w
    for z in range(1, idx.shape[1]):
        ph = ph * np.take(k, idx[:, z], axis=-1)
    if decay is not None:
        ph = ph * decay[..., None]
    return np.einsum("scf,sce->sfe", ph, v), ph.sum(axis=1)


def table_query_state(q, state, key_sum, idx, w):
    """query_state with an explicit table (_reference.py:36-50)."""
    ph = np.take(q, idx[:, 0], axis=-1) * w
    for z in range(1, idx.shape[1]):
        ph = ph * np.take(q, idx[:, z], axis=-1)
    return np.einsum("scf,sfe->sce", ph, state), np.einsum("scf,sf->sc", ph, key_sum)


def phi(x: np.ndarray, p: int) -> np.ndarray:
    """phi(x)[..., r] = w_r * prod_z x[..., idx[r, z]] (expansions.py:201-212)."""
    idx, w = ndmi_table(p, x.shape[-1])
    dt = x.dtype if x.dtype in (np.float32, np.float64) else np.float64
    out = np.take(x, idx[:, 0], axis=-1).astype(dt, copy=True)
    for z in range(1, p):
        out *= np.take(x, idx[:, z], axis=-1)
    return out * w.astype(dt)


def phi_vjp(x: np.ndarray, up: np.ndarray, p: int) -> np.ndarray:
    """d<up, phi(x)>/dx (gradients.py:46-76): for each factor position z the
    derivative is w * prod_{z' != z} x[idx[:, z']], scattered onto idx[:, z]."""
    x = np.asarray(x, dtype=np.float64)
    up = np.asarray(up, dtype=np.float64)
    d = x.shape[-1]
    idx, w = ndmi_table(p, d)
    lead = x.shape[:-1]
    xf = x.reshape(-1, d)
    uf = (up * w).reshape(xf.shape[0], -1)
    cols = [xf[:, idx[:, z]] for z in range(p)]
    dx = np.zeros_like(xf)
    for z in range(p):
        part = uf.copy()
        for z2 in range(p):
            if z2 != z:
                part *= cols[z2]
        # scatter-add along features: dx[:, idx[r, z]] += part[:, r]
        onehot = np.zeros((idx.shape[0], d))
        onehot[np.arange(idx.shape[0]), idx[:, z]] = 1.0
        dx += part @ onehot
    return dx.reshape(*lead, d)


# --------------------------------------------------------------------------
# chunk plan and gate helpers (chunked.py:66-100, 274-279)
# --------------------------------------------------------------------------
def chunk_bounds(t: int, c: int):
    """[(start, stop)] covering range(t); last chunk may be short (chunked.py:85-86)."""
    return [(s, min(s + c, t)) for s in range(0, t, c)]


def _suffix_excl(g: np.ndarray) -> np.ndarray:
    """W[..., j] = prod(g[..., j+1:]) ; last entry 1 (chunked.py:89-95)."""
    out = np.ones_like(g)
    if g.shape[-1] > 1:
        rc = np.cumprod(g[..., ::-1], axis=-1)[..., ::-1]
        out[..., :-1] = rc[..., 1:]
    return out


def _prefix_incl(g: np.ndarray) -> np.ndarray:
    """gp[..., m] = prod(g[..., :m+1]) (chunked.py:98-100)."""
    return np.cumprod(g, axis=-1)


def _pair_decay(g: np.ndarray) -> np.ndarray:
    """G[..., i, j] = prod(g[..., j+1..i]) for i >= j, 1 above the diagonal
    (attention.py:196-205; exact for zero gates)."""
    c = g.shape[-1]
    lower = np.arange(c)[:, None] > np.arange(c)[None, :]
    fac = np.where(lower, g[..., :, None], 1.0)
    return np.multiply.accumulate(fac, axis=-2)


def _streams(a: np.ndarray) -> np.ndarray:
    """[b, t, h, ...] -> [b*h, t, ...]."""
    a = np.swapaxes(a, 1, 2)
    return a.reshape(a.shape[0] * a.shape[1], *a.shape[2:])


def _unstreams(a: np.ndarray, b: int, h: int) -> np.ndarray:
    """[b*h, t, ...] -> [b, t, h, ...]."""
    return np.swapaxes(a.reshape(b, h, *a.shape[1:]), 1, 2)


# --------------------------------------------------------------------------
# the four stages (per stream arrays [S, c, x])
# --------------------------------------------------------------------------
def intra_chunk(q, k, v, g, scale, p):
    """Quadratic causal power attention inside one chunk, unnormalized
    (attention.py:273-309 direct path; called with normalize=False at
    chunked.py:323, 336).  Returns (Y [S,c,e], zeta [S,c])."""
    c = q.shape[1]
    s = (scale * q) @ np.swapaxes(k, -1, -2)
    wts = np.where(np.tril(np.ones((c, c), dtype=bool)), s**p, 0.0)
    if g is not None:
        wts = wts * _pair_decay(g)
    return wts @ v, wts.sum(-1)


def update_state(k, v, decay, p):
    """S = phi(k)^T diag(decay) v [S, D, e]; gamma = phi(k)^T decay [S, D]
    (kernels.py:55-83 -> _reference.py:16-33)."""
    f = phi(k, p)
    if decay is not None:
        f = f * decay[..., None]
    return np.swapaxes(f, -1, -2) @ v, f.sum(-2)


def discumsum(values, lams):
    """out[0] = values[0]; out[k] = lams[k-1]*out[k-1] + values[k], as a
    separate multiply and add so it equals the naive loop bit for bit
    (chunked.py:156-176).  lams has n-1 (or n, last ignored) entries."""
    values = np.asarray(values)
    lams = np.asarray(lams, dtype=values.dtype)
    n = values.shape[0]
    if lams.shape[0] not in (max(n - 1, 0), n):
        raise ValueError(f"need {n - 1} transition decays, got {lams.shape[0]}")
    if (lams < 0).any() or (lams > 1).any():
        raise ValueError("decays must lie in [0, 1]")
    out = np.empty_like(values)
    out[0] = values[0]
    for kk in range(1, n):
        prod = lams[kk - 1] * out[kk - 1]
        out[kk] = prod + values[kk]
    return out


def discumsum_vjp(values, lams, up):
    """Reverse scan (gradients.py:267-288).  Returns (dvalues, dlams) with
    dlams reduced to lams' shape."""
    fwd = discumsum(values, lams)
    n = values.shape[0]
    dvals = np.empty_like(values)
    dl = np.zeros(np.shape(lams), dtype=values.dtype)
    acc = up[n - 1]
    dvals[n - 1] = acc
    for kk in range(n - 2, -1, -1):
        full = fwd[kk] * acc
        tgt = dl[kk].shape
        extra = full.ndim - len(tgt)
        if extra:
            full = full.sum(axis=tuple(range(extra)))
        ax = tuple(i for i, s_ in enumerate(tgt) if s_ == 1 and full.shape[i] != 1)
        if ax:
            full = full.sum(axis=ax, keepdims=True)
        dl[kk] = full
        acc = up[kk] + lams[kk] * acc
        dvals[kk] = acc
    return dvals, dl


def query_state(q_scaled, state, key_sum, p):
    """(y [S,c,e], denom [S,c]) = phi(q) @ state, phi(q) @ key_sum
    (kernels.py:86-110 -> _reference.py:36-50)."""
    f = phi(q_scaled, p)
    return f @ state, np.einsum("scD,sD->sc", f, key_sum)


# --------------------------------------------------------------------------
# orchestrators
# --------------------------------------------------------------------------
def chunked_forward(q, k, v, gates, p, chunk, scale=None, normalize=False, want_trace=False):
    """Chunked pipeline (chunked.py:287-413): intra -> update -> discumsum ->
    query -> combine -> optional normalize.  Returns (y, rowsum[, trace])."""
    q = np.asarray(q)
    k = np.asarray(k)
    v = np.asarray(v)
    b, t, h, d = q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    dt = np.result_type(q, v)
    Q, K, V = _streams(q), _streams(k), _streams(v)
    G = None if gates is None else _streams(np.asarray(gates))
    bounds = chunk_bounds(t, chunk)
    n = len(bounds)
    yat, zet, S, Gam, lam, W, GP = [], [], [], [], [], [], []
    for s0, s1 in bounds:
        g = None if G is None else G[:, s0:s1]
        ya, z = intra_chunk(Q[:, s0:s1], K[:, s0:s1], V[:, s0:s1], g, scale, p)
        yat.append(ya)
        zet.append(z)
        w = None if g is None else _suffix_excl(g)
        W.append(w)
        GP.append(None if g is None else _prefix_incl(g))
        lam.append(None if g is None else g.prod(-1))
        st, gm = update_state(K[:, s0:s1], V[:, s0:s1], w, p)
        S.append(st)
        Gam.append(gm)
    if n > 1:
        if G is None:
            trans = np.ones((n - 1, 1, 1, 1), dtype=S[0].dtype)
        else:
            trans = np.stack(lam[1:])[..., None, None]
        A = discumsum(np.stack(S), trans)
        Ag = discumsum(np.stack(Gam), trans[..., 0])
    else:
        trans = None
        A, Ag = np.stack(S), np.stack(Gam)
    Y = np.empty((Q.shape[0], t, V.shape[-1]), dtype=dt)
    R = np.empty((Q.shape[0], t), dtype=dt)
    for kk, (s0, s1) in enumerate(bounds):
        if kk == 0:
            Y[:, s0:s1] = yat[kk]
            R[:, s0:s1] = zet[kk]
            continue
        ys, den = query_state(scale * Q[:, s0:s1], A[kk - 1], Ag[kk - 1], p)
        if GP[kk] is not None:
            ys = ys * GP[kk][..., None]
            den = den * GP[kk]
        Y[:, s0:s1] = yat[kk] + ys
        R[:, s0:s1] = zet[kk] + den
    if normalize:
        if (R <= 0).any():
            raise ZeroDivisionError("zeta + phi(q).key_sum is not positive")
        Y = Y / R[..., None]
    y, rowsum = _unstreams(Y, b, h), _unstreams(R, b, h)
    if want_trace:
        return y, rowsum, dict(bounds=bounds, A=A, Ag=Ag, S=S, Gam=Gam, W=W, GP=GP,
                               lam=lam, trans=trans, scale=scale, Y=Y, R=R)
    return y, rowsum


def _intra_vjp(q, k, v, g, scale, p, dy, dzeta):
    """Backward of the intra-chunk form (gradients.py:98-176, power branch,
    with the rowsum cotangent of line 145-146 and the gate rule of 79-95)."""
    c = q.shape[1]
    raw = (scale * q) @ np.swapaxes(k, -1, -2)
    mask = np.tril(np.ones((c, c), dtype=bool))
    f = np.where(mask, raw**p, 0.0)
    dec = None if g is None else _pair_decay(g)
    wts = f if dec is None else f * dec
    dw = dy @ np.swapaxes(v, -1, -2) + dzeta[..., None]
    dv = np.swapaxes(wts, -1, -2) @ dy
    dg = None
    if dec is None:
        df = np.where(mask, dw, 0.0)
    else:
        df = np.where(mask, dw * dec, 0.0)
        # d/dg_m of G[i,j] (j < m <= i) = G[i,j]/g_m -> rectangle sums
        prod = np.where(mask, dw * f, 0.0) * dec
        col = prod.cumsum(-1)
        rect = np.flip(np.flip(col, -2).cumsum(-2), -2)
        dg = np.zeros_like(g)
        if c > 1:
            m = np.arange(1, c)
            dg[:, 1:] = rect[:, m, m - 1] / g[:, 1:]
    draw = df * p * raw ** (p - 1)
    dq = scale * (draw @ k)
    dk = np.swapaxes(draw, -1, -2) @ (scale * q)
    return dq, dk, dv, dg


def chunked_backward(q, k, v, gates, p, chunk, dy, scale=None, normalize=False):
    """VJP of chunked_forward w.r.t. (q, k, v, gates) for a cotangent on y
    (gradients.py:361-483).  Returns float64 (dq, dk, dv, dgates|None)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    gates = None if gates is None else np.asarray(gates, dtype=np.float64)
    y, rowsum, tr = chunked_forward(q, k, v, gates, p, chunk, scale, normalize, want_trace=True)
    b, t, h, d = q.shape
    scale = tr["scale"]
    Q, K, V = _streams(q), _streams(k), _streams(v)
    G = None if gates is None else _streams(gates)
    DY = _streams(np.asarray(dy, dtype=np.float64))
    if normalize:
        R = tr["R"]
        Yn = _streams(y)
        dnum = DY / R[..., None]
        dden = -(DY * Yn).sum(-1) / R
    else:
        dnum = DY
        dden = np.zeros(DY.shape[:2])
    dQ = np.zeros_like(Q)
    dK = np.zeros_like(K)
    dV = np.zeros_like(V)
    dG = None if G is None else np.zeros_like(G)
    A, Ag = tr["A"], tr["Ag"]
    dA = np.zeros_like(A)
    dAg = np.zeros_like(Ag)
    bounds = tr["bounds"]
    n = len(bounds)
    for kk, (s0, s1) in enumerate(bounds):
        dyc = dnum[:, s0:s1]
        dzc = dden[:, s0:s1]
        if kk > 0:
            qs = scale * Q[:, s0:s1]
            f = phi(qs, p)
            ys = f @ A[kk - 1]
            den = np.einsum("scD,sD->sc", f, Ag[kk - 1])
            gp = tr["GP"][kk]
            if gp is not None:
                dys = dyc * gp[..., None]
                dden_s = dzc * gp
                dgp = (dyc * ys).sum(-1) + dzc * den
                # gp[m] = prod(g[:m+1]) contains g_u for u <= m (gradients.py:260-264)
                pr = dgp * gp
                dG[:, s0:s1] += np.flip(np.flip(pr, -1).cumsum(-1), -1) / G[:, s0:s1]
            else:
                dys, dden_s = dyc, dzc
            dphi = dys @ np.swapaxes(A[kk - 1], -1, -2) + dden_s[..., None] * Ag[kk - 1][:, None, :]
            dA[kk - 1] += np.swapaxes(f, -1, -2) @ dys
            dAg[kk - 1] += np.einsum("scD,sc->sD", f, dden_s)
            dQ[:, s0:s1] += scale * phi_vjp(qs, dphi, p)
        g = None if G is None else G[:, s0:s1]
        a, bk, c_, dg = _intra_vjp(Q[:, s0:s1], K[:, s0:s1], V[:, s0:s1], g, scale, p, dyc, dzc)
        dQ[:, s0:s1] += a
        dK[:, s0:s1] += bk
        dV[:, s0:s1] += c_
        if dg is not None:
            dG[:, s0:s1] += dg
    if n > 1:
        trans = tr["trans"]
        dS, dtr_s = discumsum_vjp(np.stack(tr["S"]), trans, dA)
        dGam, dtr_g = discumsum_vjp(np.stack(tr["Gam"]), trans[..., 0], dAg)
        dtrans = dtr_s[..., 0, 0] + dtr_g[..., 0]
    else:
        dS, dGam, dtrans = dA, dAg, None
    for kk, (s0, s1) in enumerate(bounds):
        kc, vc = K[:, s0:s1], V[:, s0:s1]
        w = tr["W"][kk]
        f = phi(kc, p)
        part = vc @ np.swapaxes(dS[kk], -1, -2) + dGam[kk][:, None, :]
        if w is None:
            dphi = part
            dV[:, s0:s1] += f @ dS[kk]
        else:
            dphi = w[..., None] * part
            dV[:, s0:s1] += w[..., None] * (f @ dS[kk])
            dw = (f * part).sum(-1)
            g = G[:, s0:s1]
            # suffix[j] = prod(g[j+1:]) and lam = prod(g) (gradients.py:245-257)
            pr = dw * w
            excl = np.zeros_like(pr)
            excl[:, 1:] = pr[:, :-1].cumsum(-1)
            dl = dtrans[kk - 1] if (kk >= 1 and dtrans is not None) else np.zeros(g.shape[0])
            dG[:, s0:s1] += (excl + dl[:, None] * g.prod(-1, keepdims=True)) / g
        dK[:, s0:s1] += phi_vjp(kc, dphi, p)
    out = [_unstreams(x, b, h) for x in (dQ, dK, dV)]
    out.append(None if dG is None else _unstreams(dG, b, h))
    return tuple(out)


def attention_forward(q, k, v, gates, p, scale=None, normalize=False):
    """Quadratic power attention over the whole sequence (attention.py:273-309)."""
    b, t, h, d = q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    Q, K, V = _streams(q), _streams(k), _streams(v)
    G = None if gates is None else _streams(gates)
    Y, R = intra_chunk(Q, K, V, G, scale, p)
    if normalize:
        if (R <= 0).any():
            raise ZeroDivisionError("score sum is not positive")
        Y = Y / R[..., None]
    return _unstreams(Y, b, h), _unstreams(R, b, h)


# --------------------------------------------------------------------------
# log-gate surface used by power_full (north star): g = exp(log_G)
# --------------------------------------------------------------------------
def power_full(Q, K, V, log_G=None, p=2, chunk_size=None, scale=None, normalize=False):
    """y of chunked power attention with log-gates; chunk_size None or >= t is
    the attention form (reference test_chunked.py:239-243)."""
    t = Q.shape[1]
    g = None if log_G is None else np.exp(np.asarray(log_G, dtype=np.float64))
    c = t if chunk_size is None else min(chunk_size, t)
    return chunked_forward(Q, K, V, g, p, c, scale, normalize)[0]


def power_full_vjp(Q, K, V, log_G, dy, p=2, chunk_size=None, scale=None, normalize=False):
    """(dQ, dK, dV, dlog_G) with dlog_G = g * dgates."""
    t = Q.shape[1]
    g = None if log_G is None else np.exp(np.asarray(log_G, dtype=np.float64))
    c = t if chunk_size is None else min(chunk_size, t)
    dq, dk, dv, dg = chunked_backward(Q, K, V, g, p, c, dy, scale, normalize)
    return dq, dk, dv, (None if dg is None else dg * g)
