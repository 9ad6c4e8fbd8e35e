"""Sequence parallelism: the rank protocol of
paper_2507_04239_b200.parallel (local phase -> carry chain -> finish) emulated
for R virtual ranks on one GPU must reproduce power_full on the whole sequence
-- forward and every gradient -- and match the numpy oracle within the bf16
bar.  The multi-process NCCL chain itself is covered on CPU (gloo) by
test_sp_chain.py; here the carries are handed over in memory."""

import numpy as np
import pytest
import torch

from oracle import power_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2507_04239_b200")
from paper_2507_04239_b200 import parallel as SP  # noqa: E402

BF16_TOL = 2e-2


def _inputs(t, h, gated, seed):
    q, k, v, g = O.generate_inputs(1, t, h, 64, 64, seed=seed, gating=True)
    q, k, v = (torch.tensor(x).bfloat16().double().numpy() for x in (q, k, v))
    dy = np.random.default_rng(seed + 1).uniform(-1, 1, (1, t, h, 64))
    dy = torch.tensor(dy).bfloat16().double().numpy()
    return q, k, v, (g if gated else None), dy


def _norm_rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _cuda(x, dt):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)


@pytest.mark.parametrize("ranks", [2, 4])
@pytest.mark.parametrize("gated,normalize", [(True, False), (True, True), (False, True)])
def test_sp_emulated_matches_full_and_oracle(ranks, gated, normalize):
    t, h, c = 2048, 2, 256
    q, k, v, g, dy = _inputs(t, h, gated, seed=21 + ranks)
    Q, K, V = (_cuda(x, torch.bfloat16) for x in (q, k, v))
    lg = None if g is None else torch.log(_cuda(g, torch.float32))
    dY = _cuda(dy, torch.bfloat16)
    y, dq, dk, dv, dlg = SP.emulate_ranks(Q, K, V, lg, ranks=ranks, p=2, chunk_size=c, normalize=normalize, dy=dY)
    # the same kernels on the whole sequence in one launch set
    Qf, Kf, Vf = (x.clone().requires_grad_() for x in (Q, K, V))
    lgf = None if lg is None else lg.clone().requires_grad_()
    yf = P.power_full(Qf, Kf, Vf, lgf, p=2, chunk_size=c, normalize=normalize)
    ins = [Qf, Kf, Vf] + ([lgf] if lgf is not None else [])
    gf = torch.autograd.grad(yf, ins, dY)
    pairs = [(y, yf), (dq, gf[0]), (dk, gf[1]), (dv, gf[2])] + ([(dlg, gf[3])] if g is not None else [])
    for a, b in pairs:
        assert O.max_rel_error(a.detach().float().cpu().numpy(), b.detach().float().cpu().numpy()) <= 1e-2
    # and the oracle (float64 on the same bf16-representable inputs).  Ungated
    # sums are compared norm-wise: the elementwise metric is ill-conditioned
    # there under any bf16 operand rounding (precision decisions)
    err = O.max_rel_error if g is not None else _norm_rel
    y_ref, _ = O.chunked_forward(q, k, v, g, 2, c, normalize=normalize)
    assert err(y.float().cpu().numpy(), y_ref) <= BF16_TOL
    gq, gk, gv, gg = O.chunked_backward(q, k, v, g, 2, c, dy, normalize=normalize)
    for a, b in ((dq, gq), (dk, gk), (dv, gv)):
        assert err(a.float().cpu().numpy(), b) <= BF16_TOL
    if g is not None:
        assert O.max_rel_error(dlg.cpu().numpy(), gg * g) <= BF16_TOL


def test_sp_partition_validation():
    with pytest.raises(P.InvalidSpec):
        SP.SpPartition(0, 3, 2048, 256)   # 8 chunks do not split over 3 ranks
    part = SP.SpPartition(2, 4, 4096, 256)
    assert (part.chunk0, part.local_chunks, part.t0, part.nchunks) == (8, 4, 2048, 16)
