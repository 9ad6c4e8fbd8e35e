"""Per-gradient bf16 errors of power_full against the oracle (diagnostics)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import power_oracle as O  # noqa: E402
import paper_2507_04239_b200 as P  # noqa: E402

for (t, c, norm) in [(1024, 256, False), (1024, 256, True), (2048, 1024, False)]:
    q, k, v, g = O.generate_inputs(1, t, 2, 64, 64, seed=3, gating=True)
    q, k, v = (torch.tensor(x).bfloat16().double().numpy() for x in (q, k, v))
    dy = torch.tensor(np.random.default_rng(4).uniform(-1, 1, (1, t, 2, 64))).bfloat16().double().numpy()
    Q, K, V = (torch.tensor(x, device="cuda", dtype=torch.bfloat16, requires_grad=True) for x in (q, k, v))
    lg = torch.tensor(np.log(g), device="cuda", dtype=torch.float32, requires_grad=True)
    y = P.power_full(Q, K, V, lg, p=2, chunk_size=c, normalize=norm)
    gr = torch.autograd.grad(y, [Q, K, V, lg], torch.tensor(dy, device="cuda", dtype=torch.bfloat16))
    yr, _ = O.chunked_forward(q, k, v, g, 2, c, normalize=norm)
    dq, dk, dv, dg = O.chunked_backward(q, k, v, g, 2, c, dy, normalize=norm)
    print(f"t={t} c={c} norm={norm} y {O.max_rel_error(y.detach().float().cpu().numpy(), yr):.4f}", end=" ")
    for nm, a, b in (("dq", gr[0], dq), ("dk", gr[1], dk), ("dv", gr[2], dv), ("dlg", gr[3], dg * g)):
        a = a.float().cpu().numpy()
        print(f"{nm} {O.max_rel_error(a, b):.4f}", end=" ")
    a = gr[3].cpu().numpy()[0, :, 0]
    b = (dg * g)[0, :, 0]
    e = np.abs(a - b)
    pos = np.arange(t) % c
    print(" | dlg abs err by chunk pos: first16 %.4f mid %.4f last16 %.4f" % (
        e[pos < 16].max(), e[(pos > c // 2 - 8) & (pos < c // 2 + 8)].max(), e[pos >= c - 16].max()))
