import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import power_oracle as O  # noqa: E402
import paper_2507_04239_b200 as P  # noqa: E402
t, c = 1024, 256
q, k, v, g = O.generate_inputs(1, t, 2, 64, 64, seed=3, gating=True)
q, k, v = (torch.tensor(x).bfloat16().double().numpy() for x in (q, k, v))
dy = torch.tensor(np.random.default_rng(4).uniform(-1, 1, (1, t, 2, 64))).bfloat16().double().numpy()
Q, K, V = (torch.tensor(x, device="cuda", dtype=torch.bfloat16, requires_grad=True) for x in (q, k, v))
lg = torch.tensor(np.log(g), device="cuda", dtype=torch.float32, requires_grad=True)
y = P.power_full(Q, K, V, lg, p=2, chunk_size=c)
gr = torch.autograd.grad(y, [Q, K, V, lg], torch.tensor(dy, device="cuda", dtype=torch.bfloat16))
dq, dk, dv, dg = O.chunked_backward(q, k, v, g, 2, c, dy)
a = gr[3].cpu().numpy()[0, :, 0]
b = (dg * g)[0, :, 0]
np.set_printoptions(precision=4, suppress=True, linewidth=200)
for ch in range(4):
    e = (a - b)[ch * c:(ch + 1) * c]
    print("chunk", ch, "err every 8th:", e[::8])
    print("   ref every 8th:", b[ch * c:(ch + 1) * c][::8][:12])
