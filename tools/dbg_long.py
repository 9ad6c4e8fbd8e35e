"""Debug: where do bf16 errors sit at long context with gates near 1?"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import power_oracle as O
import paper_2507_04239_b200 as P

t = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
lo = float(sys.argv[2]) if len(sys.argv) > 2 else 0.999
c, d = 1024, 64
rng = np.random.default_rng(31)
q, k, v = (rng.uniform(-1, 1, (1, t, 1, d)) for _ in range(3))
q, k, v = (torch.tensor(x).bfloat16().double().numpy() for x in (q, k, v))
dy = torch.tensor(rng.uniform(-1, 1, (1, t, 1, d))).bfloat16().double().numpy()
g = rng.uniform(lo, 1.0, (1, t, 1))
Q, K, V = (torch.tensor(x, device="cuda", dtype=torch.bfloat16, requires_grad=True) for x in (q, k, v))
lg = torch.tensor(np.log(g), device="cuda", dtype=torch.float32, requires_grad=True)
y = P.power_full(Q, K, V, lg, p=2, chunk_size=c)
gr = torch.autograd.grad(y, [Q, K, V, lg], torch.tensor(dy, device="cuda", dtype=torch.bfloat16))
y = y.detach().double().cpu().numpy()
y_ref, _ = O.chunked_forward(q, k, v, g, 2, c)
dq, dk, dv, dg = O.chunked_backward(q, k, v, g, 2, c, dy)
dl_ref = dg * g
res = {"y": (y, y_ref), "dq": (gr[0].double().cpu().numpy(), dq), "dk": (gr[1].double().cpu().numpy(), dk),
       "dv": (gr[2].double().cpu().numpy(), dv), "dlog_g": (gr[3].double().cpu().numpy(), dl_ref)}
for name, (a, b) in res.items():
    err = np.abs(a - b)
    den = np.maximum(1, np.maximum(np.abs(a), np.abs(b)))
    rel = err / den
    i = np.unravel_index(np.argmax(rel), rel.shape)
    print(f"{name}: max_rel {rel.max():.4g} at {i} a={a[i]:.6g} b={b[i]:.6g} |b|max={np.abs(b).max():.4g} "
          f"norm_rel={np.linalg.norm(a - b) / np.linalg.norm(b):.3g}")
    # per-chunk summary
    ax = 1
    r2 = rel.reshape(1, t // c, c, *rel.shape[2:])
    per = r2.reshape(t // c, -1).max(axis=1)
    print("   per-chunk max_rel:", " ".join(f"{x:.3g}" for x in per[:: max(1, len(per) // 16)]))
