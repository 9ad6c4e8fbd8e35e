"""Where does the normalized bf16 backward lose precision (diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import power_oracle as O
from test_gpu_parity import run_full

for c, gated in [(384, False), (384, True), (256, False), (1024, False)]:
    t = 768 if c == 384 else 2 * c
    q, k, v, g = O.generate_inputs(1, t, 2, 64, 64, seed=t + 7 * c, gating=gated)
    q, k, v = (torch.tensor(x).bfloat16().double().numpy() for x in (q, k, v))
    dy = np.random.default_rng(t + c).uniform(-1, 1, (1, t, 2, 64))
    dyb = torch.tensor(dy).bfloat16().double().numpy()
    r = run_full(q, k, v, g, 2, c, True, dtype=torch.bfloat16, dy=dyb)
    r32 = run_full(q, k, v, g, 2, c, True, dtype=torch.float32, dy=dyb)
    y_ref, rs = O.chunked_forward(q, k, v, g, 2, c, normalize=True)
    dq, dk, dv, dg = O.chunked_backward(q, k, v, g, 2, c, dyb, normalize=True)
    for n, a, a32, b in (("dq", r["dq"], r32["dq"], dq), ("dk", r["dk"], r32["dk"], dk)):
        err = np.abs(a - b)
        i = np.unravel_index(err.argmax(), err.shape)
        print(c, gated, n, "bf16", round(O.max_rel_error(a, b), 4), "fp32", round(O.max_rel_error(a32, b), 6),
              "at", i, "val", round(float(b[i]), 4), "max|ref|", round(float(np.abs(b).max()), 4),
              "rowsum there", round(float(rs[i[0], i[1], i[2]]), 4), "min rowsum", round(float(rs.min()), 5))
