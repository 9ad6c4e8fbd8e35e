"""bf16 tcgen05 path vs the oracle for several chunk sizes (diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import power_oracle as O
from test_gpu_parity import run_full, norm_rel_error

for c in [128, 256, 384, 512, 640, 768, 1024]:
    for gated in (True,):
        t = 2 * c
        q, k, v, g = O.generate_inputs(1, t, 2, 64, 64, seed=t + 7 * c, gating=gated)
        q, k, v = (torch.tensor(x).bfloat16().double().numpy() for x in (q, k, v))
        dy = np.random.default_rng(t + c).uniform(-1, 1, (1, t, 2, 64))
        dyb = torch.tensor(dy).bfloat16().double().numpy()
        r = run_full(q, k, v, g, 2, c, False, dtype=torch.bfloat16, dy=dyb)
        y_ref, _ = O.chunked_forward(q, k, v, g, 2, c)
        dq, dk, dv, dg = O.chunked_backward(q, k, v, g, 2, c, dyb)
        e = {n: O.max_rel_error(a, b) for n, a, b in (("y", r["y"], y_ref), ("dq", r["dq"], dq), ("dk", r["dk"], dk),
                                                        ("dv", r["dv"], dv), ("dlogg", r["dlogg"], dg * g))}
        # where is dq wrong: per chunk max error
        errq = np.abs(r["dq"] - dq).max(axis=(0, 2, 3))
        per_chunk = [float(errq[i * c:(i + 1) * c].max()) for i in range(t // c)]
        sub = [float(errq[i:i + 128].max()) for i in range(0, t, 128)]
        print(c, {k_: round(v_, 4) for k_, v_ in e.items()}, "dq abs err per 128 tokens", np.round(sub, 3))
