"""Uninitialised-workspace probe: poison the caching allocator with NaN, then run
the bf16 tcgen05 path and report which outputs pick up NaN (diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import power_oracle as O
from test_gpu_parity import run_full

for c, normalize in [(256, False), (384, False), (384, True), (1024, False), (128, False)]:
    t = 2 * c
    junk = torch.full((1 << 28,), float("nan"), device="cuda")   # 1 GiB of NaN
    del junk
    q, k, v, g = O.generate_inputs(1, t, 2, 64, 64, seed=t + 7 * c, gating=True)
    q, k, v = (torch.tensor(x).bfloat16().double().numpy() for x in (q, k, v))
    dy = np.random.default_rng(t + c).uniform(-1, 1, (1, t, 2, 64))
    dyb = torch.tensor(dy).bfloat16().double().numpy()
    r = run_full(q, k, v, g, 2, c, normalize, dtype=torch.bfloat16, dy=dyb)
    y_ref, _ = O.chunked_forward(q, k, v, g, 2, c, normalize=normalize)
    dq, dk, dv, dg = O.chunked_backward(q, k, v, g, 2, c, dyb, normalize=normalize)
    out = {}
    for n, a, b in (("y", r["y"], y_ref), ("dq", r["dq"], dq), ("dk", r["dk"], dk), ("dv", r["dv"], dv),
                    ("dlogg", r["dlogg"], dg * g)):
        bad = ~np.isfinite(a)
        rows = np.unique(np.nonzero(bad)[1]) if bad.any() else []
        out[n] = (round(O.max_rel_error(np.nan_to_num(a), b), 4), int(bad.sum()), list(rows[:8]))
    print(c, normalize, out, flush=True)
