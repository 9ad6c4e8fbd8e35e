"""Quick device timing of power_full forward (and optionally backward) at a given shape."""
import argparse
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_04239_b200 import power_full  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=4)
ap.add_argument("--t", type=int, default=65536)
ap.add_argument("--h", type=int, default=16)
ap.add_argument("--c", type=int, default=1024)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--bwd", action="store_true")
ap.add_argument("--normalize", action="store_true")
a = ap.parse_args()
torch.manual_seed(0)
dev = "cuda"
Q = (torch.rand(a.b, a.t, a.h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_(a.bwd)
K = (torch.rand(a.b, a.t, a.h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_(a.bwd)
V = (torch.rand(a.b, a.t, a.h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_(a.bwd)
lg = torch.log(torch.rand(a.b, a.t, a.h, device=dev) * 0.1 + 0.9).requires_grad_(a.bwd)
dy = torch.randn(a.b, a.t, a.h, 64, device=dev).bfloat16()
for it in range(a.iters + 1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    y = power_full(Q, K, V, lg, p=2, chunk_size=a.c, normalize=a.normalize)
    e1.record()
    if a.bwd:
        e2 = torch.cuda.Event(enable_timing=True)
        torch.autograd.grad(y, [Q, K, V, lg], dy)
        e2.record()
    torch.cuda.synchronize()
    if it:
        msg = f"fwd {e0.elapsed_time(e1):.3f} ms"
        if a.bwd:
            msg += f"  bwd {e1.elapsed_time(e2):.3f} ms"
        print(msg, flush=True)
print("tokens", a.b * a.t)
