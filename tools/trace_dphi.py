"""Run one backward with the trace build and print the update-side dphi kernel stamps."""
import ctypes
import os
import sys

os.environ["PA_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpa_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_04239_b200 import _lib, power_full  # noqa: E402

b, t, h = 1, 8192, 16
dev = "cuda"
Q = (torch.rand(b, t, h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_()
K = (torch.rand(b, t, h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_()
V = (torch.rand(b, t, h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_()
lg = torch.log(torch.rand(b, t, h, device=dev) * 0.1 + 0.9).requires_grad_()
for _ in range(2):
    y = power_full(Q, K, V, lg, p=2, chunk_size=1024)
    torch.autograd.grad(y, [Q, K, V, lg], torch.ones_like(y))
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 512)()
_lib.load().pa_debug_trace2(buf, 512)
base = buf[99]
for nt in range(18):
    m = [buf[nt * 4 + i] - base for i in range(3)]
    c = [buf[100 + nt * 4 + i] - base for i in range(3)]
    print(f"tile {nt:2d}: mma b_full {m[0]:7d} d_empty {m[1]:7d} issued {m[2]:7d} | epi wait {c[0]:7d} got {c[1]:7d} done {c[2]:7d}")
print("phase2 gen start", buf[200] - base, "gen done", buf[201] - base, "fin", buf[202] - base)
print("phase2 kb issue", [buf[210 + kb] - base for kb in range(36)])
