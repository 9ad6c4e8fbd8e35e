"""Run one backward with the trace build and print the state-VJP GEMM (pa_tc_zvjp.cu) stamps.
"""
import ctypes
import os
import sys

os.environ["PA_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpa_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_04239_b200 import _lib, power_full  # noqa: E402

b, t, h = 4, 32768, 16
dev = "cuda"
Q = (torch.rand(b, t, h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_()
K = (torch.rand(b, t, h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_()
V = (torch.rand(b, t, h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_()
lg = torch.log(torch.rand(b, t, h, device=dev) * 0.1 + 0.9).requires_grad_()
for _ in range(2):
    y = power_full(Q, K, V, lg, p=2, chunk_size=1024)
    torch.autograd.grad(y, [Q, K, V, lg], torch.ones_like(y))
torch.cuda.synchronize()
allb = (ctypes.c_longlong * 2048)()
_lib.load().pa_debug_trace6(allb, 2048)
for side, off in (("update", 0), ("query", 1024)):
    buf = allb[off:off + 1024]
    base = buf[820]
    print(side)
    for it in range(1, 30):
        print(f"  tile {it:2d}: gen start {buf[820+it]-base:8d} (prep wait {buf[860+it]-buf[820+it]:6d}, period {buf[820+it]-buf[820+it-1]:6d})  acc_full {buf[900+it]-base:8d}")
