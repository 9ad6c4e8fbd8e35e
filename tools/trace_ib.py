"""Run one backward with the trace build and print the intra-backward (key side) pipeline stamps."""
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
buf = (ctypes.c_longlong * 1024)()
_lib.load().pa_debug_trace(buf, 1024)
base = buf[0]
names = ["S_commit", "P_seen", "G_issued", "c_wait", "c_got_S", "c_done"]
for n in range(16):
    row = [buf[8 + n * 8 + i] - base for i in range(6)]
    print(n, "  ".join(f"{nm}={v:7d}" for nm, v in zip(names, row)))
