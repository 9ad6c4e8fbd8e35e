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
_lib.load().pa_debug_trace3(buf, 512)
base = buf[99]
for nt in range(18):
    m = [buf[nt * 4 + i] - base for i in range(4)]
    c = [buf[100 + nt * 4 + i] - base for i in range(4)]
    gg = [buf[300 + nt * 3 + i] - base for i in range(3)]
    print(f"tile {nt:2d}: MMA b_full {m[0]:6d} d_empty {m[1]:6d} dphi_iss {buf[400 + nt] - base:6d} g_full {m[2]:6d} "
          f"dv_iss {m[3]:6d} | GEN start {gg[0]:6d} g_empty {gg[1]:6d} st_done {gg[2]:6d} | EPI got_d {c[2]:6d} "
          f"done {c[3]:6d}")
