"""Run one configs[1]-shaped backward with the trace build (tools/build_trace.sh)
and print the fused intra-chunk backward's pipeline stamps of one CTA."""
import ctypes
import os
import sys

os.environ["PA_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpa_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_04239_b200 import _lib, power_full  # noqa: E402

b, t, h = 4, 65536, 16
dev = "cuda"
Q = (torch.rand(b, t, h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_()
K = (torch.rand(b, t, h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_()
V = (torch.rand(b, t, h, 64, device=dev) * 2 - 1).bfloat16().requires_grad_()
lg = torch.log(torch.rand(b, t, h, device=dev) * 0.1 + 0.9).requires_grad_()
for _ in range(2):
    y = power_full(Q, K, V, lg, p=2, chunk_size=1024)
    torch.autograd.grad(y, [Q, K, V, lg], torch.ones_like(y))
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (16 * 64))()
_lib.load().pa_debug_trace_ix(buf, 16 * 64)
T = lambda ev, i: buf[ev * 64 + i]
base = T(0, 0)
names = ["A_go", "A_done", "c0_S", "c0_done", "-", "-", "B_got_P", "B_done"]
for n in range(40):
    print(f"hn {n:2d} " + " ".join(f"{nm}={T(e, n) - base:8d}" for e, nm in enumerate(names)))
for i in range(20):
    print(f"In {i:2d} B_dq_go={T(8, i) - base:8d} epi_got={T(9, i) - base:8d} epi_red={T(10, i) - base:8d}")
