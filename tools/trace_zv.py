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
    base = buf[0]
    print(f"side {side} (CTA 37, its third tile): epi acc_full {buf[1]-base} epi done {buf[2]-base}")
    for mw in range(2):
        print(f"  issuer {mw}: wait B {buf[700+mw*4]}, wait A {buf[701+mw*4]}, issue+commit {buf[702+mw*4]}, wait acc_empty {buf[703+mw*4]}")
    for w in range(8):
        print(f"  gen warp {w}: wait a_empty {buf[720+w*2]}, tile prologues {buf[721+w*2]} (rows wait {buf[760+w*2]}, meta wait {buf[761+w*2]})")
    b5 = buf[806]
    print("  tile 4 start -> tile 5 start", buf[805]-b5, "rows ready", buf[800]-b5, "passes", buf[801]-b5, "rows_empty", buf[802]-b5, "before meta", buf[803]-b5, "meta", buf[804]-b5, "end", buf[807]-b5)
    for j in range(0):
        print(f"stage {j:2d}: TMA issue {buf[100+j]-base:7d} | MMA b_full {buf[200+j]-base:7d} a_full {buf[300+j]-base:7d} "
              f"issued {buf[400+j]-base:7d} | GEN a_empty {buf[500+j]-base:7d} arrived {buf[600+j]-base:7d}")
