"""Run one forward with the trace build and print the feature-major GEMM stamps."""
import ctypes
import os
import sys

os.environ["PA_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpa_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_04239_b200 import _lib, power_full  # noqa: E402

b, t, h = 1, 8192, 16
dev = "cuda"
Q, K, V = ((torch.rand(b, t, h, 64, device=dev) * 2 - 1).bfloat16() for _ in range(3))
lg = torch.log(torch.rand(b, t, h, device=dev) * 0.1 + 0.9)
for _ in range(2):
    power_full(Q, K, V, lg, p=2, chunk_size=1024)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 1024)()
_lib.load().pa_debug_trace5(buf, 1024)
base = buf[0]
for i in range(16):
    m = [buf[8 + i * 4 + k] - base for k in range(3)]
    gg = [buf[200 + i * 4 + k] - base for k in range(4)]
    print(f"step {i:2d}: MMA full {m[0]:6d} afull {m[1]:6d} done {m[2]:6d} | GEN start {gg[0]:6d} full {gg[1]:6d} "
          f"aempty {gg[2]:6d} stored {gg[3]:6d}")
print("epilogue", [buf[190 + k] - base for k in range(3)])
