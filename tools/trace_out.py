"""Run one forward with the trace build and print the output kernel's pipeline stamps (query tile 7 of a chunk)."""
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
buf = (ctypes.c_longlong * 512)()
_lib.load().pa_debug_trace4(buf, 512)
base = buf[0]
for stp in range(18):
    m = [buf[10 + stp * 3 + i] - base for i in range(3)]
    gg = [buf[200 + stp * 2 + i] - base for i in range(2)]
    print(f"step {stp:2d}: MMA a_full {m[0]:6d} st_full {m[1]:6d} done {m[2]:6d} | GEN start {gg[0]:6d} a_empty {gg[1]:6d}")
for J in range(8):
    m = [buf[100 + J * 3 + i] - base for i in range(3)]
    p = [buf[400 + J * 3 + i] - base for i in range(3)]
    print(f"J {J}: INTRA wait_p {m[0]:6d} got_p {m[1]:6d} pv_done {m[2]:6d} | P wait_s {p[0]:6d} got_s {p[1]:6d} done {p[2]:6d}")
print("epilogue", [buf[300 + i] - base for i in range(3)])
