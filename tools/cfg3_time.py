"""configs[2]: power_full fwd+bwd bf16 p=4 d=32 (D=52360), t=16384, ungated, b=1 h=16 c=1024 (SIMT path)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2507_04239_b200 import power_full
b, t, h, d, c = 1, 16384, 16, 32, 1024
Q, K, V = ((torch.rand(b, t, h, d, device="cuda") * 2 - 1).bfloat16().requires_grad_() for _ in range(3))
dy = (torch.rand(b, t, h, d, device="cuda") * 2 - 1).bfloat16()
def step():
    y = power_full(Q, K, V, None, p=4, chunk_size=c, normalize=True)
    return torch.autograd.grad(y, [Q, K, V], dy)
step(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(2):
    step()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 2
print(f"configs[2] p=4 d=32 t=16384 b=1 h=16 c=1024 normalized, bf16 in (fp32 CUDA-core path): {ms:.1f} ms/step, "
      f"{b * t / (ms / 1e3):.0f} tokens/s")
