"""configs[1] shape with normalize=True (the score-sum columns in every state GEMM): fwd+bwd ms/step."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2507_04239_b200 import _lib, power_full
b, t, h, d, c = 4, 65536, 16, 64, 1024
g = torch.Generator(device="cuda").manual_seed(0)
Q, K, V = ((torch.rand(b, t, h, d, device="cuda", generator=g) * 2 - 1).bfloat16().requires_grad_() for _ in range(3))
LG = torch.log(torch.rand(b, t, h, device="cuda", generator=g) * 0.1 + 0.9).requires_grad_()
dY = (torch.rand(b, t, h, d, device="cuda", generator=g) * 2 - 1).bfloat16()
def step():
    y = power_full(Q, K, V, LG, p=2, chunk_size=c, normalize=True)
    return torch.autograd.grad(y, [Q, K, V, LG], dY)
for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    step()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"configs[1] normalized: {ms:.2f} ms/step, {b * t / ms * 1e3 / 1e6:.2f} M tokens/s")
_lib.profile_reset(); _lib.profile_enable(True)
step(); torch.cuda.synchronize()
_lib.profile_enable(False)
print({k: round(v[0], 3) for k, v in _lib.profile_read().items()})
