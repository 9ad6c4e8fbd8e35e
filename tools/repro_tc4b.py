"""Small degree-4 fwd + bwd on the tensor-core path (for compute-sanitizer)."""
import torch

import paper_2507_04239_b200 as P

torch.manual_seed(0)
b, t, h, d, c = 1, 256, 1, 32, 128
Q, K, V = ((torch.rand(b, t, h, d, device="cuda") * 2 - 1).bfloat16().requires_grad_() for _ in range(3))
y = P.power_full(Q, K, V, None, p=4, chunk_size=c, normalize=True)
g = torch.autograd.grad(y, [Q, K, V], torch.ones_like(y))
torch.cuda.synchronize()
print("ok", float(y.float().abs().sum()), [float(x.float().abs().sum()) for x in g])
