import sys, torch
sys.path.insert(0, ".")
from paper_2507_04239_b200 import power_full
for (b, t, h) in [(1, 4096, 2), (1, 16384, 8), (1, 65536, 16), (4, 65536, 16)]:
    Q = (torch.rand(b, t, h, 64, device="cuda") * 2 - 1).bfloat16().requires_grad_()
    K = (torch.rand(b, t, h, 64, device="cuda") * 2 - 1).bfloat16().requires_grad_()
    V = (torch.rand(b, t, h, 64, device="cuda") * 2 - 1).bfloat16().requires_grad_()
    lg = torch.log(torch.rand(b, t, h, device="cuda") * 0.1 + 0.9).requires_grad_()
    y = power_full(Q, K, V, lg, p=2, chunk_size=1024)
    g = torch.autograd.grad(y, [Q, K, V, lg], torch.ones_like(y))
    torch.cuda.synchronize()
    print("ok", b, t, h, flush=True)
