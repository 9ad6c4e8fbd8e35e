"""Compare the tensor-core degree-4 intra-chunk VJP against the CUDA-core one
(same inputs, PA_TC4_INTRA_BWD_OFF toggled): where do dq / dk differ?"""
import os

import torch

import paper_2507_04239_b200 as P

torch.manual_seed(0)
b, t, h, d, c = 1, 2048, 1, 32, 1024
Q, K, V = ((torch.rand(b, t, h, d, device="cuda") * 2 - 1).bfloat16().requires_grad_() for _ in range(3))
dy = (torch.rand(b, t, h, d, device="cuda") * 2 - 1).bfloat16()
for norm in (False, True):
    res = []
    for off in ("1", "0"):
        os.environ["PA_TC4_INTRA_BWD_OFF"] = off
        y = P.power_full(Q, K, V, None, p=4, chunk_size=c, normalize=norm)
        res.append([x.float() for x in torch.autograd.grad(y, [Q, K, V], dy)])
    for name, a, bb in zip("qkv", res[0], res[1]):
        diff = (a - bb).abs()[0, :, 0, :]
        rel = diff.max() / a.abs().max()
        row = diff.max(dim=1).values
        top = torch.topk(row, 5)
        col = diff.max(dim=0).values
        print(f"norm={norm} d{name}: rel {rel.item():.4g}; worst rows {top.indices.tolist()} {[round(v, 5) for v in top.values.tolist()]}; "
              f"per-128-tile max {[round(row[i*128:(i+1)*128].max().item(), 4) for i in range(t // 128)]}; worst cols {torch.topk(col, 4).indices.tolist()}")
