"""Plain-PyTorch fp32 restatement of power attention (quadratic form, reference
attention.py:273-309 with the gate decay of 196-205) -- TEST INFRASTRUCTURE.
Autograd-capable, CPU or GPU; used to check the LM stack's plumbing (DDP on
CPU, and the CUDA op inside the model on the GPU)."""

import math

import torch


def power_attention_ref(q, k, v, log_g, p, chunk=None, scale=None):
    """q, k [b, t, h, d]; v [b, t, h, e]; log_g [b, t, h] or None -> y [b, t, h, e]
    in q's dtype (computed in fp32; `chunk` does not change the result)."""
    dt = q.dtype
    q, k, v = (x.float().permute(0, 2, 1, 3) for x in (q, k, v))   # [b, h, t, x]
    sc = 1.0 / math.sqrt(q.shape[-1]) if scale is None else scale
    s = (sc * q) @ k.transpose(-1, -2)
    t = q.shape[2]
    causal = torch.ones(t, t, dtype=torch.bool, device=q.device).tril()
    if log_g is not None:
        L = torch.cumsum(log_g.float().permute(0, 2, 1), dim=-1)      # [b, h, t]
        diff = L[..., :, None] - L[..., None, :]
        decay = torch.exp(torch.where(causal, diff, torch.full_like(diff, -float("inf"))))
    else:
        decay = causal.float()
    y = (s ** p * decay) @ v
    return y.permute(0, 2, 1, 3).to(dt)


def attn_fn(q, k, v, log_g, p, chunk):
    return power_attention_ref(q, k, v, log_g, p, chunk)
