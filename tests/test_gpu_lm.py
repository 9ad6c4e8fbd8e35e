"""configs[4] on the GPU: the power-attention LM with the CUDA op inside
(bf16 autocast, the tcgen05 path at d=64, chunk 1024) against the same model
with the plain-torch fp32 attention (tests/torch_ref.py), same weights and
tokens: loss and every parameter gradient agree (norm-wise, bf16 bar)."""

import pytest
import torch

from torch_ref import attn_fn

pytestmark = pytest.mark.gpu


def test_lm_with_cuda_attention_matches_torch_reference():
    from paper_2507_04239_b200 import _lib
    from paper_2507_04239_b200.lm import LMConfig, PowerLM, lm_loss

    cfg = LMConfig(vocab=1000, width=128, layers=2, heads=2, chunk=1024)
    torch.manual_seed(0)
    ours = PowerLM(cfg).cuda()
    ref = PowerLM(cfg, attn_fn=attn_fn).cuda()
    ref.load_state_dict(ours.state_dict())
    tok = torch.randint(0, cfg.vocab, (1, 2049), device="cuda")
    x, y = tok[:, :-1], tok[:, 1:]
    losses = []
    n0 = _lib.launch_count()
    for m in (ours, ref):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = lm_loss(m, x, y)
        loss.backward()
        losses.append(float(loss))
    assert _lib.launch_count() > n0
    assert abs(losses[0] - losses[1]) <= 1e-3 * abs(losses[1]), losses
    worst = 0.0
    for (n, a), (_, b) in zip(ours.named_parameters(), ref.named_parameters()):
        err = float((a.grad - b.grad).norm() / b.grad.norm().clamp_min(1e-30))
        worst = max(worst, err)
        assert err <= 3e-2, (n, err)
    print(f"LM loss {losses}, worst parameter-gradient norm error {worst:.3e}")


def test_lm_train_step_124m_runs():
    """The full configs[4] geometry trains one step at a 4096-token sequence."""
    from paper_2507_04239_b200.lm import LMConfig, PowerLM, train_step

    torch.manual_seed(0)
    model = PowerLM(LMConfig()).cuda()
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, fused=True)
    tok = torch.randint(0, 50257, (1, 4097), device="cuda")
    l0 = float(train_step(model, opt, tok[:, :-1], tok[:, 1:]))
    l1 = float(train_step(model, opt, tok[:, :-1], tok[:, 1:]))
    assert torch.isfinite(torch.tensor([l0, l1])).all() and l1 < l0, (l0, l1)
