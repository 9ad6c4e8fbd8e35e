"""configs[4] plumbing on CPU: the power-attention LM under
DistributedDataParallel at world size 2 (gloo) produces, on every rank, the
gradient of the mean loss over both ranks' sequences -- the same gradient one
process computes on the two sequences directly.  The attention op here is the
plain-torch fp32 reference (tests/torch_ref.py); the CUDA op inside the model is
checked in tests/test_gpu_lm.py."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from torch_ref import attn_fn

from paper_2507_04239_b200.lm import LMConfig, PowerLM, lm_loss, non_embedding_params

TINY = LMConfig(vocab=97, width=32, layers=2, heads=2, chunk=8)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(rank):
    g = torch.Generator().manual_seed(10 + rank)
    tok = torch.randint(0, TINY.vocab, (1, 25), generator=g)
    return tok[:, :-1], tok[:, 1:]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.manual_seed(0)
        model = PowerLM(TINY, attn_fn=attn_fn).double()
        ddp = torch.nn.parallel.DistributedDataParallel(model, bucket_cap_mb=0.01)   # several buckets
        x, y = _data(rank)
        lm_loss(ddp, x, y).backward()
        torch.save({n: p.grad.clone() for n, p in model.named_parameters()}, os.path.join(out, f"g{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_ddp_gradients_equal_single_process(tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    torch.manual_seed(0)
    model = PowerLM(TINY, attn_fn=attn_fn).double()
    loss = sum(lm_loss(model, *_data(r)) for r in range(2)) / 2
    loss.backward()
    for r in range(2):
        got = torch.load(os.path.join(tmp_path, f"g{r}.pt"))
        for n, p in model.named_parameters():
            torch.testing.assert_close(got[n], p.grad, rtol=1e-9, atol=1e-12, msg=n)


def test_lm_geometry_is_gpt2_small():
    cfg = LMConfig()
    assert (cfg.layers, cfg.width, cfg.heads, cfg.head_dim) == (12, 768, 12, 64)
    assert non_embedding_params(cfg) == 84_934_656          # reference flops.py:92-94
    with torch.device("meta"):
        m = PowerLM(cfg)
    n = sum(p.numel() for p in m.parameters())
    assert 123e6 < n < 125e6, n
