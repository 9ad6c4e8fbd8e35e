"""power_full_sp across two real processes (torch.distributed, gloo, both
ranks on cuda:0; the carries are staged through host memory because gloo moves
CPU tensors).  The whole protocol runs: _PowerFullSP's forward and backward,
pa_sp_fwd_local / pa_sp_combine / pa_sp_fwd_finish and the backward mirror,
and the chain over dist.send / dist.recv.  Each rank's slice of y and of the
gradients must equal the single-process power_full result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(b, t, h, d):
    g = torch.Generator().manual_seed(77)
    Q, K, V = ((torch.rand(b, t, h, d, generator=g) * 2 - 1).bfloat16() for _ in range(3))
    lg = torch.log(torch.rand(b, t, h, generator=g) * 0.01 + 0.99)
    dY = (torch.rand(b, t, h, d, generator=g) * 2 - 1).bfloat16()
    return Q, K, V, lg, dY


def _worker(rank, world, port, out_dir, normalize):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_04239_b200 import _lib
        from paper_2507_04239_b200.parallel import power_full_sp

        b, t, h, d, c = 1, 4096, 2, 64, 512
        Q, K, V, lg, dY = _inputs(b, t, h, d)
        tl = t // world
        sl = slice(rank * tl, (rank + 1) * tl)
        q, k, v = (x[:, sl].cuda().requires_grad_() for x in (Q, K, V))
        l = lg[:, sl].cuda().requires_grad_()
        n0 = _lib.launch_count()
        y = power_full_sp(q, k, v, l, p=2, chunk_size=c, normalize=normalize)
        grads = torch.autograd.grad(y, [q, k, v, l], dY[:, sl].cuda())
        torch.cuda.synchronize()
        assert _lib.launch_count() > n0
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), y=y.detach().float().cpu().numpy(),
                 **{n: gr.float().cpu().numpy() for n, gr in zip(("dq", "dk", "dv", "dl"), grads)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("normalize", [False, True])
def test_power_full_sp_two_processes(tmp_path, normalize):
    import paper_2507_04239_b200 as P

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), normalize), nprocs=world, join=True)
    b, t, h, d, c = 1, 4096, 2, 64, 512
    Q, K, V, lg, dY = _inputs(b, t, h, d)
    q, k, v = (x.cuda().requires_grad_() for x in (Q, K, V))
    l = lg.cuda().requires_grad_()
    y = P.power_full(q, k, v, l, p=2, chunk_size=c, normalize=normalize)
    ref = [y.detach()] + list(torch.autograd.grad(y, [q, k, v, l], dY.cuda()))
    ref = [x.float().cpu().numpy() for x in ref]
    parts = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    for i, name in enumerate(("y", "dq", "dk", "dv", "dl")):
        got = np.concatenate([p_[name] for p_ in parts], axis=1)
        err = float(np.abs(got - ref[i]).max() / max(1.0, np.abs(ref[i]).max()))
        print(f"normalize={normalize} {name}: max abs err / max(1, |ref|) = {err:.3e}")
        assert err <= 1e-2, (name, err)
