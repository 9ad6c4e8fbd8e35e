"""Sequence-parallel carry chains over real processes (gloo, CPU).

paper_2507_04239_b200.parallel.chain_forward / chain_backward are the
rank-to-rank part of the sequence-parallel protocol (on GPUs the same calls
run over NCCL).  Here every rank holds a contiguous range of chunk states of a
synthetic discumsum problem; the chain, with the combine
exp(L_r) * carry + local, must hand every rank exactly the state (forward) and
the state cotangent (backward) the serial recurrence of the reference
(discumsum chunked.py:156-176, discumsum_vjp gradients.py:267-288) gives at
that rank's boundary."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(n, seed=5):
    rng = np.random.default_rng(seed)
    S = rng.standard_normal((n, 2, 6, 3))            # chunk states [n, streams, D, e]
    lam = rng.uniform(0.5, 1.0, (n, 2))              # per-chunk decay per stream
    dA = rng.standard_normal((n, 2, 6, 3))           # direct cotangent of slot j (state before chunk j)
    return S, lam, dA


def _worker(rank, world, port, n):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_04239_b200.parallel import chain_backward, chain_forward

        S, lam, dA = _problem(n)
        nl = n // world
        lo, hi = rank * nl, (rank + 1) * nl
        L = np.log(lam[lo:hi]).sum(0)                 # [streams]

        def combine(carry, local):
            c = torch.zeros_like(local) if carry is None else carry
            return torch.from_numpy(np.exp(L))[:, None, None] * c + local

        # forward: end state of the local range from a zero carry
        loc = np.zeros_like(S[0])
        for k in range(lo, hi):
            loc = lam[k][:, None, None] * loc + S[k]
        carry = chain_forward(torch.from_numpy(loc), combine, rank, world)
        # serial reference: A_k = lam_k A_{k-1} + S_k from A_{-1} = 0
        A = np.zeros_like(S[0])
        for k in range(lo):
            A = lam[k][:, None, None] * A + S[k]
        if rank == 0:
            assert carry is None
        else:
            np.testing.assert_allclose(carry.numpy(), A, rtol=1e-12, atol=1e-12)

        # backward: cotangent of the prefix slot from a zero end-state cotangent
        G = np.zeros_like(S[0])
        for j in range(hi - 1, lo - 1, -1):
            G = dA[j] + lam[j][:, None, None] * G
        cot = chain_backward(torch.from_numpy(G), combine, rank, world)
        # serial reference: total cotangent of the end slot of this range
        T = np.zeros_like(S[0])
        for j in range(n - 1, hi - 1, -1):
            T = dA[j] + lam[j][:, None, None] * T
        if rank == world - 1:
            assert cot is None
        else:
            np.testing.assert_allclose(cot.numpy(), T, rtol=1e-12, atol=1e-12)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sp_carry_chains_gloo(world):
    mp.spawn(_worker, args=(world, _free_port(), 6 * world), nprocs=world, join=True)


def _subgroup_worker(rank, world, port):
    """A chain over the subgroup {1, 2} of a 3-process job (rank 0 is not in
    it): the group ranks must map to the right global peers."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_04239_b200.parallel import chain_backward, chain_forward

        grp = dist.new_group([1, 2])
        if rank == 0:
            return
        gr = dist.get_rank(grp)
        local = torch.full((4,), float(10 * rank))

        def combine(carry, loc):
            return loc if carry is None else 0.5 * carry + loc

        carry = chain_forward(local, combine, gr, 2, grp)
        back = chain_backward(local, combine, gr, 2, grp)
        if gr == 0:
            assert carry is None and torch.equal(back, torch.full((4,), 20.0))
        else:
            assert torch.equal(carry, torch.full((4,), 10.0)) and back is None
    finally:
        dist.destroy_process_group()


def test_sp_chain_on_subgroup_without_rank0():
    mp.spawn(_subgroup_worker, args=(3, _free_port()), nprocs=3, join=True)


def test_sp_partition_math_cpu():
    from paper_2507_04239_b200.parallel import SpPartition

    p = SpPartition(1, 2, 4096, 1024)
    assert (p.chunk0, p.local_chunks, p.t0, p.t_local) == (2, 2, 2048, 2048)
