"""CPU, multi-process (gloo, world_size 2 and 4): the N>1 host path of the LSS
exchange -- TorchDistComm's in-place packed all-gather, reduce-scatter, the
folded world all-reduce, the hybrid grid groups and the ledger schedule.
Mirrors the reference's collective tests (test_collectives.py:19-154) and
hybrid traffic/averaging tests (test_hybrid.py:100-147)."""

import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_seq(rank, world, port):
    import torch
    import torch.distributed as dist
    from paper_2311_02382_b200.comm import Ledger, TorchDistComm

    _init(rank, world, port)
    try:
        comm = TorchDistComm(None, None, Ledger())
        B, m, E = 2, 3, 4
        # packed gather: each rank writes its own slot, gathers in place
        full = torch.full((world, B, m, 2 * E), -1.0)
        own = torch.arange(B * m * 2 * E, dtype=torch.float32).view(B, m, 2 * E) + 100 * rank
        full[rank].copy_(own)
        comm.all_gather_rows(full)
        for r in range(world):
            want = torch.arange(B * m * 2 * E, dtype=torch.float32).view(B, m, 2 * E) + 100 * r
            assert torch.equal(full[r], want), "gather is not the rank-ordered concatenation"
        # reduce-scatter: rank r receives block r of the sum over ranks
        contrib = torch.stack([torch.full((B, m, 2 * E), float(10 * rank + j)) for j in range(world)])
        out = torch.empty(B, m, 2 * E)
        comm.reduce_scatter_rows(out, contrib)
        want = sum(10 * q + rank for q in range(world))
        assert torch.all(out == want)
        # adjoint pairing <AG(x), y> == <x, RS(y)>  (test_collectives.py:113-130)
        g = torch.Generator().manual_seed(rank)
        x = torch.randn(B, m, 2 * E, generator=g, dtype=torch.float64)
        y = torch.randn(world, B, m, 2 * E, generator=g, dtype=torch.float64)
        gx = torch.zeros(world, B, m, 2 * E, dtype=torch.float64)
        gx[rank].copy_(x)
        comm.all_gather_rows(gx)
        lhs = torch.tensor([(gx * y).sum().item()], dtype=torch.float64)
        rs = torch.empty(B, m, 2 * E, dtype=torch.float64)
        comm.reduce_scatter_rows(rs, y.clone())
        rhs = torch.tensor([(x * rs).sum().item()], dtype=torch.float64)
        dist.all_reduce(lhs)
        dist.all_reduce(rhs)
        assert abs(lhs.item() - rhs.item()) < 1e-9 * max(1.0, abs(lhs.item()))
        # folded sync
        grads = torch.full((7,), float(rank + 1)) / world
        comm.all_reduce_sum(grads)
        assert torch.allclose(grads, torch.full((7,), sum(range(1, world + 1)) / world))
        assert comm.ledger.count("all-gather") == 2 and comm.ledger.count("reduce-scatter") == 2
        assert comm.ledger.count("all-reduce") == 1
    finally:
        dist.destroy_process_group()


def _worker_hybrid(rank, world, port):
    import torch
    import torch.distributed as dist
    from paper_2311_02382_b200.comm import Ledger, TorchDistComm
    from paper_2311_02382_b200.hybrid import GridLayout, make_groups

    _init(rank, world, port)
    try:
        lay = GridLayout(2, 2)
        seq_g, data_g, world_g = make_groups(lay)
        comm = TorchDistComm(seq_g, world_g, Ledger())
        d, s = lay.coords(rank)
        assert comm.seq_rank == s and comm.seq_size == 2
        # per-layer traffic stays inside the sequence group (test_hybrid.py:130-147)
        full = torch.zeros(2, 3)
        full[s] = rank + 1
        comm.all_gather_rows(full)
        members = lay.seq_members(d)
        assert full[:, 0].tolist() == [members[0] + 1, members[1] + 1]
        # folded double averaging == seq-group mean then data-group mean
        g = torch.tensor([float(rank) ** 2 + 1, 3.0 * rank - 1])
        two = g.clone()
        dist.all_reduce(two, group=seq_g)
        two /= 2
        dist.all_reduce(two, group=data_g)
        two /= 2
        folded = g * lay.grad_scale
        comm.all_reduce_sum(folded)
        assert torch.allclose(folded, two, rtol=1e-6), (folded, two)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_lss_collectives_gloo(world):
    import torch.multiprocessing as mp

    mp.spawn(_worker_seq, args=(world, _free_port()), nprocs=world, join=True)


def test_hybrid_grid_folded_sync_gloo():
    import torch.multiprocessing as mp

    mp.spawn(_worker_hybrid, args=(4, _free_port()), nprocs=4, join=True)
