"""CPU: the reference-signature communicator (paper_2311_02382_b200/collectives.py).

Ports of the reference's collective tests (tests/test_collectives.py in the
reference): rank-ordered concatenation, reduce-scatter == scatter of the
ascending-rank sum (bitwise), all-reduce mean, all_gather / reduce_scatter
adjoint pairing, one ledger record per call, and the failure semantics --
a peer that never arrives raises CommTimeout, a peer that raises surfaces its
own error, mismatched metadata aborts the group, a communicator used after an
abort raises CommAborted.  Both fabrics: worker threads of one process, and
torch.distributed (gloo, world_size 2) for the one-process-per-GPU path.
"""

import os
import socket
import time

import pytest
import torch

from paper_2311_02382_b200.collectives import Communicator, DistCommunicator, run_workers
from paper_2311_02382_b200.errors import CommAborted, CommTimeout, PartitionError


def _shards(world, shape=(2, 3, 4), dtype=torch.float64):
    return [torch.arange(int(torch.tensor(shape).prod()), dtype=dtype).view(shape) + 100 * r for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3])
def test_thread_collectives_semantics(world):
    comm = Communicator(world, timeout=10.0)
    group = comm.group("sequence", tuple(range(world)))
    xs = _shards(world)
    g = torch.Generator().manual_seed(7)
    ys = [torch.randn(2, 3 * world, 4, generator=g, dtype=torch.float64) for _ in range(world)]

    def worker(rank):
        full = comm.all_gather(group, rank, xs[rank], dim=1, step=0, phase="forward", layer=0)
        rs = comm.reduce_scatter(group, rank, ys[rank], dim=1, step=0, phase="backward", layer=0)
        mean = comm.all_reduce_mean(group, rank, xs[rank], step=0, phase="sync")
        total = comm.all_reduce(group, rank, xs[rank], op="sum", step=0, phase="sync")
        comm.barrier(group, rank)
        return full, rs, mean, total

    res = run_workers(world, worker, comm=comm)
    want_full = torch.cat(xs, dim=1)
    acc = ys[0].clone()
    for y in ys[1:]:
        acc += y  # ascending rank order
    blocks = torch.tensor_split(acc, world, dim=1)
    for r, (full, rs, mean, total) in enumerate(res):
        assert torch.equal(full, want_full)
        assert torch.equal(rs, blocks[r])  # bitwise: same fold order
        assert torch.equal(total, sum(xs[1:], xs[0].clone()))
        assert torch.allclose(mean, total / world)
    kinds = [rec.kind for rec in comm.ledger.records]
    assert kinds == ["all-gather", "reduce-scatter", "all-reduce", "all-reduce"]  # one record per call
    assert comm.ledger.records[0].elements == want_full.numel()


def test_thread_adjoint_pairing():
    """<AG(x), y> == <x, RS(y)>: the backward of the gather is the reduce-scatter."""
    world = 3
    comm = Communicator(world)
    group = comm.group("sequence", range(world))
    g = torch.Generator().manual_seed(1)
    xs = [torch.randn(2, 4, generator=g, dtype=torch.float64) for _ in range(world)]
    ys = [torch.randn(2, 4 * world, generator=g, dtype=torch.float64) for _ in range(world)]

    def worker(rank):
        ag = comm.all_gather(group, rank, xs[rank], dim=1, step=0, phase="forward")
        rs = comm.reduce_scatter(group, rank, ys[rank], dim=1, step=0, phase="backward")
        return float((ag * ys[rank]).sum()), float((xs[rank] * rs).sum())

    res = run_workers(world, worker, comm=comm)
    lhs, rhs = sum(a for a, _ in res), sum(b for _, b in res)
    assert abs(lhs - rhs) < 1e-10 * max(1.0, abs(lhs))


def test_thread_peer_never_arrives_times_out():
    comm = Communicator(2, timeout=0.3)
    group = comm.group("sequence", (0, 1))

    def worker(rank):
        if rank == 1:
            time.sleep(1.0)
            return None
        return comm.all_reduce_mean(group, rank, torch.ones(3), step=0, phase="sync")

    t0 = time.monotonic()
    with pytest.raises(CommTimeout):
        run_workers(2, worker, comm=comm)
    assert time.monotonic() - t0 < 5


def test_thread_peer_error_surfaces_and_aborts():
    comm = Communicator(3, timeout=30.0)
    group = comm.group("sequence", (0, 1, 2))

    def worker(rank):
        if rank == 2:
            raise KeyError("boom")
        return comm.all_gather(group, rank, torch.ones(1), step=0, phase="forward")

    t0 = time.monotonic()
    with pytest.raises(KeyError, match="boom"):
        run_workers(3, worker, comm=comm)
    assert time.monotonic() - t0 < 10  # peers unwound with CommAborted, not the 30 s timeout
    with pytest.raises(CommAborted):  # use after abort
        comm.barrier(group, 0)


def test_thread_metadata_mismatch_aborts():
    comm = Communicator(2, timeout=10.0)
    group = comm.group("sequence", (0, 1))

    def worker(rank):
        return comm.all_gather(group, rank, torch.ones(1), step=rank, phase="forward")

    with pytest.raises((RuntimeError, CommAborted)):
        run_workers(2, worker, comm=comm)


def test_thread_partition_and_membership_errors():
    comm = Communicator(2)
    group = comm.group("sequence", (0, 1))
    with pytest.raises(ValueError):
        comm.group("tensor", (0, 1))
    with pytest.raises(ValueError):
        comm.group("sequence", (0, 2))

    def worker(rank):
        return comm.reduce_scatter(group, rank, torch.ones(3), dim=0, step=0, phase="backward")

    with pytest.raises(PartitionError):
        run_workers(2, worker, comm=comm)


# ---------------------------------------------------------------- torch.distributed (gloo)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dist_worker(rank, world, port, mode):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = DistCommunicator(timeout=3.0 if mode == "timeout" else 30.0)
        world_g = comm.group("world", range(world))
        if mode == "semantics":
            xs = _shards(world)
            full = comm.all_gather(world_g, rank, xs[rank], dim=1, step=0, phase="forward", layer=0)
            assert torch.equal(full, torch.cat(xs, 1))
            y = torch.full((2, 3 * world, 4), float(rank + 1), dtype=torch.float64)
            rs = comm.reduce_scatter(world_g, rank, y, dim=1, step=0, phase="backward", layer=0)
            assert rs.shape == (2, 3, 4) and torch.all(rs == sum(range(1, world + 1)))
            m = comm.all_reduce_mean(world_g, rank, torch.tensor([float(rank)]), step=0, phase="sync")
            assert abs(float(m) - (world - 1) / 2) < 1e-12
            sc = comm.scatter(world_g, rank, torch.arange(8.0).view(2, 4) if rank == 0 else None, src=0, dim=1,
                              step=0, phase="forward")
            assert torch.equal(sc, torch.arange(8.0).view(2, 4).tensor_split(world, 1)[rank])
            assert [r.kind for r in comm.ledger.records] == ["all-gather", "reduce-scatter", "all-reduce", "scatter"]
        elif mode == "mismatch":
            with pytest.raises(CommAborted):
                comm.all_reduce_mean(world_g, rank, torch.ones(2), step=rank, phase="sync")
            with pytest.raises(CommAborted):  # aborted communicator
                comm.barrier(world_g, rank)
        elif mode == "timeout":
            if rank == 1:
                time.sleep(8.0)  # never joins the collective in time
            else:
                with pytest.raises(CommTimeout):
                    comm.all_reduce_mean(world_g, rank, torch.ones(2), step=0, phase="sync")
    finally:
        if mode != "timeout":
            dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["semantics", "mismatch"])
def test_dist_communicator_gloo(mode):
    import torch.multiprocessing as mp

    mp.spawn(_dist_worker, args=(2, _free_port(), mode), nprocs=2, join=True)


def test_dist_communicator_timeout_gloo():
    import torch.multiprocessing as mp

    mp.spawn(_dist_worker, args=(2, _free_port(), "timeout"), nprocs=2, join=True)
