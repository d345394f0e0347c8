"""D x N hybrid grid: D data-parallel replicas of an N-worker LSS sequence group
(reference: seqpar/hybrid.py).

Rank layout is replica-major, exactly as GridLayout (hybrid.py:36-61): world
rank = d*N + s; sequence group d = [d*N, (d+1)*N); data group s =
{s, N+s, 2N+s, ...}.  Per-layer traffic (the K/V all-gather and the dK/dV
reduce-scatter) stays inside the sequence group (test_hybrid.py:130-147).

The reference averages gradients twice per step: over the sequence group
(sharded.sync, PE excluded) and then over the data group
(hybrid.vertical_sync, hybrid.py:76-92).  For every replicated parameter the
composition is (1/D) sum_d (1/N) sum_n g = (1/(D*N)) sum_{d,n} g, so the B200
path produces each gradient pre-scaled by 1/(D*N) inside the kernel that
writes it and issues ONE world all-reduce (sum) -- the paper's "double
gradient averaging" folded into a single collective.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import model
from .dropout import as_policy


@dataclass(frozen=True)
class GridLayout:
    """hybrid.GridLayout (hybrid.py:36-61)."""

    replicas: int
    seq_workers: int

    def __post_init__(self) -> None:
        if self.replicas < 1 or self.seq_workers < 1:
            raise ValueError("grid dimensions must be positive")

    @property
    def world(self) -> int:
        return self.replicas * self.seq_workers

    def coords(self, rank: int) -> tuple[int, int]:
        """(replica index, sequence index) of a world rank."""
        return divmod(rank, self.seq_workers)

    def seq_members(self, replica: int) -> tuple[int, ...]:
        base = replica * self.seq_workers
        return tuple(range(base, base + self.seq_workers))

    def data_members(self, seq_index: int) -> tuple[int, ...]:
        return tuple(seq_index + d * self.seq_workers for d in range(self.replicas))

    @property
    def grad_scale(self) -> float:
        """Pre-scale that folds both averaging steps into one world sum."""
        return 1.0 / self.world


def make_groups(comm_or_layout, layout: GridLayout | None = None):
    """Two forms.

    ``make_groups(comm, layout)`` -- hybrid.make_groups (hybrid.py:64-73): every
    sequence group (indexed by replica) and data group (indexed by sequence
    position) of a :mod:`collectives` communicator, as two lists.

    ``make_groups(layout)`` -- for the resident engine: create the torch.distributed
    sequence and data process groups (every rank must call this, in the same
    order); returns (my_seq_group, my_data_group, world_group)."""
    if layout is not None:
        comm = comm_or_layout
        seq_groups = [comm.group("sequence", layout.seq_members(d)) for d in range(layout.replicas)]
        data_groups = [comm.group("data", layout.data_members(s)) for s in range(layout.seq_workers)]
        return seq_groups, data_groups
    layout = comm_or_layout
    import torch.distributed as dist

    rank = dist.get_rank()
    if dist.get_world_size() != layout.world:
        raise ValueError(f"world size {dist.get_world_size()} != grid {layout.world}")
    my_seq = my_data = None
    for d in range(layout.replicas):
        g = dist.new_group(list(layout.seq_members(d)))
        if rank in layout.seq_members(d):
            my_seq = g
    for s in range(layout.seq_workers):
        g = dist.new_group(list(layout.data_members(s)))
        if rank in layout.data_members(s):
            my_data = g
    return my_seq, my_data, dist.group.WORLD


def run_engine_steps(engine, comm, batches, opt, *, layer: int = 0, policy=None, replica: int = 0):
    """Drive ``len(batches)`` training steps of ONE rank of a D x N grid on the
    resident engine (hybrid.run_steps / train_step, hybrid.py:95-126, 140-190, at
    layer level): each step runs the layer forward + backward with the folded
    gradient all-reduce (sequence x data, scale 1/(D*N) in the kernels) and then
    the optimizer update of the bound parameters (``engine.bind_params``).

    ``batches[s]`` = (x_seg, grad_y_seg) of this rank's sequence block.  The
    dropout policy of step s is ``policy.at_step(s).fork(replica)`` as in the
    reference runner (hybrid.py:172-174).  Returns the post-sync gradient norm of
    every step (HybridRun.grad_norms, folded in fp64 like model.grad_norm)."""
    base = as_policy(policy)
    norms = []
    for s, (x, gy) in enumerate(batches):
        pol = base.at_step(s).fork(replica) if base.active else None
        engine.step(x, gy, comm, step=s, layer=layer, policy=pol)
        norms.append(float(torch.linalg.vector_norm(engine.grads.double())))
        engine.optimizer_step(opt)
    return norms


# ------------------------------------------------------------ the reference's functions, same signatures


def vertical_sync(comm, data_group, rank: int, grads, loss: float, *, step: int = 0):
    """hybrid.vertical_sync (hybrid.py:76-92): average every gradient (position rows
    included) and the loss over the replicas sharing this sequence block."""
    arrays = grads.arrays()
    flat = model.flatten_arrays(arrays)
    vec = torch.cat([flat, torch.tensor([float(loss)], dtype=flat.dtype, device=flat.device)])
    out = comm.all_reduce_mean(data_group, rank, vec, step=step, phase="sync")
    return grads.replace_arrays(model.unflatten_like(out[:-1], arrays)), float(out[-1])


def train_step(comm, seq_group, data_group, dist, cfg, tokens_seg, targets_seg, *, lr: float, policy=None,
               step: int = 0, fused: bool = True):
    """hybrid.train_step (hybrid.py:95-126): sequence-group forward / backward /
    sync, then the data-group vertical sync, then SGD.  Returns (grid-mean loss,
    counters, synced grads)."""
    from . import sharded
    from .tensor import StepCounters

    rank = seq_group.members[dist.spec.rank]
    counters = StepCounters()
    partial, cache = sharded.forward(comm, seq_group, dist, cfg, tokens_seg, targets_seg, policy=policy, step=step,
                                     counters=counters, fused=fused)
    grads = sharded.backward(comm, seq_group, dist, cfg, cache, step=step)
    grads, replica_loss = sharded.sync(comm, seq_group, rank, grads, step=step, extra=partial)
    grads, grid_loss = vertical_sync(comm, data_group, rank, grads, replica_loss, step=step)
    dist.params = model.sgd_step(dist.params, grads, lr)
    return grid_loss, counters, grads


@dataclass
class HybridRun:
    """hybrid.HybridRun (hybrid.py:129-137)."""

    comm: object
    layout: GridLayout
    workers: list
    step_losses: list
    counters: list
    grad_norms: list
    last_grads: list | None


def run_steps(cfg, params_full, layout: GridLayout, batches, *, lr: float, policy=None, fused: bool = True,
              keep_last_grads: bool = False, timeout: float = 60.0) -> HybridRun:
    """hybrid.run_steps (hybrid.py:140-190): ``len(batches)`` steps on a D x N grid
    of worker threads on the current GPU; ``batches[s][d]`` is replica d's
    full-width (tokens, targets) of step s."""
    from . import sharded
    from .collectives import Communicator, run_workers

    for row in batches:
        if len(row) != layout.replicas:
            raise ValueError(f"each step needs {layout.replicas} replica batches, got {len(row)}")
    comm = Communicator(layout.world, timeout=timeout)
    seq_groups, data_groups = make_groups(comm, layout)
    base = as_policy(policy)

    def worker(rank: int):
        replica, seq_index = layout.coords(rank)
        spec = sharded.ShardSpec(seq_index, layout.seq_workers, cfg.seq_len)
        dist = sharded.shard_params(params_full, spec)
        losses, counts, norms, grads_out = [], [], [], None
        for s, row in enumerate(batches):
            tokens, targets = row[replica]
            pol = base.at_step(s).fork(replica) if base.active else base
            loss, counters, grads = train_step(comm, seq_groups[replica], data_groups[seq_index], dist, cfg,
                                               sharded.slice_batch(tokens, spec), sharded.slice_batch(targets, spec),
                                               lr=lr, policy=pol, step=s, fused=fused)
            if keep_last_grads and s == len(batches) - 1:
                grads_out = grads
            losses.append(loss)
            counts.append(counters)
            norms.append(model.grad_norm(grads))
        return dist, losses, counts, norms, grads_out

    res = run_workers(layout.world, worker, comm=comm)
    return HybridRun(comm, layout, [r[0] for r in res], res[0][1], [r[2] for r in res], [r[3] for r in res],
                     [r[4] for r in res] if keep_last_grads else None)
