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


def make_groups(layout: GridLayout):
    """Create the torch.distributed sequence and data groups (every rank must call
    this, in the same order).  Returns (my_seq_group, my_data_group, world_group)."""
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


def run_steps(engine, comm, batches, opt, *, layer: int = 0):
    """Drive ``len(batches)`` training steps of ONE rank of a D x N grid
    (hybrid.run_steps / train_step, hybrid.py:95-126, 140-190, at layer level):
    each step runs the layer forward + backward with the folded gradient
    all-reduce (sequence x data, scale 1/(D*N) in the kernels) and then the
    optimizer update of the bound parameters (``engine.bind_params``).

    ``batches[s]`` = (x_seg, grad_y_seg) of this rank's sequence block.
    Returns the post-sync gradient norm of every step (HybridRun.grad_norms,
    folded in fp64 like model.grad_norm)."""
    import torch

    norms = []
    for s, (x, gy) in enumerate(batches):
        engine.step(x, gy, comm, step=s, layer=layer)
        norms.append(float(torch.linalg.vector_norm(engine.grads.double())))
        engine.optimizer_step(opt)
    return norms
