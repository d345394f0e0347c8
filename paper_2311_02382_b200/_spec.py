"""Sequence ownership (reference sharded.py:37-61, 84-88): which contiguous block
of the sequence a worker owns.  Bit-exact with the reference (tests/test_host.py)."""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import PartitionError, ShapeError


@dataclass(frozen=True)
class ShardSpec:
    """sharded.py:37-61: which contiguous block of the sequence a worker owns."""

    rank: int
    workers: int
    seq_len: int

    def __post_init__(self) -> None:
        if self.workers < 1:
            raise ValueError("worker count must be positive")
        if not 0 <= self.rank < self.workers:
            raise ValueError(f"rank {self.rank} outside worker range [0, {self.workers})")
        if self.seq_len % self.workers != 0:
            raise PartitionError(f"sequence length {self.seq_len} not divisible by {self.workers} workers")

    @property
    def block(self) -> int:
        return self.seq_len // self.workers

    @property
    def offset(self) -> int:
        return self.rank * self.block


def slice_batch(x: torch.Tensor, spec: ShardSpec) -> torch.Tensor:
    """sharded.py:84-88: this worker's rows [offset, offset+block) along dim 1."""
    if x.shape[1] != spec.seq_len:
        raise ShapeError(f"expected {spec.seq_len} columns, got {x.shape[1]}")
    return x[:, spec.offset:spec.offset + spec.block].contiguous()
