"""The reference's communicator API (seqpar/collectives.py) over device tensors.

Same names, signatures and failure semantics as the reference so that
``sharded.forward / backward / sync`` and ``hybrid.vertical_sync`` can be
written exactly as there:

  Communicator.group(kind, members)            collectives.py:169-185
  .scatter / .gather / .all_gather / .reduce_scatter / .all_reduce /
  .all_reduce_mean / .barrier(group, rank, x, *, dim, step, phase, layer)
                                               collectives.py:280-410
  .abort(exc) -> peers raise CommAborted        collectives.py:200-209
  a peer that never arrives -> CommTimeout      collectives.py:242-252
  metadata (kind, step, phase, layer) validated at every rendezvous
  one ledger record per call, elements = full logical size
  run_workers(world_size, fn, comm=)            collectives.py:414-445

Two fabrics:

* :class:`Communicator` -- worker threads of ONE process (the reference's own
  model of a job): the payloads are torch tensors (CUDA or CPU), the last
  arriver combines them exactly once, reductions fold in ascending rank order
  (bit-for-bit reproducible, collectives.py:5-7).  Used to run G sequence
  workers on one GPU in tests.
* :class:`DistCommunicator` -- one process per GPU through torch.distributed
  (NCCL over NVLink; gloo for CPU tests).  Groups are process groups created
  collectively; NCCL's reduction order is its own (tolerance-level, not
  bitwise).  A collective that does not complete within
  ``timeout`` raises CommTimeout; after :meth:`abort` every call raises
  CommAborted.

The hot engine (``sharded.LSSAttention`` / ``lss_step``) does not go through
this module: it fuses the exchanges into its kernels (comm.py).  This is the
reference-shaped boundary a caller of ``sharded.forward`` keeps using.
"""

from __future__ import annotations

import threading
import time
import zlib
from dataclasses import dataclass, field

import torch

from .comm import Ledger
from .errors import CommAborted, CommTimeout, PartitionError, ShapeError

GROUP_KINDS = {"sequence": "seq", "data": "data", "world": "world"}  # collectives.py:29


@dataclass(frozen=True)
class WorkerGroup:
    """collectives.WorkerGroup (collectives.py:33-49); ``pg`` is the torch process
    group of a DistCommunicator group (None for the thread fabric)."""

    group_id: str
    kind: str
    members: tuple
    pg: object = field(default=None, compare=False, repr=False)

    @property
    def size(self) -> int:
        return len(self.members)

    def index_of(self, rank: int) -> int:
        try:
            return self.members.index(rank)
        except ValueError:
            raise ValueError(f"rank {rank} is not a member of group {self.group_id}") from None


@dataclass(frozen=True)
class _Meta:
    kind: str
    step: int
    phase: str
    layer: object


def _split(x: torch.Tensor, parts: int, dim: int):
    if x.shape[dim] % parts != 0:
        raise PartitionError(f"dimension {dim} of size {x.shape[dim]} not divisible into {parts} blocks")
    return list(torch.tensor_split(x, parts, dim=dim))


class _CommonAPI:
    """Argument handling shared by both fabrics."""

    world_size: int
    ledger: Ledger

    def _make_group(self, kind, members):
        if kind not in GROUP_KINDS:
            raise ValueError(f"unknown group kind {kind!r}, expected one of {sorted(GROUP_KINDS)}")
        members = tuple(members)
        if len(set(members)) != len(members) or not members:
            raise ValueError("group members must be a non-empty set of distinct ranks")
        if any(r < 0 or r >= self.world_size for r in members):
            raise ValueError(f"group members {members} outside world of {self.world_size}")
        n = self._kind_counts.get(kind, 0)
        self._kind_counts[kind] = n + 1
        return GROUP_KINDS[kind] if kind == "world" else f"{GROUP_KINDS[kind]}{n}", members

    def _record(self, group: WorkerGroup, meta: _Meta, elements: int) -> None:
        self.ledger.record(meta.kind, group.group_id, int(elements), meta.step, meta.phase, meta.layer)

    def all_reduce_mean(self, group, rank, x, **kw):
        return self.all_reduce(group, rank, x, op="mean", **kw)


class Communicator(_CommonAPI):
    """In-process rendezvous hub (collectives.Communicator) over torch tensors."""

    def __init__(self, world_size: int, *, timeout: float = 60.0) -> None:
        if world_size < 1:
            raise ValueError("world_size must be at least 1")
        self.world_size = world_size
        self.ledger = Ledger()
        self._timeout = timeout
        self._slots: dict = {}
        self._kind_counts: dict = {}
        self._lock = threading.Lock()
        self._abort_exc = None

    def group(self, kind: str, members) -> WorkerGroup:
        with self._lock:
            gid, members = self._make_group(kind, members)
            self._slots[gid] = dict(cond=threading.Condition(), inbox={}, outbox={}, gen=0)
        return WorkerGroup(gid, kind, members)

    def abort(self, exc: BaseException) -> None:
        """Unblock every waiting worker; they raise CommAborted."""
        self._abort_exc = exc
        for slot in list(self._slots.values()):
            with slot["cond"]:
                slot["cond"].notify_all()

    def _check_abort(self) -> None:
        if self._abort_exc is not None:
            raise CommAborted("communicator aborted") from self._abort_exc

    def _rendezvous(self, group: WorkerGroup, rank: int, payload, meta: _Meta, combine):
        group.index_of(rank)
        slot = self._slots[group.group_id]
        with slot["cond"]:
            self._check_abort()
            if rank in slot["inbox"]:
                raise RuntimeError(f"rank {rank} deposited twice in group {group.group_id}")
            slot["inbox"][rank] = (payload, meta)
            if len(slot["inbox"]) == group.size:
                metas = {m for _, m in slot["inbox"].values()}
                if len(metas) != 1:
                    exc = RuntimeError(f"collective metadata mismatch in group {group.group_id}: "
                                       f"{sorted(map(str, metas))}")
                    self.abort(exc)
                    raise exc
                try:
                    slot["outbox"] = combine({r: p for r, (p, _) in slot["inbox"].items()})
                except BaseException as exc:
                    self.abort(exc)
                    raise
                slot["inbox"] = {}
                slot["gen"] += 1
                slot["cond"].notify_all()
            else:
                gen = slot["gen"]
                deadline = time.monotonic() + self._timeout
                while slot["gen"] == gen and self._abort_exc is None:
                    remaining = deadline - time.monotonic()
                    if remaining <= 0:
                        exc = CommTimeout(f"rank {rank} waited over {self._timeout}s in group {group.group_id}")
                        self.abort(exc)
                        raise exc
                    slot["cond"].wait(timeout=remaining)
                self._check_abort()
            return slot["outbox"][rank]

    # -- collectives (collectives.py:280-410) --

    def scatter(self, group, rank, x, *, src, dim=0, step, phase, layer=None):
        meta = _Meta("scatter", step, phase, layer)

        def combine(payloads):
            data = payloads[src]
            if data is None:
                raise ShapeError(f"scatter source rank {src} supplied no tensor")
            parts = _split(data, group.size, dim)
            self._record(group, meta, data.numel())
            return {r: parts[i].contiguous() for i, r in enumerate(group.members)}

        return self._rendezvous(group, rank, x if rank == src else None, meta, combine)

    def gather(self, group, rank, shard, *, dst, dim=0, step, phase, layer=None):
        meta = _Meta("gather", step, phase, layer)

        def combine(payloads):
            full = torch.cat([payloads[r] for r in group.members], dim=dim)
            self._record(group, meta, full.numel())
            return {r: (full if r == dst else None) for r in group.members}

        return self._rendezvous(group, rank, shard, meta, combine)

    def all_gather(self, group, rank, shard, *, dim=0, step, phase, layer=None):
        """Concatenate shards in rank order; every member receives the result."""
        meta = _Meta("all-gather", step, phase, layer)

        def combine(payloads):
            full = torch.cat([payloads[r] for r in group.members], dim=dim)
            self._record(group, meta, full.numel())
            return {r: full for r in group.members}

        return self._rendezvous(group, rank, shard, meta, combine)

    def _sum(self, group, payloads):
        shapes = {tuple(payloads[r].shape) for r in group.members}
        if len(shapes) != 1:
            raise ShapeError(f"contributions disagree on shape: {shapes}")
        acc = payloads[group.members[0]].clone()
        for r in group.members[1:]:  # ascending rank order (collectives.py:365-367)
            acc += payloads[r]
        return acc

    def reduce_scatter(self, group, rank, x, *, dim=0, step, phase, layer=None):
        """Sum full-size contributions (ascending rank), member i gets block i."""
        meta = _Meta("reduce-scatter", step, phase, layer)

        def combine(payloads):
            acc = self._sum(group, payloads)
            parts = _split(acc, group.size, dim)
            self._record(group, meta, acc.numel())
            return {r: parts[i].contiguous() for i, r in enumerate(group.members)}

        return self._rendezvous(group, rank, x, meta, combine)

    def all_reduce(self, group, rank, x, *, op="mean", step, phase, layer=None):
        if op not in ("mean", "sum"):
            raise ValueError(f"unknown all_reduce op {op!r}")
        meta = _Meta("all-reduce", step, phase, layer)

        def combine(payloads):
            acc = self._sum(group, payloads)
            if op == "mean":
                acc = acc / group.size
            self._record(group, meta, acc.numel())
            return {r: acc for r in group.members}

        return self._rendezvous(group, rank, x, meta, combine)

    def barrier(self, group, rank) -> None:
        self._rendezvous(group, rank, None, _Meta("barrier", -1, "sync", None), lambda p: {r: None for r in p})


def run_workers(world_size: int, fn, *, comm: Communicator | None = None) -> list:
    """collectives.run_workers (collectives.py:414-445): ``fn(rank)`` on one thread
    per rank; the first worker exception aborts the communicator (peers unwind
    with CommAborted) and the primary error is re-raised here."""
    results = [None] * world_size
    errors = []
    lock = threading.Lock()
    dev = torch.cuda.current_device() if torch.cuda.is_available() else None

    def body(rank: int) -> None:
        try:
            if dev is not None:
                torch.cuda.set_device(dev)  # worker threads share the caller's device
            results[rank] = fn(rank)
        except BaseException as exc:  # noqa: BLE001 - must not kill the process silently
            with lock:
                errors.append((rank, exc))
            if comm is not None:
                comm.abort(exc)

    threads = [threading.Thread(target=body, args=(r,), name=f"worker-{r}") for r in range(world_size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        errors.sort(key=lambda pair: pair[0])
        primary = [e for _, e in errors if not isinstance(e, CommAborted)]
        raise primary[0] if primary else errors[0][1]
    return results


class DistCommunicator(_CommonAPI):
    """The same API over torch.distributed: one process per rank (world rank ==
    ``dist.get_rank()``), NCCL for CUDA tensors, gloo for CPU tensors.

    ``validate``: check (kind, step, phase, layer) across the group at every call
    (one extra 4-word all-reduce, default on for gloo, off for NCCL where the hot
    path must not pay a host round trip).  ``timeout`` bounds every call (the
    process groups are created with it); a timed-out call raises CommTimeout and
    aborts the communicator."""

    def __init__(self, *, timeout: float = 60.0, validate: bool | None = None) -> None:
        import torch.distributed as dist

        if not dist.is_initialized():
            raise RuntimeError("DistCommunicator needs torch.distributed.init_process_group first")
        self.dist = dist
        self.world_size = dist.get_world_size()
        self.rank = dist.get_rank()
        self.ledger = Ledger()
        self._timeout = timeout
        self._kind_counts: dict = {}
        self._abort_exc = None
        self.backend = dist.get_backend()
        self.validate = (self.backend == "gloo") if validate is None else validate

    def group(self, kind: str, members) -> WorkerGroup:
        """Collective: every rank creates every group, in the same order
        (torch.distributed.new_group); members outside the group get a handle too."""
        from datetime import timedelta

        gid, members = self._make_group(kind, members)
        pg = self.dist.new_group(list(members), timeout=timedelta(seconds=self._timeout))
        return WorkerGroup(gid, kind, members, pg)

    def abort(self, exc: BaseException) -> None:
        self._abort_exc = exc

    def _call(self, group: WorkerGroup, rank: int, meta: _Meta, fn):
        if self._abort_exc is not None:
            raise CommAborted("communicator aborted") from self._abort_exc
        group.index_of(rank)
        if rank != self.rank:
            raise ValueError(f"rank {rank} is not this process (world rank {self.rank})")
        try:
            if self.validate:
                self._check_meta(group, meta)
            return fn()
        except (CommAborted, ShapeError, PartitionError):
            raise
        except Exception as exc:  # noqa: BLE001 - map backend failures onto the reference's errors
            text = str(exc).lower()
            err = CommTimeout(f"rank {rank}: {meta.kind} in group {group.group_id} did not complete within "
                              f"{self._timeout}s") if ("timeout" in text or "timed out" in text) else \
                CommAborted(f"rank {rank}: {meta.kind} in group {group.group_id} failed: {exc}")
            self.abort(err)
            raise err from exc

    def _check_meta(self, group, meta: _Meta) -> None:
        h = zlib.crc32(repr((meta.kind, meta.step, meta.phase, meta.layer)).encode()) & 0x7FFFFFFF  # process-stable
        t = torch.tensor([h, -h], dtype=torch.int64, device=self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=group.pg)
        if int(t[0]) != h or int(-t[1]) != h:  # some member called with other (kind, step, phase, layer)
            err = CommAborted(f"collective metadata mismatch in group {group.group_id} at {meta}")
            self.abort(err)
            raise err

    def _dev(self):
        return torch.device("cuda", torch.cuda.current_device()) if self.backend == "nccl" else torch.device("cpu")

    def all_gather(self, group, rank, shard, *, dim=0, step, phase, layer=None):
        meta = _Meta("all-gather", step, phase, layer)

        def run():
            s = shard.contiguous()
            out = torch.empty((group.size,) + tuple(s.shape), dtype=s.dtype, device=s.device)
            self.dist.all_gather_into_tensor(out.view(-1), s.view(-1), group=group.pg)
            full = torch.cat(out.unbind(0), dim=dim) if dim != 0 or s.dim() == 0 else \
                out.view((group.size * s.shape[0],) + tuple(s.shape[1:]))
            self._record(group, meta, full.numel())
            return full

        return self._call(group, rank, meta, run)

    def reduce_scatter(self, group, rank, x, *, dim=0, step, phase, layer=None):
        meta = _Meta("reduce-scatter", step, phase, layer)

        def run():
            parts = _split(x, group.size, dim)
            stacked = torch.stack([p.contiguous() for p in parts])
            if self.backend == "gloo":  # gloo has no reduce-scatter: all-reduce, keep own block
                self.dist.all_reduce(stacked, group=group.pg)
                out = stacked[group.index_of(rank)].clone()
            else:
                out = torch.empty_like(stacked[0])
                self.dist.reduce_scatter_tensor(out.view(-1), stacked.view(-1), group=group.pg)
            self._record(group, meta, x.numel())
            return out

        return self._call(group, rank, meta, run)

    def all_reduce(self, group, rank, x, *, op="mean", step, phase, layer=None):
        if op not in ("mean", "sum"):
            raise ValueError(f"unknown all_reduce op {op!r}")
        meta = _Meta("all-reduce", step, phase, layer)

        def run():
            out = x.clone()
            self.dist.all_reduce(out, group=group.pg)
            if op == "mean":
                out /= group.size
            self._record(group, meta, out.numel())
            return out

        return self._call(group, rank, meta, run)

    def scatter(self, group, rank, x, *, src, dim=0, step, phase, layer=None):
        meta = _Meta("scatter", step, phase, layer)

        def run():
            group.index_of(src)
            if rank == src and x is None:
                raise ShapeError(f"scatter source rank {src} supplied no tensor")
            hdr = [(tuple(x.shape), x.dtype) if rank == src else None]
            self.dist.broadcast_object_list(hdr, src=src, group=group.pg)
            shp, dt = hdr[0]
            full = x.contiguous() if rank == src else torch.empty(shp, dtype=dt, device=self._dev())
            self.dist.broadcast(full, src, group=group.pg)
            self._record(group, meta, full.numel())
            return _split(full, group.size, dim)[group.index_of(rank)].contiguous()

        return self._call(group, rank, meta, run)

    def gather(self, group, rank, shard, *, dst, dim=0, step, phase, layer=None):
        full = self.all_gather(group, rank, shard, dim=dim, step=step, phase=phase, layer=layer)
        rec = self.ledger.records[-1]
        rec.kind = "gather"
        return full if rank == dst else None

    def barrier(self, group, rank) -> None:
        meta = _Meta("barrier", -1, "sync", None)
        self._call(group, rank, meta, lambda: self.dist.barrier(group=group.pg))


__all__ = ["GROUP_KINDS", "WorkerGroup", "Communicator", "DistCommunicator", "run_workers"]
