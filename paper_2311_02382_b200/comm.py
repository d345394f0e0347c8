"""Collectives of the LSS hot path, with the reference's ledger semantics.

Reference: collectives.py (Communicator.all_gather / reduce_scatter /
all_reduce, 325-406; CommLedger, 52-143).  On B200 the fabric is NCCL over
NVLink 5 / NVSwitch via torch.distributed (one process per GPU).  Per LSS
layer and step the path issues exactly:

  forward   1 all-gather of the packed [K_r | V_r] segments      (phase "forward")
  backward  1 reduce-scatter of the packed partial [dK | dV]      (phase "backward")
  sync      1 all-reduce (sum) of the pre-scaled gradients        (phase "sync")

On one NVLink/NVSwitch domain the backward reduce-scatter is FUSED into the
attention backward kernel (lss_attn_bwd_p2p): each key segment's partial
[dK | dV] is stored straight into its owner's receive slot through CUDA IPC
peer memory, overlapped with the math; ``peer_addresses`` maps the slots and
``device_barrier`` (a one-element all-reduce) orders the peers' stores before
the owner's slot sum.  The ledger still records one "reduce-scatter" per step
(group "<seq>:nvlink"), plus the barrier.

The packed exchange is the arithmetic of the reference's ``fused=False``
ablation (sharded.py:144-154, 192-202) done as ONE collective per direction;
the ledger records it as one call whose element count is the full logical
payload (2*B*l*E), like collectives.py:341/369.

``SimComm`` is the single-process fabric used by the GPU tests to run G
virtual ranks on one device (the role the reference's in-process
Communicator plays): rank-ordered concatenation / ascending-rank sums.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .errors import CommAborted


@dataclass
class LedgerRecord:
    kind: str
    group: str
    elements: int
    step: int
    phase: str
    layer: int | None


@dataclass
class Ledger:
    """collectives.CommLedger (collectives.py:52-143), Python-side log of NCCL calls."""

    records: list = field(default_factory=list)

    def record(self, kind, group, elements, step, phase, layer=None):
        self.records.append(LedgerRecord(kind, group, int(elements), step, phase, layer))

    def count(self, kind=None, phase=None):
        return sum(1 for r in self.records
                   if (kind is None or r.kind == kind) and (phase is None or r.phase == phase))

    def clear(self):
        self.records.clear()


class TorchDistComm:
    """NCCL (or gloo on CPU tests) through torch.distributed.

    ``seq_group``: the sequence-parallel group of this rank (ranks ordered by
    sequence segment); ``world_group``: every rank that shares the parameters
    (seq x data), used for the single folded gradient all-reduce."""

    def __init__(self, seq_group=None, world_group=None, ledger: Ledger | None = None,
                 seq_name="sequence", world_name="world", *, use_flags: bool = True, timeout: float = 60.0,
                 bounded_waits="kernel"):
        import torch.distributed as dist

        self.dist = dist
        self.seq_group = seq_group
        self.world_group = world_group
        self.ledger = ledger if ledger is not None else Ledger()
        self.seq_name, self.world_name = seq_name, world_name
        self.seq_size = dist.get_world_size(seq_group)
        self.seq_rank = dist.get_rank(seq_group)
        self._peers = {}
        self._flag = None
        self._board = None     # flag words [channel][source rank] of every rank (stream signals)
        self._seq = {}
        # cross-GPU dependencies as stream-signal flag boards over IPC (no NCCL kernel);
        # False restores NCCL's one-element all-reduce barrier
        self.use_flags = use_flags
        # a peer that never signals: every wait on a flag gives up after `timeout` ->
        # CommTimeout, and abort() releases them at once -> CommAborted.  Stream waits
        # (same-box A/B at N=2 / 4): "kernel" (default) = a one-warp spin
        # kernel on the waiting stream, 11.54 / 5.86-5.90 ms per step; "guarded" =
        # front-end cuStreamWaitValue32 + a guard kernel on a high-priority stream that
        # releases the flags on failure, 11.63-11.70 / 6.07; "frontend" = unbounded
        # cuStreamWaitValue32, 11.44-11.48 / 5.88-5.92.  The attention kernels'
        # in-kernel waits always carry the deadline.
        self.timeout = timeout
        self.waits = {True: "kernel", False: "frontend"}.get(bounded_waits, bounded_waits)
        self._aborted = None

    def _ipc_capable(self) -> bool:
        """CUDA IPC data plane available: GPU processes whose process group is NCCL, or
        gloo (e.g. several ranks per GPU, which NCCL refuses) -- the peer mapping then
        decides per pair (same node, P2P or same device)."""
        return torch.cuda.is_available() and self.dist.get_backend(self.seq_group) in ("nccl", "gloo")

    def peer_addresses(self, t: torch.Tensor):
        """Device addresses, in this process, of every sequence-group rank's copy of
        ``t`` (same shape everywhere), mapped through CUDA IPC; None when some pair
        of ranks cannot reach each other's memory (other node, no P2P, gloo/CPU)."""
        key = (t.data_ptr(), t.numel())
        if key in self._peers:
            hit = self._peers[key]
            return None if hit is None else hit[0]
        if not t.is_cuda or not self._ipc_capable() or self.seq_size == 1:
            return None
        import socket

        from . import kernels as K

        dev = t.device.index
        try:  # legacy CUDA IPC cannot export e.g. expandable-segment / cudaMallocAsync memory
            handle, off = K.ipc_export(t)
        except Exception:  # noqa: BLE001 - contribute None: every rank then falls back together
            handle, off = None, 0
        info = [None] * self.seq_size
        self.dist.all_gather_object(info, (socket.gethostname(), dev, handle, off), group=self.seq_group)
        ok = all(hd is not None for _, _, hd, _ in info)
        ok = ok and all(h == info[self.seq_rank][0] for h, *_ in info)
        ok = ok and all(K.peer_access(dev, d) for r, (_, d, _, _) in enumerate(info) if r != self.seq_rank)
        addrs, opened = [], []
        if ok:
            try:
                for r, (_, _, h, o) in enumerate(info):
                    if r == self.seq_rank:
                        addrs.append(t.data_ptr())
                    else:
                        a = K.ipc_import(h, o)
                        opened.append((a, o))
                        addrs.append(a)
            except Exception:  # noqa: BLE001 - any rank failing disables the fused path for all
                ok = False
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=t.device)
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=self.seq_group)
        if not flag.item():
            for a, o in opened:
                K.ipc_close(a, o)
            self._peers[key] = None
            return None
        self._peers[key] = (addrs, t)  # keep the tensor alive while peers may write into it
        return addrs

    def map_named(self, named: dict):
        """Collective: every rank contributes {name: tensor or None}; returns, per rank,
        {name: device address in this process} (own tensors: their pointers; peers':
        CUDA IPC mappings), or None when some pair of ranks cannot map each other."""
        if not self._ipc_capable() or self.seq_size == 1:
            return None
        import socket

        from . import kernels as K

        dev = torch.cuda.current_device()
        try:  # an export failure disables the path on every rank (no rank left blocked below)
            mine = {n: (K.ipc_export(t) if t is not None else None) for n, t in named.items()}
        except Exception:  # noqa: BLE001
            mine = None
        info = [None] * self.seq_size
        self.dist.all_gather_object(info, (socket.gethostname(), dev, mine), group=self.seq_group)
        ok = all(entries is not None for _, _, entries in info)
        ok = ok and all(h == info[self.seq_rank][0] for h, _, _ in info)
        ok = ok and all(K.peer_access(dev, d) for r, (_, d, _) in enumerate(info) if r != self.seq_rank)
        out, opened = [], []
        if ok:
            try:
                for r, (_, _, entries) in enumerate(info):
                    if r == self.seq_rank:
                        out.append({n: t.data_ptr() for n, t in named.items() if t is not None})
                        continue
                    d = {}
                    for n, e in entries.items():
                        if e is not None:
                            d[n] = K.ipc_import(*e)
                            opened.append((d[n], e[1]))
                    out.append(d)
            except Exception:  # noqa: BLE001 - any rank failing disables the path for all
                ok = False
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=torch.device("cuda", dev))
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=self.seq_group)
        if not flag.item():
            for a, o in opened:
                K.ipc_close(a, o)
            return None
        self._keep = getattr(self, "_keep", []) + [named]  # peers may write into these
        return out

    # ------------------------------------------------ stream signals (no SM, no NCCL kernel)
    N_CHANNELS = 8  # 0 forward barrier, 1 backward barrier, 2-5 F1/F2/B1/B2 hand-offs

    def flags_ready(self) -> bool:
        """Map every rank's flag board once (collective); False when unavailable."""
        if self._board is None:
            if not self.use_flags or self.seq_size == 1 or not self._ipc_capable():
                self._board = False
                return False
            from . import kernels as K

            dev = torch.device("cuda", torch.cuda.current_device())
            K.runtime_config(wait_timeout_s=self.timeout, device=dev)  # in-kernel wait deadline
            board = torch.zeros(self.N_CHANNELS * self.seq_size, dtype=torch.int32, device=dev)
            torch.cuda.synchronize()  # zeroed before any peer can signal into it
            addrs = self.map_named({"board": board})
            self._board = False if addrs is None else (board, [a["board"] for a in addrs])
        return self._board is not False

    def abort(self, exc: BaseException | None = None) -> None:
        """Communicator.abort (collectives.py:200-209): release every bounded wait of
        this process at once; later check() / steps raise CommAborted."""
        from . import kernels as K

        self._aborted = exc if exc is not None else RuntimeError("aborted")
        K.abort_waits(True)

    def check(self) -> None:
        """Raise CommAborted after abort(), CommTimeout if a wait of a previous step ran
        past its deadline (collectives.py:242-252).  Host-only, no synchronisation."""
        from . import kernels as K

        if self._aborted is not None:
            raise CommAborted("communicator aborted") from self._aborted
        if self._board:
            K.raise_status(clear=True)

    def _wait(self, base: int, count: int, skip: int, seq: int, stream=None) -> None:
        """Stream-ordered wait for flag words [base, base + 4*count) (except ``skip``)."""
        from . import kernels as K

        if self.waits == "guarded":
            K.stream_wait_guarded(base, count, skip, seq, stream)
        elif self.waits == "kernel":
            K.stream_wait_bounded(base, count, skip, seq, stream)
        else:
            for p in range(count):
                if p != skip:
                    K.stream_wait(base + 4 * p, seq, stream)

    def _flag_addr(self, rank: int, channel: int, source: int) -> int:
        return self._board[1][rank] + 4 * (channel * self.seq_size + source)

    def flag_barrier(self, channel: int, step=0, phase="backward", layer=None, stream=None):
        """Stream-ordered barrier through the flag boards: signal every peer, then wait
        for every peer's signal.  Same contract as device_barrier."""
        from . import kernels as K

        self.ledger.record("barrier", self.seq_name, 1, step, phase, layer)
        seq = self._seq[("bar", channel)] = self._seq.get(("bar", channel), 0) + 1
        me = self.seq_rank
        for p in range(self.seq_size):
            if p != me:
                K.stream_signal(self._flag_addr(p, channel, me), seq, stream)
        self._wait(self._flag_addr(me, channel, 0), self.seq_size, me, seq, stream)

    def notify(self, peer: int, channel: int, stream=None) -> None:
        """Signal `peer` on `channel` once everything enqueued on `stream` is done."""
        from . import kernels as K

        seq = self._seq[("out", channel, peer)] = self._seq.get(("out", channel, peer), 0) + 1
        K.stream_signal(self._flag_addr(peer, channel, self.seq_rank), seq, stream)

    def expect(self, peer: int, channel: int):
        """Handle whose wait() blocks the caller's current stream until `peer`'s next
        notify on `channel` (the NCCL Work.wait() contract)."""
        seq = self._seq[("in", channel, peer)] = self._seq.get(("in", channel, peer), 0) + 1
        return _FlagWait(self, self._flag_addr(self.seq_rank, channel, peer), seq)

    def push_stream(self) -> torch.cuda.Stream:
        if getattr(self, "_push_stream", None) is None:
            self._push_stream = torch.cuda.Stream(device=torch.cuda.current_device())
        return self._push_stream

    def gather_pull(self, full: torch.Tensor, step=0, layer=0, segments=None, ready=None):
        """K/V all-gather on the copy engines: after a device barrier (every rank's
        slot is written), pull each peer's own slot full[p] from its IPC-mapped
        buffer on a copy stream -- no SMs taken from the overlapped attention.
        ``segments``: the peers' slots this rank's attention actually reads (the
        causal schedule never touches the others); default all.  Returns an
        event the consumer waits on, or None when peers do not map (the caller
        then falls back to the NCCL all-gather).

        ``ready`` = (flags int32 [G], seq): fused gather -- after each segment's copy
        the copy stream signals flags[p] = seq, and the attention kernels wait per
        segment (in their TMA producer) instead of the consumer waiting on the event.
        Segments are pulled nearest-first (the order the kernels visit them)."""
        addrs = self.peer_addresses(full)
        if addrs is None:
            return None
        from . import kernels as K

        self.ledger.record("all-gather", self.seq_name + ":nvlink-ce", full.numel(), step, "forward", layer)
        cur = torch.cuda.current_stream()
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream(device=full.device)
        cs = self._copy_stream
        # barrier on the compute stream: every rank then starts its diagonal tiles
        # together, which aligns the later hand-offs (measured N=4: 6.6 ms vs 6.8
        # with the barrier on the copy stream or with the NCCL all-gather)
        if self.flags_ready() and self.use_flags:
            self.flag_barrier(0, step, "forward", layer)
        else:
            self.device_barrier(step, "forward", layer)
        cs.wait_stream(cur)
        slot = full[0].numel() * full.element_size()
        me = self.seq_rank
        order = sorted((p for p in (range(self.seq_size) if segments is None else segments) if p != me),
                       key=lambda p: (p > me, abs(p - me)))
        for p in order:
            K.copy_d2d(full[p].data_ptr(), addrs[p] + p * slot, slot, cs)
            if ready is not None:
                K.stream_signal(ready[0].data_ptr() + 4 * p, ready[1], cs)
        ev = torch.cuda.Event()
        ev.record(cs)
        return ev

    def device_barrier(self, step=0, phase="backward", layer=None):
        """Stream-ordered barrier of the sequence group: returns (on the device) only
        after every rank's prior work on its stream completed."""
        self.ledger.record("barrier", self.seq_name, 1, step, phase, layer)
        if self.seq_size == 1:
            return
        if self._flag is None:
            self._flag = torch.zeros(1, dtype=torch.float32, device=torch.device("cuda", torch.cuda.current_device()))
        self.dist.all_reduce(self._flag, group=self.seq_group)

    def all_gather_rows(self, full: torch.Tensor, step=0, layer=0, async_op=False):
        """In-place all-gather: ``full`` is [G, ...]; this rank's slot full[seq_rank]
        is already written; afterwards full holds every rank's slot in rank order."""
        self.ledger.record("all-gather", self.seq_name, full.numel(), step, "forward", layer)
        if self.seq_size == 1:
            return None
        return self.dist.all_gather_into_tensor(full.view(-1), full[self.seq_rank].view(-1),
                                                group=self.seq_group, async_op=async_op)

    def reduce_scatter_rows(self, out: torch.Tensor, full: torch.Tensor, step=0, layer=0, async_op=False):
        """out = sum over ranks of full[seq_rank] (rank-ordered blocks, collectives.py:346-372)."""
        self.ledger.record("reduce-scatter", self.seq_name, full.numel(), step, "backward", layer)
        if self.seq_size == 1:
            out.copy_(full[0])
            return None
        return self.dist.reduce_scatter_tensor(out.view(-1), full.view(-1), group=self.seq_group,
                                               async_op=async_op)

    def all_reduce_sum(self, buf: torch.Tensor, step=0, async_op=False):
        """Folded double gradient averaging: one world all-reduce of gradients that
        were pre-scaled by 1/(D*N) in the kernels that produced them."""
        self.ledger.record("all-reduce", self.world_name, buf.numel(), step, "sync", None)
        world = self.dist.get_world_size(self.world_group)
        if world == 1:
            return None
        return self.dist.all_reduce(buf, group=self.world_group, async_op=async_op)

    def p2p(self, sends, recvs, peer: int, step=0, phase="", layer=None, async_op=False):
        """Point-to-point exchange with sequence-group member `peer` (balanced causal
        schedule).  Stream-ordered: the current stream waits for completion, or, with
        async_op, the caller waits on the returned works when it needs the data."""
        peer_g = peer if self.seq_group is None else self.dist.get_global_rank(self.seq_group, peer)
        ops = [self.dist.P2POp(self.dist.isend, t.view(-1), peer_g, group=self.seq_group) for t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t.view(-1), peer_g, group=self.seq_group) for t in recvs]
        if sends:
            self.ledger.record("send", self.seq_name, sum(t.numel() for t in sends), step, phase, layer)
        if recvs:
            self.ledger.record("recv", self.seq_name, sum(t.numel() for t in recvs), step, phase, layer)
        works = self.dist.batch_isend_irecv(ops)
        if async_op:
            return works
        for w in works:
            w.wait()
        return None


class _FlagWait:
    """Pending stream signal (see TorchDistComm.expect)."""

    def __init__(self, comm, addr: int, seq: int):
        self.comm, self.addr, self.seq = comm, addr, seq

    def wait(self) -> None:
        self.comm._wait(self.addr, 1, -1, self.seq)


class SoloComm:
    """One rank, no process group (G = D = 1): collectives are identities."""

    seq_size = 1
    seq_rank = 0

    def __init__(self, ledger: Ledger | None = None):
        self.ledger = ledger if ledger is not None else Ledger()

    def all_gather_rows(self, full, step=0, layer=0, async_op=False):
        self.ledger.record("all-gather", "sequence", full.numel(), step, "forward", layer)

    def reduce_scatter_rows(self, out, full, step=0, layer=0, async_op=False):
        self.ledger.record("reduce-scatter", "sequence", full.numel(), step, "backward", layer)
        if out.data_ptr() != full.data_ptr():
            out.copy_(full[0])

    def all_reduce_sum(self, buf, step=0, async_op=False):
        self.ledger.record("all-reduce", "world", buf.numel(), step, "sync", None)


class SimComm:
    """G virtual ranks in one process (tests): deterministic, ascending-rank folds."""

    def __init__(self, ledger: Ledger | None = None):
        self.ledger = ledger if ledger is not None else Ledger()

    def all_gather_rows(self, fulls, step=0, layer=0):
        g = len(fulls)
        self.ledger.record("all-gather", "sequence", fulls[0].numel(), step, "forward", layer)
        for dst in range(g):
            for src in range(g):
                if src != dst:
                    fulls[dst][src].copy_(fulls[src][src])

    def reduce_scatter_rows(self, outs, fulls, step=0, layer=0):
        g = len(fulls)
        self.ledger.record("reduce-scatter", "sequence", fulls[0].numel(), step, "backward", layer)
        for r in range(g):
            acc = fulls[0][r].clone()
            for j in range(1, g):
                acc += fulls[j][r]
            outs[r].copy_(acc)

    def device_barrier(self, step=0, phase="backward", layer=None):
        self.ledger.record("barrier", "sequence", 1, step, phase, layer)

    def all_reduce_sum(self, bufs, step=0):
        self.ledger.record("all-reduce", "world", bufs[0].numel(), step, "sync", None)
        acc = bufs[0].clone()
        for b in bufs[1:]:
            acc += b
        for b in bufs:
            b.copy_(acc)
