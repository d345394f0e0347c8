"""The LSS engine: one rank's attention sublayer (optionally the complete layer)
with every buffer resident in HBM, and the drivers that run a step over a
sequence group (reference: seqpar/sharded.py forward / backward / sync, with
model.layer_fwd / layer_bwd's attention half, model.py:442-448 / 479-486).

Per layer and step:

  forward   LN1 -> one tcgen05 GEMM writes Q locally and [K_r|V_r] straight into
            this rank's slot of the packed gather buffer -> ONE all-gather ->
            segment attention (tcgen05 flash kernel) -> out-projection with the
            residual fused in the epilogue.
  backward  out-projection dgrad/wgrad -> attention backward writes this rank's
            partial [dK|dV] for the whole sequence -> ONE reduce-scatter ->
            fused cast/bias-sum -> dgrad/wgrad of [Wq|Wk|Wv] -> LN1 backward
            fused with the residual.
  sync      every gradient is produced pre-scaled by 1/(D*N) in the kernel that
            writes it, so ONE world all-reduce (sum) equals the reference's
            sequence-group mean followed by the data-group mean
            (sharded.sync 219-244 + hybrid.vertical_sync 76-92).

The engine issues no host synchronisation; all compute is liblss.so kernels on
the current stream.  Execution choices are explicit (:class:`EngineOptions`).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, fields

import torch

from . import kernels as K
from ._spec import ShardSpec, slice_batch  # noqa: F401  (re-exported)
from .balance import BalancePlan, block_pairs, choose_fwd_splits, make_plan
from .comm import Ledger, SimComm, TorchDistComm  # noqa: F401
from .dropout import as_policy
from .errors import ShapeError, UnsupportedError
from .model import LayerParams, LinearParams, ModelConfig

GRAD_NAMES = ("ln1_gain", "ln1_bias", "attn_q.weight", "attn_q.bias", "attn_k.weight", "attn_k.bias",
              "attn_v.weight", "attn_v.bias", "attn_out.weight", "attn_out.bias")


@dataclass(frozen=True)
class EngineOptions:
    """Execution choices of the engine.  The defaults are the measured-best
    production path (each has a same-box A/B in DESIGN.md §4/§6); the others
    exist for those A/Bs and for diagnostics.  Nothing is read from the
    environment implicitly -- :meth:`from_env` does it on request (bench / tools)."""

    balanced: bool | None = None   # balanced causal schedule (None: on for causal bf16)
    split_bias: int = 0            # BalancePlan bias_tiles (hand whole 128-row tiles to the light rank)
    fwd_split: bool = True         # key-split grids for short partial forward launches
    fused_rs: bool = True          # dK|dV reduce-scatter fused into the backward epilogue over NVLink
    ce_gather: bool = True         # K/V all-gather as copy-engine pulls of the peers' slots
    fused_gather: bool = True      # attention waits per gathered segment (gather fused into the forward)
    ce_p2p: bool = True            # balanced-schedule hand-offs as copy-engine pushes + stream flags
    b1_in_kernel: bool = True      # backward waits in-kernel for the partner's pushed dO / lse / delta
    fold_slots: bool = True        # fused-RS owner sum folded into the projection-backward cast
    wgrad_side: bool = True        # weight-gradient GEMMs on a side stream
    prefetch_at_bwd: bool = True   # step_from_host: next step's H2D issued between forward and backward
    no_overlap: bool = False       # diagnostic: serialise the gather with the compute
    phases: int = 0                # diagnostic: 1 per-phase CUDA-event timeline, 2 + cross-rank stamps

    _ENV = {"balanced": "LSS_BALANCED", "split_bias": "LSS_SPLIT_BIAS", "fwd_split": "LSS_FWD_SPLIT",
            "fused_rs": "LSS_FUSED_RS", "ce_gather": "LSS_CE_GATHER", "fused_gather": "LSS_FUSED_GATHER",
            "ce_p2p": "LSS_CE_P2P", "b1_in_kernel": "LSS_B1_IN_KERNEL", "fold_slots": "LSS_FOLD_SLOTS",
            "wgrad_side": "LSS_WGRAD_SIDE", "prefetch_at_bwd": "LSS_PREFETCH_AT_BWD",
            "no_overlap": "LSS_NO_OVERLAP", "phases": "LSS_PHASES"}

    @classmethod
    def from_env(cls, environ=None) -> "EngineOptions":
        """Options overridden by LSS_<FIELD> variables ("0"/"1", ints for split_bias /
        phases) -- for the A/B tools and bench.py, never read implicitly."""
        env = os.environ if environ is None else environ
        kw = {}
        for f in fields(cls):
            var = cls._ENV.get(f.name)
            if var is None or var not in env:
                continue
            v = env[var]
            kw[f.name] = int(v) if f.name in ("split_bias", "phases") else v != "0"
        return cls(**kw)

class LSSAttention:
    """One rank's attention sublayer with resident HBM buffers.

    cfg.seq_len is the FULL sequence length l; spec gives this rank's block.
    ``grad_scale`` = 1/(D*N) folds the two averaging steps into the kernels.
    ``balanced`` (default: on for causal bf16) enables the BalancePlan schedule.
    """

    def __init__(self, cfg: ModelConfig, spec: ShardSpec, *, grad_scale: float | None = None,
                 device=None, balanced: bool | None = None, fused_rs: bool | None = None,
                 with_ffn: bool = False, grads: torch.Tensor | None = None, split_bias: int | None = None,
                 options: EngineOptions | None = None):
        if spec.seq_len != cfg.seq_len:
            raise ShapeError(f"shard spec length {spec.seq_len} != config seq_len {cfg.seq_len}")
        self.cfg, self.spec = cfg, spec
        self.options = options if options is not None else EngineOptions()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.grad_scale = 1.0 / spec.workers if grad_scale is None else grad_scale
        B, m, G, E, H = cfg.batch, spec.block, spec.workers, cfg.embed_dim, cfg.n_heads
        self.B, self.m, self.G, self.E, self.H = B, m, G, E, H
        ad = cfg.act_dtype
        f32 = torch.float32
        dev = self.device
        mp = K.rows_pad(m)
        self.mp = mp
        z = lambda *s, dt=f32: torch.empty(*s, dtype=dt, device=dev)  # noqa: E731
        if balanced is None:
            balanced = self.options.balanced if self.options.balanced is not None else cfg.precision == "bf16"
        self.plan_bias = split_bias if split_bias is not None else self.options.split_bias
        self.balanced = bool(balanced) and cfg.precision == "bf16"
        self.plan = make_plan(spec.rank, G, m, cfg.causal, self.plan_bias) if self.balanced else BalancePlan()
        # forward
        self.xh = z(B, m, E, dt=ad)
        self.mean, self.rstd = z(B * m), z(B * m)
        self.q = z(B, m, E, dt=ad)
        self.kv_full = z(G, B, m, 2 * E, dt=ad)          # packed gather buffer (slot r = rank r)
        self.ctx = z(B, m, E, dt=ad)
        self.lse2 = z(B, H, mp)
        # partial attention of own rows over remote segments (merged into ctx); the
        # split lets the diagonal (local) segment run while the gather is in flight
        self.split_fwd = G > 1 and cfg.precision == "bf16"
        if self.split_fwd:
            self.o_tmp, self.lse_tmp = z(B, m, E, dt=ad), z(B, H, mp)
        self.y = z(B, m, E)
        # backward
        self.gy = z(B, m, E, dt=ad)
        self.dctx = z(B, m, E, dt=ad)
        self.delta = z(B, H, mp)
        self.dq = z(B, m, E)
        self.dkv_full = z(G, B, m, 2 * E)                 # partial [dK|dV] over the whole sequence
        # reduce-scatter output (own block); with one worker it IS the full buffer
        self.dkv_own = self.dkv_full[0] if G == 1 else z(B, m, 2 * E)
        self.dqkv = z(B, m, 3 * E, dt=ad)
        self.dxh = z(B, m, E)
        self.dx = z(B, m, E)
        # balanced-schedule exchange buffers
        if self.plan.role == "heavy":
            self.o_help, self.lse_help, self.dq_help = z(B, m, E, dt=ad), z(B, H, mp), z(B, m, E)
        elif self.plan.role == "light":
            self.q_peer, self.o_peer, self.lse_peer = z(B, m, E, dt=ad), z(B, m, E, dt=ad), z(B, H, mp)
            self.do_peer, self.lsef_peer, self.delta_peer = z(B, m, E, dt=ad), z(B, H, mp), z(B, H, mp)
            self.dq_peer = z(B, m, E)
        # gradients, one flat buffer: [Wq Wk Wv | Wo | bq bk bv | bo | ln_g | ln_b | extra]
        # (+ with_ffn, 64-byte aligned: [ln2_g | ln2_b | W_in | b_in | W_out | b_out])
        F = cfg.ff_dim
        self.with_ffn = with_ffn
        n_attn = 4 * E * E + 6 * E + 1
        ffn0 = (n_attn + 15) // 16 * 16  # FFN grads start 64-byte aligned (vectorised epilogues)
        n = ffn0 + (2 * E * F + F + 3 * E) if with_ffn else n_attn
        self._ffn0 = ffn0
        if grads is not None and (grads.numel() != n or grads.dtype != f32 or grads.data_ptr() % 64):
            raise ShapeError(f"external gradient buffer must be {n} fp32, 64-byte aligned")
        self.grads = grads if grads is not None else torch.zeros(n, dtype=f32, device=dev)
        self.params = None  # flat fp32 parameters in the same layout (bind_params)
        self.param_lp = None
        o = 0
        self.g_wqkv = self.grads[o:o + 3 * E * E]; o += 3 * E * E
        self.g_wo = self.grads[o:o + E * E].view(E, E); o += E * E
        self.g_bqkv = self.grads[o:o + 3 * E]; o += 3 * E
        self.g_bo = self.grads[o:o + E]; o += E
        self.g_ln_g = self.grads[o:o + E]; o += E
        self.g_ln_b = self.grads[o:o + E]; o += E
        self.g_extra = self.grads[o:o + 1]; o += 1
        if with_ffn:  # LN2 + FFN half: rank-local, same all-reduce
            o = ffn0
            self.g_ln2_g = self.grads[o:o + E]; o += E
            self.g_ln2_b = self.grads[o:o + E]; o += E
            self.g_win = self.grads[o:o + E * F].view(E, F); o += E * F
            self.g_bin = self.grads[o:o + F]; o += F
            self.g_wout = self.grads[o:o + F * E].view(F, E); o += F * E
            self.g_bout = self.grads[o:o + E]; o += E
            M = B * m
            self.mean2, self.rstd2 = z(M), z(M)
            self.yh = z(B, m, E, dt=ad)
            self.h_pre, self.h = z(M, F, dt=ad), z(M, F, dt=ad)
            self.y_out = z(B, m, E)
            self.g_out = z(M, E, dt=ad)
            self.g_pre32, self.g_pre = z(M, F), z(M, F, dt=ad)
            self.g_yh = z(M, E)
            self.grad_mid = z(B, m, E)
        self.staged = None
        self.x = None
        # fused dK|dV reduce-scatter (lss_attn_bwd_p2p): dkv_full becomes the receive
        # buffer, slot s = rank s's partial for THIS rank's segment
        if fused_rs is None:
            fused_rs = self.options.fused_rs
        self.fused_rs = bool(fused_rs) and G > 1 and cfg.precision == "bf16"
        self.seg_dst = None
        self.peer_mem = False
        self.set_dropout(None, 0)
        self._scratch = {}
        self._slots_pending = False  # fused RS slots not yet summed (folded into bwd_project's cast)
        # fused gather: per-segment arrival flags signalled by the copy stream (int32 [G])
        self._ready = torch.zeros(G, dtype=torch.int32, device=self.device) if G > 1 else None
        self._ready_seq = 0
        self._ready_tok = None  # (flags, seq, own segment) while a fused-gather forward is in flight
        self._sms = torch.cuda.get_device_properties(self.device).multi_processor_count if self.device.type == "cuda" \
            else 148
        K.ensure_runtime(self.device)  # bounded cross-GPU waits, numerics check setting

    # ------------------------------------------------------------ dropout
    def set_dropout(self, policy, layer: int) -> None:
        """Dropout policy of the next step(s) at ``layer`` (model.layer_fwd's
        ``policy, layer``): masks are keyed by global positions, so every rank (and
        the partner computing delegated rows) draws exactly the sequential masks."""
        pol = as_policy(policy)
        if pol.active and self.cfg.precision != "bf16":
            raise UnsupportedError("dropout > 0 runs on the bf16 path only (no fp32 check-mode dropout kernels)")
        self.policy, self.layer = pol, layer
        self._dd = pol.desc(layer) if pol.active else None  # score-site descriptor for the attention kernels

    def _drop_rows(self, x, out, tag: str, residual=None):
        """dropout_fwd / dropout_bwd of this rank's rows (positions offset..offset+m)."""
        pol = self.policy
        return K.dropout_rows(x, out, rows_per_sample=self.m, offset=self.spec.offset,
                              site_key=pol.site_key(self.layer, tag), thresh=pol.thresh, scale=pol.scale,
                              residual=residual)

    def _attn_part(self, q, *, rows, row0, offset, g_begin, g_end, out, lse2) -> None:
        """One partial forward launch (rows [row0, row0+rows) of q at global position
        offset + row0, key segments [g_begin, g_end)), key-split inside the launch
        when few query tiles face a long key range (choose_fwd_splits)."""
        kf, vf, common = self._fwd_common()
        S = 1
        if self.options.fwd_split:
            S = choose_fwd_splits(rows, offset + row0, g_begin, g_end, self.m, self.cfg.causal, self.B * self.H,
                                  self._sms, self.E)
        K.attn_fwd_partial(q, kf, vf, rows=rows, row0=row0, offset=offset, g_begin=g_begin, g_end=g_end, out=out,
                           lse2=lse2, splits=S, scratch=self._split_scratch(S) if S > 1 else None,
                           ready=self._ready_tok, **common)

    def _split_scratch(self, S: int):
        """Partial (O, lse) slots of the key-split forward, one set per stream (the
        split launches of two streams run concurrently)."""
        key = torch.cuda.current_stream().cuda_stream
        have = self._scratch.get(key)
        if have is None or have[0].shape[0] < S - 1:
            ad = self.cfg.act_dtype
            have = (torch.empty(S - 1, self.B, self.m, self.E, dtype=ad, device=self.device),
                    torch.empty(S - 1, self.B, self.H, self.mp, dtype=torch.float32, device=self.device))
            self._scratch[key] = have
        return have

    def _drop_tmp(self) -> torch.Tensor:
        """fp32 [B*m, E] scratch for the dropped sites (forward temp, masked gradients)."""
        if getattr(self, "_dtmp", None) is None:
            self._dtmp = torch.empty(self.B * self.m, self.E, dtype=torch.float32, device=self.device)
        return self._dtmp

    # ------------------------------------------------------------ parameters
    def load_params(self, lp: LayerParams) -> None:
        """Stage the reference-layout fp32 weights into the GEMM operand layouts."""
        self.lp = lp
        self.staged = K.stage_weights(lp.attn_q.weight, lp.attn_k.weight, lp.attn_v.weight,
                                      lp.attn_out.weight, lp.attn_q.bias, lp.attn_k.bias,
                                      lp.attn_v.bias, self.cfg.precision, bufs=self.staged)
        if self.with_ffn:
            if not lp.has_ffn:
                raise ShapeError("engine built with_ffn but the LayerParams carry no FFN half")
            ad = self.cfg.act_dtype
            self.w_in = lp.ff_in.weight.to(ad).contiguous()    # [E][F]: B operand N-major / K-major
            self.w_out = lp.ff_out.weight.to(ad).contiguous()  # [F][E]

    def _flat_views(self, buf: torch.Tensor) -> dict:
        """Named views (reference names, model.LayerParams order) into a flat buffer
        with the gradient layout."""
        E, F = self.E, self.cfg.ff_dim
        o = 0
        w = buf[o:o + 3 * E * E].view(3, E, E); o += 3 * E * E
        wo = buf[o:o + E * E].view(E, E); o += E * E
        b = buf[o:o + 3 * E].view(3, E); o += 3 * E
        bo = buf[o:o + E]; o += E
        d = {"ln1_gain": buf[o:o + E], "ln1_bias": buf[o + E:o + 2 * E],
             "attn_q.weight": w[0], "attn_q.bias": b[0], "attn_k.weight": w[1], "attn_k.bias": b[1],
             "attn_v.weight": w[2], "attn_v.bias": b[2], "attn_out.weight": wo, "attn_out.bias": bo}
        if self.with_ffn:
            o = self._ffn0
            d["ln2_gain"] = buf[o:o + E]; o += E
            d["ln2_bias"] = buf[o:o + E]; o += E
            d["ff_in.weight"] = buf[o:o + E * F].view(E, F); o += E * F
            d["ff_in.bias"] = buf[o:o + F]; o += F
            d["ff_out.weight"] = buf[o:o + F * E].view(F, E); o += F * E
            d["ff_out.bias"] = buf[o:o + E]
        return d

    def _layer_params(self, d: dict) -> LayerParams:
        lp = LayerParams(d["ln1_gain"], d["ln1_bias"], LinearParams(d["attn_q.weight"], d["attn_q.bias"]),
                         LinearParams(d["attn_k.weight"], d["attn_k.bias"]),
                         LinearParams(d["attn_v.weight"], d["attn_v.bias"]),
                         LinearParams(d["attn_out.weight"], d["attn_out.bias"]))
        if self.with_ffn:
            lp.ln2_gain, lp.ln2_bias = d["ln2_gain"], d["ln2_bias"]
            lp.ff_in = LinearParams(d["ff_in.weight"], d["ff_in.bias"])
            lp.ff_out = LinearParams(d["ff_out.weight"], d["ff_out.bias"])
        return lp

    def grad_views(self) -> dict:
        """Gradients by reference name (model.LayerParams field order)."""
        return self._flat_views(self.grads)

    def grad_params(self) -> LayerParams:
        return self._layer_params(self.grad_views())

    # ------------------------------------------------------------ training step
    def bind_params(self, lp: LayerParams, params: torch.Tensor | None = None) -> LayerParams:
        """Copy ``lp`` into the engine's flat fp32 parameter buffer (the gradient
        layout; ``params`` may be a view into a larger model buffer) and stage it;
        returns LayerParams views of that buffer, which :meth:`optimizer_step`
        updates in place (the DistParameters of the reference)."""
        if params is not None:
            if params.numel() != self.grads.numel():
                raise ShapeError("parameter buffer does not match the gradient layout")
            self.params = params
        elif self.params is None:
            self.params = torch.zeros_like(self.grads)
        views = self._flat_views(self.params)
        for name, t in lp.named_arrays():
            if name not in views:
                raise ShapeError(f"parameter {name} has no slot (engine with_ffn={self.with_ffn})")
            views[name].copy_(t)
        self.param_lp = self._layer_params(views)
        self.load_params(self.param_lp)
        return self.param_lp

    def optimizer_step(self, opt) -> None:
        """Apply ``opt`` (optim.SGD / optim.Adam) to the bound parameters with the
        synced gradients -- hybrid.train_step's sgd_step after vertical_sync
        (hybrid.py:119-125) -- and restage the operand copies."""
        if self.params is None:
            raise ValueError("optimizer_step needs bind_params first")
        opt.step(self.params, self.grads)
        self.load_params(self.param_lp)

    def attention_work(self):
        """(rows, global position of row 0, g_begin, g_end) blocks of query rows x key
        segments this rank's attention kernels compute (own rows and delegated ones)."""
        m, pl, r, off = self.m, self.plan, self.spec.rank, self.spec.offset
        if pl.role == "heavy":
            return [(pl.split, off, pl.a, r + 1), (m - pl.split, off + pl.split, pl.b, r + 1)]
        items = [(m, off, 0, self.G)]
        if pl.role == "light":
            items.append((pl.split, pl.partner * m, 0, pl.a))
            if pl.b > 0:
                items.append((m - pl.split, pl.partner * m + pl.split, 0, pl.b))
        return items

    def needed_segments(self) -> list:
        """Key segments any of this rank's attention work reads (forward and
        backward use the same ranges); the copy-engine gather pulls only these."""
        need = set()
        for _row0, _rows, g0, g1 in self.own_ranges():  # causal-trimmed own ranges
            need.update(range(g0, g1))
        pl = self.plan
        if pl.role == "light":  # the partner's delegated rows
            need.update(range(0, max(pl.a, pl.b)))
        return sorted(need)

    def computed_pairs(self) -> int:
        """Unmasked (query, key) pairs per (batch, head) computed by this rank."""
        return sum(block_pairs(rows, p0, g0 * self.m, g1 * self.m, self.cfg.causal)
                   for rows, p0, g0, g1 in self.attention_work())

    def bind_peers(self, addrs, peer: bool) -> None:
        """addrs[g] = address of rank g's dkv_full (receive buffer); this rank's
        partial for segment g goes to slot [rank] of it."""
        slot = self.B * self.m * 2 * self.E * 4
        self.seg_dst = [int(a) + self.spec.rank * slot for a in addrs]
        self.peer_mem = peer

    def gather_slots(self) -> None:
        """Owner side of the fused reduce-scatter: dK|dV of this rank's segment =
        sum of the received slots (after the device barrier) -- only the slots of
        ranks that attend this segment are written (bwd_segments), ascending."""
        K.sum_slots(self.dkv_own, self.dkv_full, mask=self.writer_mask())

    def bwd_segments(self, rank: int | None = None):
        """Key segments [lo, hi) the backward sources of `rank` (default: this one)
        read -- the range its fused dK|dV stores cover (lss_attn_bwd_p2p)."""
        r = self.spec.rank if rank is None else rank
        G = self.G
        if not self.cfg.causal:
            return 0, G
        if rank is None:
            pl = self.plan
        else:  # every engine of the group is built with the same balance setting
            pl = make_plan(r, G, self.m, True, self.plan_bias) if self.balanced else BalancePlan()
        if pl.role == "heavy":
            return min(pl.a, pl.b), r + 1
        if pl.role == "light":
            return 0, max(r + 1, pl.a, pl.b)
        return 0, r + 1

    def writer_mask(self) -> int:
        """Bit s set iff rank s stores a partial for this rank's key segment."""
        me = self.spec.rank
        mask = 0
        for s in range(self.G):
            lo, hi = self.bwd_segments(s)
            if lo <= me < hi:
                mask |= 1 << s
        return mask

    # ------------------------------------------------------------ point-to-point exchanges
    def xfer(self, phase: str):
        """(sends, recvs) of the balanced schedule for `phase` in {"F1","F2","B1","B2"}.
        Tensors pair up positionally between this rank and plan.partner."""
        pl = self.plan
        if not pl.active:
            return [], []
        heavy = pl.role == "heavy"
        if phase == "F1":  # heavy rank's query rows -> partner
            return ([self.q], []) if heavy else ([], [self.q_peer])
        if phase == "F2":  # partner's partial contexts + lse -> heavy rank
            return ([], [self.o_help, self.lse_help]) if heavy else ([self.o_peer, self.lse_peer], [])
        if phase == "B1":  # dO, merged lse, delta of the delegated rows -> partner
            return ([self.dctx, self.lse2, self.delta], []) if heavy else \
                ([], [self.do_peer, self.lsef_peer, self.delta_peer])
        if phase == "B2":  # partner's dQ rows -> heavy rank
            return ([], [self.dq_help]) if heavy else ([self.dq_peer], [])
        raise ValueError(phase)

    # ------------------------------------------------------------ forward
    @property
    def kv_slot(self) -> torch.Tensor:
        return self.kv_full[self.spec.rank]

    def fwd_project(self, x: torch.Tensor) -> None:
        """LN1 + [Q | K_r | V_r] projection; K_r|V_r land in this rank's gather slot."""
        B, m, E = self.B, self.m, self.E
        if x.shape != (B, m, E) or x.dtype != torch.float32 or not x.is_contiguous():
            raise ShapeError(f"x must be contiguous fp32 {(B, m, E)}, got {tuple(x.shape)} {x.dtype}")
        self.x = x
        self.grads.zero_()  # every kernel of the step accumulates its pre-scaled share
        lp, st = self.lp, self.staged
        K.layernorm_fwd(x, lp.ln1_gain, lp.ln1_bias, out=self.xh, mean=self.mean, rstd=self.rstd)
        slot = self.kv_slot.view(B * m, 2 * E)
        K.gemm(self.xh.view(B * m, E), st["wqkv_t"], bias=st["bqkv"], seg_width=E,
               out=[(self.q.view(B * m, E), E), (slot[:, :E], 2 * E), (slot[:, E:], 2 * E)],
               M=B * m, N=3 * E, K=E)

    def fwd_attend(self) -> None:
        """Segment attention over the gathered K/V (own rows; plus the partner's
        delegated rows on a light rank of the balanced schedule)."""
        m, E, pl, r = self.m, self.E, self.plan, self.spec.rank
        kf, vf = self.kv_full[..., :E], self.kv_full[..., E:]
        common = dict(workers=self.G, seg_len=m, heads=self.H, causal=self.cfg.causal)
        if pl.role == "heavy":
            self._attn_part(self.q, rows=pl.split, row0=0, offset=self.spec.offset, g_begin=pl.a,
                            g_end=r + 1, out=self.ctx, lse2=self.lse2)
            self._attn_part(self.q, rows=m - pl.split, row0=pl.split, offset=self.spec.offset,
                            g_begin=pl.b, g_end=r + 1, out=self.ctx, lse2=self.lse2)
            return
        if self._dd is not None:  # dropout lives in the partial (tcgen05) launch
            self._attn_part(self.q, rows=m, row0=0, offset=self.spec.offset, g_begin=0,
                            g_end=r + 1 if self.cfg.causal else self.G, out=self.ctx, lse2=self.lse2)
        else:
            K.attn_fwd(self.q, kf, vf, offset=self.spec.offset, out=self.ctx, lse2=self.lse2, **common)
        if pl.role == "light":
            off = pl.partner * m
            self._attn_part(self.q_peer, rows=pl.split, row0=0, offset=off, g_begin=0, g_end=pl.a,
                            out=self.o_peer, lse2=self.lse_peer)
            if pl.b > 0:
                self._attn_part(self.q_peer, rows=m - pl.split, row0=pl.split, offset=off,
                                g_begin=0, g_end=pl.b, out=self.o_peer, lse2=self.lse_peer)

    def own_ranges(self):
        """(row0, rows, g_begin, g_end) blocks of this rank's own query rows."""
        m, pl, r = self.m, self.plan, self.spec.rank
        if pl.role == "heavy":
            return [(0, pl.split, pl.a, r + 1), (pl.split, m - pl.split, pl.b, r + 1)]
        return [(0, m, 0, r + 1 if self.cfg.causal else self.G)]

    def _fwd_common(self):
        E = self.E
        return (self.kv_full[..., :E], self.kv_full[..., E:],
                dict(workers=self.G, seg_len=self.m, heads=self.H, causal=self.cfg.causal, dropout=self._dd))

    def fwd_attend_own(self, part: int) -> None:
        """Own rows over every key segment they see, in ONE launch per row range
        (part 0: the first range, 1: the heavy rank's second); with the fused gather
        the kernel waits per remote segment, so no local/remote split or merge."""
        ranges = self.own_ranges()
        ranges = ranges[:1] if part == 0 else ranges[1:]
        for row0, rows, g0, g1 in ranges:
            self._attn_part(self.q, rows=rows, row0=row0, offset=self.spec.offset, g_begin=g0, g_end=g1,
                            out=self.ctx, lse2=self.lse2)

    def fwd_attend_local(self, part: int | None = None) -> None:
        """Own rows x own key segment: needs no remote K/V, so it runs while the
        all-gather (and the balanced schedule's Q hand-off) are in flight.
        ``part`` as in :meth:`fwd_attend_remote`."""
        kf, vf, common = self._fwd_common()
        r, off = self.spec.rank, self.spec.offset
        if part in (None, 0):
            self._ctx_written = set()
        ranges = self.own_ranges()
        if part is not None:
            ranges = ranges[:1] if part == 0 else ranges[1:]
        for row0, rows, g0, g1 in ranges:
            if g0 <= r < g1:
                self._attn_part(self.q, rows=rows, row0=row0, offset=off, g_begin=r, g_end=r + 1,
                                out=self.ctx, lse2=self.lse2)
                self._ctx_written.add(row0)

    def fwd_attend_remote(self, part: int | None = None) -> None:
        """Own rows x remote key segments (after the gather), log-sum-exp merged into
        ctx.  ``part`` selects the row range (0: the first, 1: the rest) so the
        heavy rank's two ranges can run on two streams."""
        kf, vf, common = self._fwd_common()
        r, off = self.spec.rank, self.spec.offset
        ranges = self.own_ranges()
        if part is not None:
            ranges = ranges[:1] if part == 0 else ranges[1:]
        for row0, rows, g0, g1 in ranges:
            for lo, hi in ((g0, min(g1, r)), (max(g0, r + 1), g1)):
                if lo >= hi:
                    continue
                if row0 not in self._ctx_written:
                    self._attn_part(self.q, rows=rows, row0=row0, offset=off, g_begin=lo, g_end=hi,
                                    out=self.ctx, lse2=self.lse2)
                    self._ctx_written.add(row0)
                    continue
                self._attn_part(self.q, rows=rows, row0=row0, offset=off, g_begin=lo, g_end=hi,
                                out=self.o_tmp, lse2=self.lse_tmp)
                K.attn_merge(self.ctx, self.lse2, self.o_tmp, self.lse_tmp, row0=row0, rows=rows, heads=self.H)

    def fwd_attend_delegated(self) -> None:
        """Light rank of the balanced schedule: the partner's delegated rows."""
        pl = self.plan
        if pl.role != "light":
            return
        kf, vf, common = self._fwd_common()
        m, off = self.m, pl.partner * self.m
        self._attn_part(self.q_peer, rows=pl.split, row0=0, offset=off, g_begin=0, g_end=pl.a,
                        out=self.o_peer, lse2=self.lse_peer)
        if pl.b > 0:
            self._attn_part(self.q_peer, rows=m - pl.split, row0=pl.split, offset=off, g_begin=0,
                            g_end=pl.b, out=self.o_peer, lse2=self.lse_peer)

    def fwd_out(self) -> torch.Tensor:
        """(merge the partner's partials,) out-projection + residual."""
        B, m, E, pl = self.B, self.m, self.E, self.plan
        if pl.role == "heavy":
            K.attn_merge(self.ctx, self.lse2, self.o_help, self.lse_help, row0=0, rows=pl.split, heads=self.H)
            if pl.b > 0:
                K.attn_merge(self.ctx, self.lse2, self.o_help, self.lse_help, row0=pl.split, rows=m - pl.split,
                             heads=self.H)
        if self._dd is not None:  # x_mid = x + dropout3(attn_out) (model.py:447-448)
            att = self._drop_tmp()
            K.gemm(self.ctx.view(B * m, E), self.staged["wo_t"], bias=self.lp.attn_out.bias, out=att,
                   M=B * m, N=E, K=E)
            self._drop_rows(att, self.y.view(B * m, E), "attn_out", residual=self.x.view(B * m, E))
            return self.y
        K.gemm(self.ctx.view(B * m, E), self.staged["wo_t"], bias=self.lp.attn_out.bias,
               residual=self.x.view(B * m, E), out=self.y.view(B * m, E), M=B * m, N=E, K=E)
        return self.y

    # ------------------------------------------------------------ FFN half (rank-local)
    def ffn_forward(self, x_mid: torch.Tensor) -> torch.Tensor:
        """LN2 -> ff_in -> GeLU -> ff_out -> residual (model.py:449-452); the GeLU and
        the pre-activation store run in the ff_in GEMM's epilogue."""
        B, m, E, F = self.B, self.m, self.E, self.cfg.ff_dim
        M = B * m
        lp = self.lp
        self.x_mid_ref = x_mid
        K.layernorm_fwd(x_mid, lp.ln2_gain, lp.ln2_bias, out=self.yh, mean=self.mean2, rstd=self.rstd2)
        K.gemm(self.yh.view(M, E), self.w_in, b_mn_major=True, bias=lp.ff_in.bias, out=self.h, act="gelu",
               pre=self.h_pre, M=M, N=F, K=E)
        if self._dd is not None:  # ffn_hidden / ffn_out sites (model.py:377, 451)
            self._drop_rows(self.h, self.h, "ffn_hidden")
            K.gemm(self.h, self.w_out, b_mn_major=True, bias=lp.ff_out.bias, out=self.y_out.view(M, E),
                   M=M, N=E, K=F)
            self._drop_rows(self.y_out.view(M, E), self.y_out.view(M, E), "ffn_out", residual=x_mid.view(M, E))
            return self.y_out
        K.gemm(self.h, self.w_out, b_mn_major=True, bias=lp.ff_out.bias, residual=x_mid.view(M, E),
               out=self.y_out.view(M, E), M=M, N=E, K=F)
        return self.y_out

    def ffn_backward(self, grad_out: torch.Tensor) -> torch.Tensor:
        """Backward of :meth:`ffn_forward` (model.py:474-477): returns grad_mid =
        grad_out + LN2'(FFN'(grad_out)); grads pre-scaled into the flat buffer."""
        B, m, E, F = self.B, self.m, self.E, self.cfg.ff_dim
        M = B * m
        a = self.grad_scale
        lp = self.lp
        if grad_out.shape != (B, m, E) or grad_out.dtype != torch.float32 or not grad_out.is_contiguous():
            raise ShapeError(f"grad_y must be contiguous fp32 {(B, m, E)}")
        g32 = grad_out.view(M, E)
        g_ffn = self._drop_rows(g32, self._drop_tmp(), "ffn_out") if self._dd is not None else g32
        K.cat_cast_colsum([(g_ffn, E, E)], M, dst=self.g_out, colsum=self.g_bout, alpha=a)
        K.gemm(self.g_out, self.w_out, out=self.g_pre32, act="gelu_bwd", aux=self.h_pre, M=M, N=F, K=E)
        if self._dd is not None:  # dropout_bwd(ffn_hidden): elementwise, commutes with GeLU'
            self._drop_rows(self.g_pre32, self.g_pre32, "ffn_hidden")
        K.gemm(self.h, self.g_out, a_mn_major=True, b_mn_major=True, alpha=a, out=self.g_wout, M=F, N=E, K=M)
        K.cat_cast_colsum([(self.g_pre32, F, F)], M, dst=self.g_pre, colsum=self.g_bin, alpha=a)
        K.gemm(self.g_pre, self.w_in, out=self.g_yh, M=M, N=E, K=F)
        K.gemm(self.yh.view(M, E), self.g_pre, a_mn_major=True, b_mn_major=True, alpha=a, out=self.g_win,
               M=E, N=F, K=M)
        K.layernorm_bwd(self.g_yh, self.x_mid_ref.view(M, E), self.mean2, self.rstd2, lp.ln2_gain,
                        grad_res=g32, grad_x=self.grad_mid.view(M, E), grad_gain=self.g_ln2_g,
                        grad_bias=self.g_ln2_b, alpha=a)
        return self.grad_mid

    # ------------------------------------------------------------ backward
    def bwd_pre(self, grad_y: torch.Tensor) -> None:
        """Out-projection backward (+ the delta row term in the balanced schedule)."""
        B, m, E = self.B, self.m, self.E
        if grad_y.shape != (B, m, E) or grad_y.dtype != torch.float32 or not grad_y.is_contiguous():
            raise ShapeError(f"grad_y must be contiguous fp32 {(B, m, E)}")
        self.grad_y = grad_y
        a = self.grad_scale
        # gy -> operand dtype, d b_out = alpha * column sums (nnops.py:192)
        g_att = grad_y.view(B * m, E)
        if self._dd is not None:  # dropout3_bwd(attn_out), model.py:479; LN1 keeps the unmasked residual
            g_att = self._drop_rows(g_att, self._drop_tmp(), "attn_out")
        K.cat_cast_colsum([(g_att, E, E)], B * m, dst=self.gy.view(B * m, E), colsum=self.g_bo, alpha=a)
        # dctx = gy . Wo^T  (Wo [in][out] is the K-major B operand)
        K.gemm(self.gy.view(B * m, E), self.staged["wo"], out=self.dctx.view(B * m, E), M=B * m, N=E, K=E)
        if self.plan.active or self.seg_dst is not None or self._dd is not None or K.deterministic():
            K.attn_delta(self.ctx, self.dctx, self.delta, heads=self.H, scaled=True)

    def _wgrad_stream(self) -> torch.cuda.Stream:
        """Side stream for the weight-gradient GEMMs: their output grids are small
        (E/128 x N/256 tiles, 32-96 CTAs), so they run beside the attention backward /
        the input-gradient GEMM instead of leaving most SMs idle."""
        if not self.options.wgrad_side:
            return torch.cuda.current_stream()
        if getattr(self, "_wstream", None) is None:
            self._wstream = torch.cuda.Stream(device=self.device)
        return self._wstream

    def bwd_pre_weights(self) -> None:
        """dWo = ctx^T . gy (both operands MN-major), pre-scaled, on the weight-gradient
        stream (overlaps the dO / lse / delta hand-off and the attention backward)."""
        B, m, E = self.B, self.m, self.E
        ws = self._wgrad_stream()
        ws.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(ws):
            K.gemm(self.ctx.view(B * m, E), self.gy.view(B * m, E), a_mn_major=True, b_mn_major=True,
                   alpha=self.grad_scale, out=self.g_wo, M=E, N=E, K=B * m)

    def bwd_attend(self, peer_ready=None) -> None:
        """Attention backward: dQ for the rows this rank computes, partial dK|dV for all.
        ``peer_ready`` = (flag address, seq): the partner's dO / lse / delta are still
        being pushed; the kernel runs the own rows first and waits for them in-kernel."""
        m, E, pl, r = self.m, self.E, self.plan, self.spec.rank
        kf, vf = self.kv_full[..., :E], self.kv_full[..., E:]
        if self.seg_dst is not None:  # fused reduce-scatter: dK|dV straight to the owners
            out = dict(seg_dst=self.seg_dst, peer=self.peer_mem, ld_dkv=2 * E)
        else:
            out = dict(grad_k=self.dkv_full[..., :E], grad_v=self.dkv_full[..., E:])
        det = K.deterministic()  # fixed-point dQ (integer adds): bitwise repeatable
        if not pl.active and self.seg_dst is None and self._dd is None and not det:
            K.attn_bwd(self.q, kf, vf, self.ctx, self.dctx, self.lse2, workers=self.G, seg_len=m,
                       heads=self.H, offset=self.spec.offset, causal=self.cfg.causal, grad_q=self.dq,
                       grad_k=self.dkv_full[..., :E], grad_v=self.dkv_full[..., E:], delta=self.delta)
            return
        own = dict(q=self.q, grad_o=self.dctx, grad_q=self.dq, pos0=self.spec.offset, lse2=self.lse2,
                   delta=self.delta)
        if det:
            if getattr(self, "dq64", None) is None:
                self.dq64 = torch.empty(self.dq.shape, dtype=torch.int64, device=self.device)
            self.dq64.zero_()
            own["grad_q_fixed"] = self.dq64
        else:
            self.dq.zero_()
        if pl.role == "heavy":
            srcs = [dict(own, row0=0, rows=pl.split, g_begin=pl.a, g_end=r + 1),
                    dict(own, row0=pl.split, rows=m - pl.split, g_begin=pl.b, g_end=r + 1)]
        elif pl.role == "light":
            peer = dict(q=self.q_peer, grad_o=self.do_peer, grad_q=self.dq_peer, pos0=pl.partner * m,
                        lse2=self.lsef_peer, delta=self.delta_peer, ready=peer_ready)
            if det:
                if getattr(self, "dq_peer64", None) is None:
                    self.dq_peer64 = torch.empty(self.dq_peer.shape, dtype=torch.int64, device=self.device)
                self.dq_peer64.zero_()
                peer["grad_q_fixed"] = self.dq_peer64
            else:
                self.dq_peer.zero_()
            srcs = [dict(own, row0=0, rows=m, g_begin=0, g_end=r + 1),
                    dict(peer, row0=0, rows=pl.split, g_begin=0, g_end=pl.a)]
            if pl.b > 0:
                srcs.append(dict(peer, row0=pl.split, rows=m - pl.split, g_begin=0, g_end=pl.b))
        else:
            srcs = [dict(own, row0=0, rows=m, g_begin=0, g_end=self.G if not self.cfg.causal else r + 1)]
        K.attn_bwd_sources(kf, vf, srcs, workers=self.G, seg_len=m, heads=self.H, causal=self.cfg.causal,
                           dropout=self._dd, **out)
        if det:
            K.fixed_to_f32(self.dq, self.dq64)
            if pl.role == "light":
                K.fixed_to_f32(self.dq_peer, self.dq_peer64)

    def bwd_fold(self) -> None:
        """Heavy rank of the balanced schedule: fold the partner's dQ rows in."""
        if self.plan.role == "heavy":
            K.add_(self.dq, self.dq_help)

    def bwd_project(self) -> torch.Tensor:
        """After the reduce-scatter: [dQ|dK|dV] -> dx̂ and dW_qkv, LN1 backward + residual."""
        B, m, E = self.B, self.m, self.E
        a = self.grad_scale
        M = B * m
        if self._slots_pending:  # fused reduce-scatter: sum the writers' slots inside the cast
            dkv = (self.dkv_full, 2 * E, 2 * E, self.G, self.writer_mask(), self.dkv_full[0].numel())
            self._slots_pending = False
        else:
            dkv = (self.dkv_own.view(M, 2 * E), 2 * E, 2 * E)
        K.cat_cast_colsum([(self.dq.view(M, E), E, E), dkv], M,
                          dst=self.dqkv.view(M, 3 * E), colsum=self.g_bqkv, alpha=a)
        main, ws = torch.cuda.current_stream(), self._wgrad_stream()
        ws.wait_stream(main)
        with torch.cuda.stream(ws):  # dW_qkv (96 tiles) beside the dx̂ GEMM
            gw = self.g_wqkv.view(3, E, E)
            K.gemm(self.xh.view(M, E), self.dqkv.view(M, 3 * E), a_mn_major=True, b_mn_major=True, alpha=a,
                   seg_width=E, out=[(gw[0], E), (gw[1], E), (gw[2], E)], M=E, N=3 * E, K=M)
        K.gemm(self.dqkv.view(M, 3 * E), self.staged["wqkv"], out=self.dxh.view(M, E), M=M, N=E, K=3 * E)
        K.layernorm_bwd(self.dxh.view(M, E), self.x.view(M, E), self.mean, self.rstd, self.lp.ln1_gain,
                        grad_res=self.grad_y.view(M, E), grad_x=self.dx.view(M, E),
                        grad_gain=self.g_ln_g, grad_bias=self.g_ln_b, alpha=a)
        main.wait_stream(ws)  # every weight gradient is in the flat buffer before the all-reduce
        return self.dx

    # ------------------------------------------------------------ public step API
    def step(self, x: torch.Tensor, grad_y: torch.Tensor, comm, *, step: int = 0, layer: int = 0,
             sync: bool = True, policy=None):
        """Forward + backward (+ folded gradient sync) of this rank's block, device
        tensors in and out.  Returns (y, dx); gradients are in ``grads`` /
        ``grad_views()`` (already averaged over the group(s) when sync=True)."""
        (y, dx), = lss_step([self], comm, [x], [grad_y], step=step, layer=layer, sync=sync, policy=policy)
        return y, dx

    def step_from_host(self, x_host: torch.Tensor, grad_y_host: torch.Tensor, comm, grads_host=None,
                       *, step: int = 0, layer: int = 0, next_inputs=None, policy=None):
        """End-to-end call with HOST buffers: pinned x / grad_y are copied in and the
        averaged gradients are copied back to ``grads_host`` (pinned).  Inputs are
        double-buffered: with ``next_inputs`` = (x_host, grad_y_host) of the NEXT
        step, their copy is issued on the copy stream during this step's compute
        (input prefetch), and the next call finds them resident.  Every step's
        inputs are still copied once, by this engine, per step.  Stream-ordered;
        the gradient read-back runs on the copy stream (overlapping the next step):
        the caller synchronises the device, or waits on :meth:`host_sync_event`,
        before reading ``grads_host``."""
        cur = torch.cuda.current_stream()
        if not hasattr(self, "_in_bufs"):
            mk = lambda: torch.empty(self.B, self.m, self.E, dtype=torch.float32, device=self.device)  # noqa: E731
            self._in_bufs = [(mk(), mk()), (mk(), mk())]
            self._in_ready = [torch.cuda.Event(), torch.cuda.Event()]   # x of the slot resident
            self._gy_ready = [torch.cuda.Event(), torch.cuda.Event()]   # grad_y of the slot resident
            self._in_free = [torch.cuda.Event(), torch.cuda.Event()]
            self._copy_stream = torch.cuda.Stream(device=self.device)
            self._prefetched = None  # (slot, x_host, grad_y_host) already in flight
            self._slot = 0

        def issue(slot, xh, gyh):
            cs = self._copy_stream
            cs.wait_stream(cur)
            cs.wait_event(self._in_free[slot])  # the step that last read this slot is done
            with torch.cuda.stream(cs):
                x_d, gy_d = self._in_bufs[slot]
                x_d.copy_(xh, non_blocking=True)
                self._in_ready[slot].record()
                gy_d.copy_(gyh, non_blocking=True)  # needed only by the backward: lands under the forward
                self._gy_ready[slot].record()

        pf = self._prefetched
        if pf is not None and pf[1] is x_host and pf[2] is grad_y_host:
            slot = pf[0]
        else:
            slot = self._slot
            issue(slot, x_host, grad_y_host)
        self._prefetched = None
        prefetch = None
        if next_inputs is not None:  # overlap the next step's H2D with this step's backward
            nxt = 1 - slot
            # issued between the forward and the backward: the forward's copy-engine
            # gather and hand-offs then never queue behind the host copy
            prefetch = lambda: issue(nxt, *next_inputs)  # noqa: E731
            self._prefetched = (nxt, next_inputs[0], next_inputs[1])
        self._slot = 1 - slot
        cur.wait_event(self._in_ready[slot])
        x_d, gy_d = self._in_bufs[slot]
        if prefetch is not None and not self.options.prefetch_at_bwd:
            prefetch()
            prefetch = None
        gy_ev = self._gy_ready[slot]

        def before_bwd():
            cur.wait_event(gy_ev)  # grad_y's copy overlapped the forward
            if prefetch is not None:
                prefetch()

        out = lss_step([self], comm, [x_d], [gy_d], step=step, layer=layer, policy=policy, before_bwd=before_bwd)
        self._in_free[slot].record(cur)
        if grads_host is not None:
            # read-back off the critical path: snapshot the averaged gradients on the
            # compute stream (D2D), then D2H on the copy stream, overlapping the next
            # step (whose first kernel re-zeroes self.grads)
            if getattr(self, "_grads_stage", None) is None:
                self._grads_stage = torch.empty_like(self.grads)
                self._d2h_done = torch.cuda.Event()
                self._d2h_done.record(cur)
            cur.wait_event(self._d2h_done)  # previous read-back finished with the stage
            self._grads_stage.copy_(self.grads)
            cs = self._copy_stream
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                grads_host.copy_(self._grads_stage, non_blocking=True)
                self._d2h_done.record(cs)
        return out[0]

    def host_sync_event(self) -> torch.cuda.Event | None:
        """Event after the last step_from_host read-back (None before the first):
        the caller waits on it (or synchronises) before reading grads_host."""
        return getattr(self, "_d2h_done", None)


# ---------------------------------------------------------------- drivers


_CHANNEL = {"F1": 2, "F2": 3, "B1": 4, "B2": 5}  # flag-board channels of the hand-offs


def _ce_targets(e, comm):
    """The partner's receive buffers of every hand-off phase, mapped into this process
    once (collective over the sequence group); False when the fabric cannot."""
    if getattr(e, "_ce_map", None) is None:
        e._ce_map = False
        if hasattr(comm, "flags_ready") and comm.flags_ready():
            named = {}
            for ph in _CHANNEL:
                for i, t in enumerate(e.xfer(ph)[1]):
                    named[f"{ph}:{i}"] = t
            addrs = comm.map_named(named)
            if addrs is not None:
                e._ce_map = addrs[e.plan.partner] if e.plan.active else {}
    return e._ce_map


def _exchange_ce(e, comm, phase, step, layer):
    """Hand-off on the copy engines: the sender pushes its tensors into the partner's
    receive buffers (peer memory) on a push stream and signals the partner's flag;
    the receiver gets a handle whose wait() blocks its stream on that flag.  No SM
    and no NCCL kernel is involved.  Every push is enqueued after the forward's
    group barrier, which the partner has passed only after finishing the previous
    step's reads of its receive buffers."""
    sends, recvs = e.xfer(phase)
    ch = _CHANNEL[phase]
    if sends:
        ps = comm.push_stream()
        ps.wait_stream(torch.cuda.current_stream())
        for i, t in enumerate(sends):
            K.copy_d2d(e._ce_map[f"{phase}:{i}"], t.data_ptr(), t.numel() * t.element_size(), ps)
        comm.notify(e.plan.partner, ch, ps)
        comm.ledger.record("send", comm.seq_name + ":ce", sum(t.numel() for t in sends), step, phase, layer)
    if recvs:
        comm.ledger.record("recv", comm.seq_name + ":ce", sum(t.numel() for t in recvs), step, phase, layer)
        return [comm.expect(e.plan.partner, ch)]
    return []


def _exchange(engines, comm, phase, step, layer, async_op=False):
    """Balanced-schedule point-to-point phase; returns the pending works (async_op)."""
    if engines[0].options.ce_p2p and not isinstance(comm, SimComm) and len(engines) == 1 and _ce_targets(engines[0], comm):
        works = _exchange_ce(engines[0], comm, phase, step, layer)
        if not async_op:
            _wait(works)
            return []
        return works
    if isinstance(comm, SimComm):
        for e in engines:
            sends, _ = e.xfer(phase)
            if not sends:
                continue
            _, recvs = engines[e.plan.partner].xfer(phase)
            for src, dst in zip(sends, recvs):
                dst.copy_(src)
            comm.ledger.record("send", "sequence", sum(t.numel() for t in sends), step, phase, layer)
        return []
    works = []
    for e in engines:
        sends, recvs = e.xfer(phase)
        if sends or recvs:
            w = comm.p2p(sends, recvs, e.plan.partner, step=step, phase=phase, layer=layer, async_op=async_op)
            works.extend(w or [])
    return works


def _wait(works) -> None:
    """Make the current stream wait for pending collectives / copy events (no host block)."""
    for w in works or []:
        if isinstance(w, torch.cuda.Event):
            torch.cuda.current_stream().wait_event(w)
        elif w is not None:
            w.wait()


def _bind_fused(engines, comm) -> bool:
    """Enable the fused dK|dV reduce-scatter when every engine wants it and the
    fabric can map the peers' receive buffers (same device in the simulation,
    CUDA IPC over NVLink for real ranks)."""
    if not all(e.fused_rs for e in engines):
        return False
    if all(e.seg_dst is not None for e in engines):
        return True
    if isinstance(comm, SimComm):
        addrs = [e.dkv_full.data_ptr() for e in engines]
        for e in engines:
            e.bind_peers(addrs, peer=False)
        return True
    if not hasattr(comm, "peer_addresses"):
        return False
    e = engines[0]
    addrs = comm.peer_addresses(e.dkv_full)
    if addrs is None:
        for e in engines:
            e.fused_rs = False
        return False
    e.bind_peers(addrs, peer=True)
    return True


def layer_grad_size(cfg: ModelConfig, with_ffn: bool) -> int:
    """Elements of one engine's flat gradient buffer (LSSAttention layout)."""
    E, F = cfg.embed_dim, cfg.ff_dim
    n_attn = 4 * E * E + 6 * E + 1
    return (n_attn + 15) // 16 * 16 + (2 * E * F + F + 3 * E) if with_ffn else n_attn


class PhaseClock:
    """Opt-in (EngineOptions.phases=1) per-phase CUDA-event timeline of lss_step; the
    bench prints it to explain where a multi-GPU step goes.  phases=2 also stamps
    the GPU global timer at every mark (``last_stamps``), comparable across ranks."""

    def __init__(self, stamps: bool = False):
        self.marks = []
        self.stamps = torch.zeros(128, dtype=torch.int64, device="cuda") if stamps else None

    def mark(self, name):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        if self.stamps is not None and len(self.marks) < self.stamps.numel():
            K.timestamp(self.stamps[len(self.marks)])
        self.marks.append((name, ev))

    def report(self):
        torch.cuda.synchronize()
        global last_stamps
        if self.stamps is not None:
            ns = self.stamps.cpu().tolist()
            last_stamps = [(n, ns[i]) for i, (n, _) in enumerate(self.marks)]
        return {n: self.marks[i - 1][1].elapsed_time(ev) for i, (n, ev) in enumerate(self.marks) if i > 0}


last_stamps: list = []
last_clock = None
last_phases: dict = {}


def _no_mark(name):
    return None


_SIDE = {}


def _side_stream(device) -> torch.cuda.Stream:
    """One side stream per device for concurrent attention launches."""
    key = torch.device(device).index
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=device)
    return _SIDE[key]


def lss_forward(engines, comm, xs, *, step=0, layer=0, mark=_no_mark):
    """Forward of one layer on every engine (model.layer_fwd distributed, the
    fwd half of sharded.forward): LN1, [Q|K|V], the packed K/V all-gather
    overlapped with the diagonal segment, attention, out-projection + residual,
    and the LN2 / FFN half for complete-layer engines.  Returns the outputs."""
    sim = isinstance(comm, SimComm)
    one = lambda f: f([e for e in engines]) if sim else f(engines[0])  # noqa: E731
    opts = engines[0].options
    split = all(e.split_fwd for e in engines)
    for e, x in zip(engines, xs):
        e.fwd_project(x)
    mark("fwd_project")
    gather = None
    fused = False
    if not sim and split and opts.ce_gather and hasattr(comm, "gather_pull") and comm.seq_size > 1:
        e0 = engines[0]
        ready = None
        if opts.fused_gather and not opts.no_overlap and comm.flags_ready():
            e0._ready_seq += 1
            ready = (e0._ready, e0._ready_seq)
        gather = comm.gather_pull(e0.kv_full, step, layer,  # copy engines, no SMs
                                  segments=e0.needed_segments(), ready=ready)
        mark("gather_barrier")
        if gather is not None and ready is not None:
            fused = True
            e0._ready_tok = (e0._ready, e0._ready_seq, e0.spec.rank)
    if fused:
        # all-gather fused into the attention: every launch starts at once and its
        # producer warp waits per remote segment; own rows in one launch per range
        # (main stream / side stream), the light rank's delegated rows on the side
        # stream after the Q hand-off, their partials pushed back right after
        e0 = engines[0]
        f1 = _exchange(engines, comm, "F1", step, layer, async_op=True)
        main = torch.cuda.current_stream()
        side = _side_stream(e0.device)
        side.wait_stream(main)
        e0.fwd_attend_own(part=0)
        with torch.cuda.stream(side):
            _wait(f1)
            e0.fwd_attend_delegated()
            e0.fwd_attend_own(part=1)
            f2 = _exchange(engines, comm, "F2", step, layer, async_op=True)
        main.wait_stream(side)
        mark("fwd_attend")
        _wait(f2)
        _wait([gather])  # every segment resident before the backward reads them
        e0._ready_tok = None
        mark("p2p_F2")
        ys = [e.fwd_out() for e in engines]
        mark("fwd_out")
        if all(e.with_ffn for e in engines):
            ys = [e.ffn_forward(y) for e, y in zip(engines, ys)]
            mark("ffn_fwd")
        return ys
    if gather is None:
        gather = one(lambda t: comm.all_gather_rows([e.kv_full for e in t] if sim else t.kv_full, step, layer,
                                                    **({} if sim else {"async_op": split})))
    f1 = _exchange(engines, comm, "F1", step, layer, async_op=split)
    if opts.no_overlap:  # diagnostic: serialise the collectives with the compute
        _wait([gather] + f1)
        gather, f1 = None, []
    if split:
        # diagonal segment while the gather / Q hand-off are in flight; the light
        # rank then does the partner's rows first so their partials travel back
        # while it finishes its own remote segments
        main = torch.cuda.current_stream()
        side = _side_stream(engines[0].device)
        for e in engines:
            e.fwd_attend_local(part=0)
        side.wait_stream(main)
        with torch.cuda.stream(side):  # the heavy rank's second row range
            for e in engines:
                e.fwd_attend_local(part=1)
        main.wait_stream(side)
        mark("fwd_local")
        _wait([gather] + f1)
        mark("all_gather")
        # two streams so the launches' tails overlap: the light rank's delegated rows
        # (whose partials then travel back) and the heavy rank's second row range on
        # a side stream, own rows on the main stream
        side.wait_stream(main)
        with torch.cuda.stream(side):
            for e in engines:
                e.fwd_attend_delegated()
                e.fwd_attend_remote(part=1)
            f2 = _exchange(engines, comm, "F2", step, layer, async_op=True)
        for e in engines:
            e.fwd_attend_remote(part=0)
        main.wait_stream(side)
        mark("fwd_attend")
        _wait(f2)
        mark("p2p_F2")
    else:
        _wait([gather] + f1)
        mark("all_gather")
        for e in engines:
            e.fwd_attend()
        mark("fwd_attend")
        _exchange(engines, comm, "F2", step, layer)
        mark("p2p_F2")
    ys = [e.fwd_out() for e in engines]
    mark("fwd_out")
    if all(e.with_ffn for e in engines):  # complete layer: rank-local LN2 / FFN half
        ys = [e.ffn_forward(y) for e, y in zip(engines, ys)]
        mark("ffn_fwd")
    return ys


def lss_backward(engines, comm, grad_ys, *, step=0, layer=0, sync=True, mark=_no_mark):
    """Backward of one layer (model.layer_bwd distributed, the bwd half of
    sharded.backward): FFN / LN2 half, out-projection, attention backward with the
    dK|dV reduce-scatter (fused into the kernel over NVLink when the peers map),
    projections, LN1 + residual; with ``sync`` the folded gradient all-reduce.
    Returns the input gradients."""
    sim = isinstance(comm, SimComm)
    one = lambda f: f([e for e in engines]) if sim else f(engines[0])  # noqa: E731
    opts = engines[0].options
    fused = _bind_fused(engines, comm)
    if all(e.with_ffn for e in engines):
        grad_ys = [e.ffn_backward(gy) for e, gy in zip(engines, grad_ys)]
        mark("ffn_bwd")
    for e, gy in zip(engines, grad_ys):
        e.bwd_pre(gy)
    b1 = _exchange(engines, comm, "B1", step, layer, async_op=True)
    for e in engines:
        e.bwd_pre_weights()
    mark("bwd_pre")
    peer_ready = None
    if opts.b1_in_kernel and len(engines) == 1 and b1 and all(hasattr(w, "addr") for w in b1):  # wait in-kernel
        peer_ready = (b1[0].addr, b1[0].seq)
    else:
        _wait(b1)
    mark("p2p_B1")
    for e in engines:
        e.bwd_attend(peer_ready=peer_ready)
    mark("bwd_attend")
    b2 = _exchange(engines, comm, "B2", step, layer, async_op=True)
    if fused:  # the reduce-scatter already happened inside the backward kernels
        comm.ledger.record("reduce-scatter", "sequence:nvlink", engines[0].dkv_full.numel(), step, "backward",
                           layer)
        if not sim and comm.flags_ready() and comm.use_flags:
            comm.flag_barrier(1, step, "backward", layer)
        else:
            comm.device_barrier(step, "backward", layer)
        mark("rs_barrier")
        for e in engines:
            if opts.fold_slots:
                e._slots_pending = True  # summed inside bwd_project's cast (no dK|dV round trip)
            else:
                e.gather_slots()
    else:
        one(lambda t: comm.reduce_scatter_rows([e.dkv_own for e in t] if sim else t.dkv_own,
                                               [e.dkv_full for e in t] if sim else t.dkv_full, step, layer))
    mark("reduce_scatter")
    _wait(b2)
    for e in engines:
        e.bwd_fold()
    mark("p2p_B2")
    dxs = [e.bwd_project() for e in engines]
    mark("bwd_project")
    if sync:
        one(lambda t: comm.all_reduce_sum([e.grads for e in t] if sim else t.grads, step))
    mark("all_reduce")
    return dxs


def lss_step(engines, comm, xs, grad_ys, *, step=0, layer=0, sync=True, before_bwd=None, policy=None):
    """One fwd+bwd(+sync) of the layer (attention sublayer, or the complete layer
    for with_ffn engines).

    Real multi-GPU: ``engines`` = [this rank's LSSAttention], ``comm`` a
    TorchDistComm (or SoloComm for one rank).  Single-process simulation: G
    engines and a SimComm.  Returns the list of (y, dx) per engine (device
    tensors, not synchronised).  ``policy``: dropout (dropout.DropoutPolicy or a
    rate; None = off), as model.layer_fwd's ``policy, layer`` -- used as given;
    multi-step drivers derive ``policy.at_step(step).fork(replica)`` per step
    (hybrid.run_engine_steps, sharded.run_steps)."""
    global last_phases
    if hasattr(comm, "check"):
        comm.check()  # a wait of the previous step ran past its deadline -> CommTimeout
    for e in engines:
        e.set_dropout(policy, layer)
    phases = engines[0].options.phases
    clk = PhaseClock(phases == 2) if phases else None
    mark = clk.mark if clk else _no_mark
    _bind_fused(engines, comm)
    mark("start")
    ys = lss_forward(engines, comm, xs, step=step, layer=layer, mark=mark)
    if before_bwd is not None:
        before_bwd()
    dxs = lss_backward(engines, comm, grad_ys, step=step, layer=layer, sync=sync, mark=mark)
    if clk:
        if clk.stamps is not None:  # phases=2: the caller reports (steady-state steps, no sync here)
            global last_clock
            last_clock = clk
        else:
            last_phases = clk.report()
    if K.numerics_enabled():  # opt-in NaN / Inf check of every kernel output (tensor.py:79-95)
        torch.cuda.current_stream().synchronize()
        K.raise_status()
    return list(zip(ys, dxs))


def make_sim_group(cfg: ModelConfig, lp: LayerParams, workers: int, *, replicas: int = 1, device=None,
                   balanced: bool | None = None, fused_rs: bool | None = None, options: EngineOptions | None = None):
    """G engines of one sequence group on one device (tests / smoke), SimComm fabric.
    LayerParams with the FFN half build complete-layer engines."""
    engines = []
    for r in range(workers):
        e = LSSAttention(cfg, ShardSpec(r, workers, cfg.seq_len), grad_scale=1.0 / (workers * replicas),
                         device=device, balanced=balanced, fused_rs=fused_rs, with_ffn=lp.has_ffn, options=options)
        e.load_params(lp)
        engines.append(e)
    return engines, SimComm(Ledger())


__all__ = ["EngineOptions", "LSSAttention", "lss_forward", "lss_backward", "lss_step", "make_sim_group",
           "layer_grad_size", "GRAD_NAMES"]
